// k_encode.cuh — K4 kernels and their launchers (templates).  The
// instantiations for each index length B are spread over k_encode_b*.cu so
// the 2 dtypes x 29 B x {plain, fused reconstruction} kernels compile in
// parallel; k_encode.cu holds the dispatch, finalize and the C-ABI.
#pragma once

// k_encode.cu — K4: fused classify + round-trip filter + B-bit packing +
// stable compaction of the incompressible values.
//
// One pass over both snapshots replaces phases 3a, 3b and 4a of
// compress_pair (pkg/src/nmk/pipeline.py:232-288):
//   nearest_center + compressible_mask (binning.py:287-301, 350-359),
//   _roundtrip_filter (pipeline.py:143-160), the sentinel substitution,
//   the element-order compaction current[~flags] and the per-block
//   incompressible prefix (pipeline.py:257-276), and pack_block MSB-first
//   (codec.py:83-92) into the block layout of codec.BlockLayout (codec.py:28-59).
//
// Work unit: a CHUNK of 256 elements = one warp x 8 consecutive elements per
// lane, laid on the grid of index blocks (chunks never straddle a block), so
// each lane's 8 codes are exactly B whole bytes of its block and a chunk's
// 32*B bytes start 16-byte aligned.  Warps run independently (no block-wide
// barrier): a chunk writes its packed bytes, its incompressible count and
// its incompressible values into its own 256-slot scratch window.  A short
// finalize pass (k_scan.cu + k_enc_finalize) turns the counts into positions,
// moves the (rare) values into the compacted list and fills the per-block
// prefix table.
#include "nmk_common.cuh"
#include "nmk_scan.cuh"

namespace nmk {

constexpr int kChunk = 32 * kGroup;   // 256 elements per warp chunk
constexpr int kEncThreads = 256;      // 8 warps per CTA
#ifndef NMK_ENC_MINB
#define NMK_ENC_MINB 4   // 64 registers: measured best (3 -> 85 regs is slower)
#endif
constexpr int kSmemCuts = 4096;       // cuts in shared memory up to this many

template <int B>
__device__ __forceinline__ void pack8(const uint32_t (&code)[kGroup], uint8_t* dst) {
  // MSB-first bit string of 8 codes = B bytes; B is a compile-time constant
  // so every shift below resolves statically.
  uint8_t out[B];
  unsigned long long acc = 0;
  int nacc = 0, ob = 0;
#pragma unroll
  for (int e = 0; e < kGroup; ++e) {
    acc = (acc << B) | code[e];
    nacc += B;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (nacc >= 8) {
        out[ob++] = (uint8_t)(acc >> (nacc - 8));
        nacc -= 8;
      }
    }
  }
  // widest aligned store the byte offset lane*B allows
  if constexpr (B % 16 == 0) {
#pragma unroll
    for (int w = 0; w < B / 16; ++w) {
      uint4 v;
      uint32_t* p = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        p[q] = out[w * 16 + q * 4] | (out[w * 16 + q * 4 + 1] << 8) | (out[w * 16 + q * 4 + 2] << 16) |
               ((uint32_t)out[w * 16 + q * 4 + 3] << 24);
      reinterpret_cast<uint4*>(dst)[w] = v;
    }
  } else if constexpr (B % 8 == 0) {
#pragma unroll
    for (int w = 0; w < B / 8; ++w) {
      uint2 v;
      v.x = out[w * 8] | (out[w * 8 + 1] << 8) | (out[w * 8 + 2] << 16) | ((uint32_t)out[w * 8 + 3] << 24);
      v.y = out[w * 8 + 4] | (out[w * 8 + 5] << 8) | (out[w * 8 + 6] << 16) | ((uint32_t)out[w * 8 + 7] << 24);
      reinterpret_cast<uint2*>(dst)[w] = v;
    }
  } else if constexpr (B % 4 == 0) {
#pragma unroll
    for (int w = 0; w < B / 4; ++w)
      reinterpret_cast<uint32_t*>(dst)[w] =
          out[w * 4] | (out[w * 4 + 1] << 8) | (out[w * 4 + 2] << 16) | ((uint32_t)out[w * 4 + 3] << 24);
  } else if constexpr (B % 2 == 0) {
#pragma unroll
    for (int w = 0; w < B / 2; ++w)
      reinterpret_cast<uint16_t*>(dst)[w] = (uint16_t)(out[w * 2] | (out[w * 2 + 1] << 8));
  } else {
#pragma unroll
    for (int w = 0; w < B; ++w) dst[w] = out[w];
  }
}

// K1's f32 ratio keys for the keyed mode (keys == nullptr: read the snapshots)
struct EncodeKeys {
  const float* keys;
  const nmk_stats* st;   // gmin, gmax, dense span (stats->reserved)
  double width;          // histogram width 2E
  uint32_t* done;        // device flag: 1 when the keyed kernel did the work (2: on its exact path only)
  int only;              // no k_encode launch follows: the keyed kernel always does the work
};

struct EncodeGeom {
  uint64_t n_local, elem0, n_total, epb, cpb, g0, nchunks, b0, stride;
  FastDiv fd_cpb;   // chunk id -> block
  // keyed K4: chunks c_first..c_last are wholly inside [elem0, elem0 + n_local);
  // key_al: every chunk start is a multiple of 4 elements from elem0
  uint32_t c_first, c_last;
  bool key_al;
  ZeroList zl;   // the chunk scan's tile status, zeroed by the encode kernels
};

// Chunk c of this range: block, in-block chunk index and element spans.
struct ChunkSpan {
  uint64_t b, ci, blk_start, blk_end, lo, hi, chunk_lo;
};

__device__ __forceinline__ ChunkSpan chunk_span(const EncodeGeom& geo, uint64_t c) {
  ChunkSpan s;
  const uint64_t g = geo.g0 + c;
  s.b = g / geo.cpb;
  s.ci = g - s.b * geo.cpb;
  s.blk_start = s.b * geo.epb;
  s.blk_end = s.blk_start + geo.epb;
  if (s.blk_end > geo.n_total) s.blk_end = geo.n_total;
  s.chunk_lo = s.blk_start + s.ci * kChunk;
  uint64_t chunk_hi = s.chunk_lo + kChunk;
  if (chunk_hi > s.blk_end) chunk_hi = s.blk_end;
  const uint64_t local_end = geo.elem0 + geo.n_local;
  s.lo = s.chunk_lo > geo.elem0 ? s.chunk_lo : geo.elem0;
  s.hi = chunk_hi < local_end ? chunk_hi : local_end;
  return s;
}

template <typename T> struct EVec;
template <> struct EVec<double> { using V = double2; static constexpr int N = 2; };
template <> struct EVec<float>  { using V = float4;  static constexpr int N = 4; };

template <typename T>
__device__ __forceinline__ void load8(const T* __restrict__ p, T (&v)[kGroup]) {
  using V = typename EVec<T>::V;
  constexpr int VN = EVec<T>::N;
#pragma unroll
  for (int q = 0; q < kGroup / VN; ++q) {
    V w = __ldg(reinterpret_cast<const V*>(p) + q);
    const T* t = reinterpret_cast<const T*>(&w);
#pragma unroll
    for (int e = 0; e < VN; ++e) v[q * VN + e] = t[e];
  }
}

// Per-element classification: returns the code (idx or sentinel).
template <typename T, typename Find>
__device__ __forceinline__ uint32_t classify(T bt, T xt, Find&& find, const double* __restrict__ centers,
                                             double tol_bin, double tol, uint32_t sentinel) {
  const double bd = to_f64(bt), xd = to_f64(xt);
  // core.py:129-136: finite(r) already implies finite(b) and finite(x)
  double r = __ddiv_rn(__dsub_rn(xd, bd), bd);
  bool valid = finite64(r);
  if (!valid) {
    valid = (bd == 0.0 && xd == 0.0);
    r = 0.0;
  }
  const uint32_t idx = find(r);
  const double c = __ldg(centers + idx);
  const bool near = valid && (fabs(__dsub_rn(r, c)) <= tol_bin);
  const bool rt = roundtrip_ok<T>(c, bd, xd, tol);   // branch-free
  return (near && rt) ? idx : sentinel;
}

// The exact classification with a binary search over the cuts in global
// memory: the fallback of the direct-grid mode (out of line, rarely taken).
template <typename T>
__device__ __noinline__ uint32_t classify_exact(T bt, T xt, const double* __restrict__ cuts_g, int ncuts,
                                                const double* __restrict__ centers_g, double tol_bin, double tol,
                                                uint32_t sentinel) {
  return classify<T>(bt, xt,
                     [&](double r) -> uint32_t {
                       int a = 0, z = ncuts;
                       while (a < z) {
                         int mid = (a + z) >> 1;
                         if (__ldg(cuts_g + mid) < r) a = mid + 1; else z = mid;
                       }
                       return (uint32_t)a;
                     },
                     centers_g, tol_bin, tol, sentinel);
}

// ---- direct-grid mode ---------------------------------------------------------
// The selected centers sit in the middles of histogram bins of width
// w = 2*tol_bin.  Lay a grid of cells of width w with origin c_0 - w/2;
// center i lies within D cells of the middle of cell q_i (D measured at set-up,
// covering quantisation to T and rounding).  For an element whose position
// u = (r - c_0)/w + 1/2 is inside cell q with margin m > D + (cut rounding):
//   * q = q_j selected:  both neighbouring cuts lie outside the cell, so
//     searchsorted(cuts, r) = j, and |r - c_j| < w/2 = tol_bin  -> code j if
//     the round-trip filter passes;
//   * q not selected:    every center is > w/2 away -> sentinel.
// u is estimated from the division-free ratio (|ra - r| <= |ra| 2^-49) as
// t' = (ra - c_0)/w ~ u - 1/2, whose nearest integer (magic-number rounding)
// is the cell; the margin m bounds the error over the table's range, and
// cells beyond it are sentinels while the error stays below half a cell
// (|t'| < 2^30, |c_0|/w < 2^40).
// Anything closer to a cell edge takes the exact path (classify_exact), so
// the codes are the exact path's codes bit for bit.
struct DirectGrid {
  double c0, iw, hm;       // first center, 1/w, 1/2 - margin
  uint32_t tab_s, opc_s;   // shared addresses: cell+1 -> center, center -> RN(1 + c)
  uint32_t span2;          // table entries: cells -1 .. span
  bool far_ok;             // |t'| < 2^30 outside the table is decisive
};

__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
// opaque copies: keep launch constants in registers instead of letting the
// compiler re-derive them (e.g. shared addresses from the CTA id) per element
__device__ __forceinline__ double opaque(double v) {
  double r;
  asm volatile("mov.b64 %0, %1;" : "=d"(r) : "d"(v));
  return r;
}
__device__ __forceinline__ uint32_t opaque(uint32_t v) {
  uint32_t r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}

// Division-free ratio for the direct grid.  The reciprocal seed is trusted
// only when its first residual |1 - b*y0| < 2^-16 (which also rejects b = 0,
// subnormal, huge, inf and NaN b); two Newton steps then give y within
// 2^-51 of 1/b, so |ra - r| <= |ra| * 2^-49 (+ 2^-1070 if ra is subnormal).
__device__ __forceinline__ double ratio_seeded(double b, double x, bool& ok) {
  const double y0 = rcp_approx(b);
  const double e0 = __fma_rn(-b, y0, 1.0);
  ok = fabs(e0) < 0x1p-16;
  double y = __fma_rn(y0, e0, y0);
  const double e1 = __fma_rn(-b, y, 1.0);
  y = __fma_rn(y, e1, y);
  return __dmul_rn(__dsub_rn(x, b), y);
}

constexpr uint32_t kNoCenter = 0xffffffffu;

// All threads: builds tab[0..span+2) (cell q at q+1, kNoCenter = none) and
// opc[0..k) = RN(1 + c_i); returns true when the mode applies (block-uniform).
__device__ __forceinline__ bool setup_direct(const double* __restrict__ centers_g, int k, double tol_bin,
                                             uint32_t* tab, double* opc, DirectGrid& g, int* s_fail,
                                             unsigned long long* s_dmax, int* s_span) {
  if (threadIdx.x == 0) { *s_fail = 0; *s_dmax = 0ULL; *s_span = 0; }
  __syncthreads();
  const double w = __dmul_rn(2.0, tol_bin);
  const double iw = __ddiv_rn(1.0, w);
  const double c0 = __ldg(centers_g);
  const bool ok0 = k >= 1 && k <= kLutCells - 2 && tol_bin > 0.0 && finite64(w) && finite64(iw) && finite64(c0);
  // cell of center i: p = (c_i - c_0)/w + 1/2, q = floor(p), offset |p - q - 1/2|
  auto cell = [&](double c, double& p) { p = __dadd_rn(__dmul_rn(__dsub_rn(c, c0), iw), 0.5); return floor(p); };
  if (ok0) {
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
      const double c = __ldg(centers_g + i);
      opc[i] = __dadd_rn(1.0, c);   // the decoder's (1 + c) (core.py:202-205)
      double p, pp;
      const double q = cell(c, p);
      const double d = fabs(__dsub_rn(p, __dadd_rn(q, 0.5)));
      bool ok = p >= 0.0 && p < (double)(kLutCells - 2) && d <= 0.25;
      if (ok && i > 0) ok = cell(__ldg(centers_g + i - 1), pp) < q;
      if (!ok) *s_fail = 1;
      else atomicMax(s_dmax, (unsigned long long)__double_as_longlong(d));   // d >= 0: bits are ordered
      if (ok && i == k - 1) *s_span = (int)q + 1;
    }
  }
  __syncthreads();
  if (!ok0 || *s_fail) return false;
  const int span = *s_span;
  for (int i = threadIdx.x; i < span + 2; i += blockDim.x) tab[i] = kNoCenter;
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    double p;
    tab[(int)cell(__ldg(centers_g + i), p) + 1] = (uint32_t)i;
  }
  // margin (cells): ratio error over the table's range (|ra| <= A, relative
  // 2^-49 taken as 2^-44, plus the subnormal floor), rounding of t' and of
  // the cell computation, of the cuts, the measured center offsets D
  const double A = fabs(c0) + (span + 2.0) * w;
  const double D = __longlong_as_double((long long)*s_dmax);
  const double m = (A * iw * 0x1p-44 + A * iw * 0x1p-50 + (span + 2.0) * 0x1p-48 + iw * 0x1p-1000) * 1.01 + D +
                   0x1p-40;
  g.hm = opaque(0.5 - m);
  g.c0 = c0;
  g.iw = iw;
  g.span2 = (uint32_t)span + 2;
  g.far_ok = fabs(c0) * iw < 0x1p+40;
  g.tab_s = opaque(smem_u32(tab));
  g.opc_s = opaque(smem_u32(opc));
  __syncthreads();
  return m < 0.02;
}

template <typename T>
__device__ __forceinline__ uint32_t classify_direct(T bt, T xt, const DirectGrid& g, double tol, uint32_t sentinel,
                                                    const double* __restrict__ cuts_g, int ncuts,
                                                    const double* __restrict__ centers_g, double tol_bin) {
  constexpr double kMagic = 6755399441055744.0;   // 1.5 * 2^52: adds round to an integer
  const double bd = to_f64(bt), xd = to_f64(xt);
  bool ok;
  const double ra = ratio_seeded(bd, xd, ok);
  const double t = __dmul_rn(__dsub_rn(ra, g.c0), g.iw);   // ~ u - 1/2
  const double mm = __dadd_rn(t, kMagic);
  const double dd = __dsub_rn(t, __dsub_rn(mm, kMagic));   // t - RN_int(t), exact
  const uint32_t q1 = (uint32_t)__double2loint(mm) + 1u;   // cell + 1 (low word of the magic sum)
  if (ok && fabs(t) < 0x1p+30) {   // the low word holds the cell exactly
    if (q1 < g.span2) {   // cells -1 .. span: the table decides with the margin
      if (fabs(dd) < g.hm) {
        const uint32_t idx = lds_u32(g.tab_s + 4 * q1);
        if (idx == kNoCenter) return sentinel;
        // round-trip filter (pipeline.py:143-160) with the stored RN(1 + c)
        const double rec = to_f64(narrow<T>(__dmul_rn(lds_f64(g.opc_s + 8 * idx), bd)));
        return fabs(__dsub_rn(rec, xd)) <= __dmul_rn(tol, fabs(bd)) ? idx : sentinel;
      }
    } else if (g.far_ok) {   // two or more cells outside: no center within w/2
      return sentinel;
    }
  }
  return classify_exact<T>(bt, xt, cuts_g, ncuts, centers_g, tol_bin, tol, sentinel);
}

// ---- keyed mode: classification from K1's f32 ratio keys ---------------------
// When K1 stored the keys (DevicePipeline, engine.encode), K4 reads 4 bytes
// per element instead of both snapshots (k_encode_keyed).  The cells are the
// histogram bins (origin gmin, width w = 2E); u = (r - gmin)/w.
//  * f32 test (classify_key / classify_key2, FFMA2/FADD2): th = RN32(key*iw32
//    + c32) estimates u - 1/2 - q_ref, q_ref the bin of r = 0, and
//      |th - (u - 1/2 - q_ref)| <= |th| 2^-23 + |key| iw 2^-22 + C0
//    per element (setup_keyed), so |d| + that bound < 1/2 - margin, with
//    d = th - RN_int(th), places u inside bin floor(u) farther than the
//    margin from its edges.  Small ratios (the bulk) get a tiny bound.
//  * f64 test (classify_key64) for the few keys the f32 test leaves open;
//    then the exact path from (b, x) for +inf keys and the rest.
// Each selected center lies within D of its bin's middle (measured at
// set-up); the margin adds D, the cut rounding and the round-trip term, so:
//   * bin selected (center j):  |r - c_j| < E - delta, both cuts around c_j
//     lie farther than that, so searchsorted gives j, the near test passes,
//     and the round-trip filter passes: with b in the safe range (K1 stores a
//     finite key only then, or for b = x = 0) the decoder's value satisfies
//     |T((1+c)b) - x| <= |b| (|c - r| + delta) with
//       delta = 4(1 + A) 2^-52 + 2E 2^-52 [+ (1 + A + E) 2^-23 + 2^-48 for f32],
//     A >= |c|, |r| (IEEE error of the sub, div, add, mul, narrowing and of
//     RN(E|b|); subnormal results absorbed by |b| >= 2^-900 / 2^-100);
//   * bin not selected: every center is more than w/2 away -> sentinel.
// NaN keys are invalid elements (sentinel).  So the codes are the exact
// path's codes bit for bit.  Incompressible positions go out as a 256-bit
// mask per chunk; k_enc_finalize gathers their values from `cur`.
constexpr uint32_t kKeySlow = 0x80000000u;   // not a code: decide again (f64 key test, exact path)
constexpr uint32_t kIncFlag = 0x40000000u;   // tags the sentinel in the keyed table (codes < 2^30)

// The keyed table holds u16 entries for B <= 15 (codes < 2^15), so twice
// as many ordinals fit in the same 32 KB; the sentinel's tag is then bit 15.
#ifndef NMK_T16_MAXB
#define NMK_T16_MAXB 15
#endif
template <bool T16>
constexpr int kTabCells = T16 ? 2 * kLutCells : kLutCells;
template <bool T16>
constexpr int kIncBit = T16 ? 15 : 30;
template <bool T16>
__device__ __forceinline__ uint32_t tab_code(uint32_t tab_s, uint32_t row) {
  if constexpr (T16) {
    uint32_t t;
    asm volatile("ld.shared.u16 %0, [%1];" : "=r"(t) : "r"(tab_s + 2 * row));
    return t;
  } else {
    return lds_u32(tab_s + 4 * row);
  }
}

struct KeyedGrid {
  unsigned long long iw2, c2;   // (iw32, iw32) and (c32, c32) as f32x2
  float iw32, c32, hi4;
  float ka;         // RU32(iw 2^-22): the key-error term of the per-element bound
  uint32_t q0m1;    // ordinal of the first center - 1 (table row 0)
  uint32_t rowbase; // magic-sum bits -> table row
  uint32_t span2;   // table rows: ordinals q0-1 .. q_last+1
  uint32_t tab_s, opc_s;
  uint32_t kd_s;    // shared double[3]: gmin, 1/w, 1/2 - margin (f64 key test)
};

// All threads: tab[row] = code of ordinal q0 - 1 + row (center index, or the
// sentinel tagged with kIncFlag), opc[i] = RN(1 + c_i); true when the mode
// applies (block-uniform).
template <typename T, bool T16>
__device__ __forceinline__ bool setup_keyed(const double* __restrict__ centers_g, int k,
                                            const nmk_stats* __restrict__ st, double width, double tol,
                                            double tol_bin, uint32_t sentinel, uint32_t* tab, double* opc,
                                            KeyedGrid& g, int* s_fail, unsigned long long* s_dmax, int* s_q,
                                            double* s_kd) {
  if (threadIdx.x == 0) { *s_fail = 0; *s_dmax = 0ULL; s_q[0] = 0; s_q[1] = 0; }
  __syncthreads();
  const double gmin = st->gmin, gmax = st->gmax;
  const unsigned long long nb = st->reserved;
  const double inv_w = __ddiv_rn(1.0, width);
  const bool ok0 = k >= 1 && nb >= 1 && nb < (1ULL << 21) && tol > 0.0 && tol < 0x1p+20 && tol_bin == tol &&
                   width == __dmul_rn(2.0, tol) && finite64(gmin) && finite64(gmax) && finite64(inv_w);
  auto pos = [&](double c) { return __dmul_rn(__dsub_rn(c, gmin), inv_w); };   // (c - gmin)/w
  if (ok0) {
    for (int i = threadIdx.x; i < k; i += blockDim.x) {
      const double c = __ldg(centers_g + i);
      opc[i] = __dadd_rn(1.0, c);   // the decoder's (1 + c) (core.py:202-205)
      const double p = pos(c);
      const double q = floor(p);
      const double d = fabs(__dsub_rn(p, __dadd_rn(q, 0.5)));
      bool ok = p >= 0.0 && p < (double)nb && d <= 0.25;   // false for NaN
      if (ok && i > 0) ok = floor(pos(__ldg(centers_g + i - 1))) < q;
      if (!ok) *s_fail = 1;
      else atomicMax(s_dmax, (unsigned long long)__double_as_longlong(d));
      if (ok && i == 0) s_q[0] = (int)q;
      if (ok && i == k - 1) s_q[1] = (int)q;
    }
  }
  __syncthreads();
  if (!ok0 || *s_fail) return false;
  const int q0 = s_q[0], span2 = s_q[1] - q0 + 3;
  if (span2 > kTabCells<T16>) return false;
  uint16_t* tab16 = reinterpret_cast<uint16_t*>(tab);
  for (int i = threadIdx.x; i < span2; i += blockDim.x) {
    if constexpr (T16) tab16[i] = (uint16_t)(sentinel | (1u << kIncBit<true>));
    else tab[i] = sentinel | kIncFlag;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) {
    const int row = (int)floor(pos(__ldg(centers_g + i))) - q0 + 1;
    if constexpr (T16) tab16[row] = (uint16_t)i;
    else tab[row] = (uint32_t)i;
  }
  const double A = fmax(fmax(fabs(gmin), fabs(gmax)), fmax(fabs(__ldg(centers_g)), fabs(__ldg(centers_g + k - 1))));
  const double D = __longlong_as_double((long long)*s_dmax);
  constexpr bool kF32 = sizeof(T) == 4;
  const double delta = (4.0 * (1.0 + A) + 2.0 * tol) * 0x1p-52 + (kF32 ? (1.0 + A + tol) * 0x1p-23 + 0x1p-48 : 0x1p-170);
  // margin terms (cells): the round trip, cut / center-position rounding
  const double mp = D + (delta * inv_w + A * inv_w * 0x1p-50 + (nb + 2.0) * 0x1p-48 + 0x1p-40) * 1.01;
  // f32 test, origin moved to the bin of r = 0 (q_ref) so the constants and
  // the FMA are small where the ratios are:  th = RN32(key*iw32 + c32) with
  // c' = -gmin/w - 1/2 - q_ref (|c'| <= 1/2), and per element
  //   |th - (u - 1/2 - q_ref)| <= |th| 2^-23 + |key| iw 2^-22 + C0
  // (FMA rounding, |key - r| <= |key| 2^-23, |iw32 - 1/w|, RN32 of c').
  const double G = fabs(gmin) * inv_w;
  const double cd = -gmin * inv_w - 0.5;
  const double qref = rint(cd);
  const double cp = cd - qref;   // exact (Sterbenz)
  const double C0 = fabs(cp) * 0x1p-24 + G * 0x1p-50 + 0x1p-40;
  const double hiT = 0.5 - mp - C0 - 0x1p-23;   // 2^-23: the f32 rounding of the bound itself
  const bool on = G < 0x1p+30 && A * inv_w < 0x1p+40 && inv_w < 0x1p+100 && A < 0x1p+100 && hiT > 0.25;
  if (threadIdx.x == 0) {
    s_kd[0] = gmin;
    s_kd[1] = inv_w;
    s_kd[2] = 0.5 - mp;
  }
  g.kd_s = opaque(smem_u32(s_kd));
  g.iw32 = __double2float_rn(inv_w);
  g.c32 = __double2float_rn(cp);
  g.ka = __double2float_ru(inv_w * 0x1p-22);
  g.iw2 = ((unsigned long long)__float_as_uint(g.iw32) << 32) | __float_as_uint(g.iw32);
  g.c2 = ((unsigned long long)__float_as_uint(g.c32) << 32) | __float_as_uint(g.c32);
  g.hi4 = on ? __double2float_rz(hiT) : -1.0f;
  g.q0m1 = (uint32_t)(q0 - 1);
  g.rowbase = 0x4B400000u + (uint32_t)(q0 - 1 - (long long)qref);   // magic-sum bits -> table row
  g.span2 = (uint32_t)span2;
  g.tab_s = opaque(smem_u32(tab));
  g.opc_s = opaque(smem_u32(opc));
  __syncthreads();
  return g.hi4 > 0.0f;
}

// The keyed mode does not apply but no k_encode launch follows (EncodeKeys::
// only, a stale hint): a grid on which every key fails both key tests, so each
// valid element takes the exact path from (b, x) -- bit-exact, only slower.
template <bool T16>
__device__ __forceinline__ void setup_keyed_exact_only(const double* __restrict__ centers_g, int k, uint32_t sentinel,
                                                       uint32_t* tab, double* opc, KeyedGrid& g, double* s_kd) {
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += blockDim.x) opc[i] = __dadd_rn(1.0, __ldg(centers_g + i));
  if (threadIdx.x == 0) {
    if constexpr (T16) reinterpret_cast<uint16_t*>(tab)[0] = (uint16_t)(sentinel | (1u << kIncBit<true>));
    else tab[0] = sentinel | kIncFlag;
    s_kd[0] = 0.0;
    s_kd[1] = 0.0;
    s_kd[2] = -1.0;   // classify_key64 never decides
  }
  g.kd_s = opaque(smem_u32(s_kd));
  g.iw32 = 0.0f;
  g.c32 = 0.0f;
  g.ka = 0.0f;
  g.iw2 = 0ULL;
  g.c2 = 0ULL;
  g.hi4 = -1.0f;      // classify_key / classify_key2 never decide
  g.q0m1 = 0u;
  g.rowbase = 0x4B400000u;
  g.span2 = 1u;
  g.tab_s = opaque(smem_u32(tab));
  g.opc_s = opaque(smem_u32(opc));
  __syncthreads();
}

// Branch-free: rows outside the table are clamped onto its last row (ordinal
// q_last + 1, never a center: the tagged sentinel); a key outside the
// margin, NaN included, gives kKeySlow.
template <bool T16>
__device__ __forceinline__ uint32_t classify_key(float key, const KeyedGrid& g) {
  constexpr float kMagic = 12582912.0f;   // 1.5 * 2^23
  const float th = __fmaf_rn(key, g.iw32, g.c32);
  const float m = __fadd_rn(th, kMagic);
  const float d = __fsub_rn(th, __fsub_rn(m, kMagic));
  const uint32_t row = min((uint32_t)__float_as_int(m) - g.rowbase, g.span2 - 1u);
  const uint32_t code = tab_code<T16>(g.tab_s, row);
  const float sb = __fmaf_rn(fabsf(th), 0x1p-23f, __fmaf_rn(fabsf(key), g.ka, fabsf(d)));   // |d| + bound
  return sb < g.hi4 ? code : kKeySlow;
}

// classify_key for two keys at once: the f32 arithmetic in f32x2 form
// (FFMA2 / FADD2, each lane IEEE round-to-nearest like the scalar ops), the
// bound test per key.  Keys outside the margin (NaN included) give kKeySlow,
// which the caller re-decides.
template <bool T16>
__device__ __forceinline__ void classify_key2(float ka, float kb, const KeyedGrid& g, uint32_t& ca, uint32_t& cb) {
  constexpr unsigned long long kMagic2 = 0x4B4000004B400000ULL;   // (1.5 * 2^23, 1.5 * 2^23)
  const unsigned long long k2 = ((unsigned long long)__float_as_uint(kb) << 32) | __float_as_uint(ka);
  unsigned long long th, m, t, d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(th) : "l"(k2), "l"(g.iw2), "l"(g.c2));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(m) : "l"(th), "l"(kMagic2));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(m), "l"(kMagic2));
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(th), "l"(t));
  const uint32_t ra = min((uint32_t)m - g.rowbase, g.span2 - 1u);
  const uint32_t rb = min((uint32_t)(m >> 32) - g.rowbase, g.span2 - 1u);
  const uint32_t ta = tab_code<T16>(g.tab_s, ra);
  const uint32_t tb = tab_code<T16>(g.tab_s, rb);
  const float sa = __fmaf_rn(fabsf(__uint_as_float((uint32_t)th)), 0x1p-23f,
                             __fmaf_rn(fabsf(ka), g.ka, fabsf(__uint_as_float((uint32_t)d))));
  const float sb = __fmaf_rn(fabsf(__uint_as_float((uint32_t)(th >> 32))), 0x1p-23f,
                             __fmaf_rn(fabsf(kb), g.ka, fabsf(__uint_as_float((uint32_t)(d >> 32)))));
  ca = sa < g.hi4 ? ta : kKeySlow;
  cb = sb < g.hi4 ? tb : kKeySlow;
}

// Second tier for keys the f32 test left undecided (near a bin edge by the
// launch-wide bound, which is loose for the small ratios of a dominant bin):
// t = RN(RN(key - gmin) / w) in f64 with the per-element bound
//   |t - u| <= et = |key| iw 2^-22 + |t| 2^-49 + 2^-60
// (|key - r| <= |key| 2^-23, three roundings of t), so with f = t - floor(t),
// |f - 1/2| < 1/2 - margin - et puts u in bin floor(t) with the margin of
// setup_keyed.  +inf keys (exact path) give NaN and fail.
template <bool T16>
__device__ __forceinline__ uint32_t classify_key64(float key, const KeyedGrid& g) {
  const double gmin = lds_f64(g.kd_s), iw = lds_f64(g.kd_s + 8), half_m = lds_f64(g.kd_s + 16);
  const double t = __dmul_rn(__dsub_rn((double)key, gmin), iw);
  const double fl = floor(t);
  const double f = __dsub_rn(t, fl);
  const double et = fabs((double)key) * iw * 0x1p-22 + fabs(t) * 0x1p-49 + 0x1p-60;
  if (!(fabs(__dsub_rn(f, 0.5)) < __dsub_rn(half_m, et)) || !(t < 0x1p+31)) return kKeySlow;
  const uint32_t row = min((uint32_t)(long long)fl - g.q0m1, g.span2 - 1u);
  return tab_code<T16>(g.tab_s, row);
}

// Packed bytes of one chunk: each lane's 8 codes are B bytes at lane * B;
// whole chunks store them directly, a chunk clipped by its block's end
// stages them per warp and stores the block's bytes only.
template <int B>
__device__ __forceinline__ void chunk_pack(const EncodeGeom& geo, uint32_t b, uint32_t ci, uint64_t blk_start,
                                           uint64_t blk_end, const uint32_t (&code)[kGroup], uint8_t* my,
                                           uint8_t* __restrict__ packed) {
  const int lane = threadIdx.x & 31;
  const uint64_t blk_bytes = ((blk_end - blk_start) * B + 7) / 8;
  const uint64_t off = (uint64_t)ci * (32 * B);
  uint8_t* dst = packed + (uint64_t)(b - geo.b0) * geo.stride + off;
  if (blk_bytes >= off + 32 * B) {
    pack8<B>(code, dst + lane * B);
    return;
  }
  const uint32_t nbytes = (uint32_t)(blk_bytes > off ? blk_bytes - off : 0);
  pack8<B>(code, my + lane * B);
  __syncwarp();
  const uint32_t nvec = nbytes / 16;
  for (uint32_t i = lane; i < nvec; i += 32)
    reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(my)[i];
  for (uint32_t i = nvec * 16 + lane; i < nbytes; i += 32) dst[i] = my[i];
  __syncwarp();
}

// Chunk epilogue of the snapshot-reading flavours: warp-level compaction of
// the incompressible values (already in registers) into the chunk's scratch
// window (element order; most chunks have none), the chunk count, and the
// packed bytes.
template <typename T, int B, typename XOf>
__device__ __forceinline__ void chunk_finish(const EncodeGeom& geo, uint32_t c, uint32_t b, uint32_t ci,
                                             uint64_t blk_start, uint64_t blk_end, const uint32_t (&code)[kGroup],
                                             unsigned inc_mask, XOf&& x_of, T* __restrict__ scratch,
                                             uint32_t* __restrict__ counts, uint8_t* my, uint8_t* __restrict__ packed) {
  const int lane = threadIdx.x & 31;
  unsigned total = 0;
  if (__any_sync(0xffffffffu, inc_mask != 0)) {
    const unsigned cnt = __popc(inc_mask);
    unsigned incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    total = __shfl_sync(0xffffffffu, incl, 31);
    T* w = scratch + (uint64_t)c * kChunk + (incl - cnt);
#pragma unroll
    for (int e = 0; e < kGroup; ++e)
      if (inc_mask >> e & 1u) *w++ = x_of(e);   // raw bits (NaN payloads kept)
  }
  if (lane == 0) counts[c] = total;
  chunk_pack<B>(geo, b, ci, blk_start, blk_end, code, my, packed);
}

// The chunk loop, instantiated once per classification flavour.
template <typename T, int B, bool kRecon, typename Cls, typename Rec>
__device__ __forceinline__ void encode_chunks(const T* __restrict__ base, const T* __restrict__ cur,
                                              const EncodeGeom& geo, uint8_t* __restrict__ packed,
                                              T* __restrict__ scratch, uint32_t* __restrict__ counts,
                                              uint8_t* my, T* __restrict__ recon, Cls&& cls, Rec&& rec_of) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t sentinel = (1u << B) - 1u;
  const uint64_t local_end = geo.elem0 + geo.n_local;
  const bool ptr_al = (((uintptr_t)base | (uintptr_t)cur | (kRecon ? (uintptr_t)recon : 0)) & 15) == 0;
  // chunk ids fit 32 bits (n < 2^40): cheap block / in-block split
  const uint32_t cpb = (uint32_t)geo.cpb;
  const uint32_t nw = gridDim.x * (kEncThreads / 32);
  for (uint32_t c = blockIdx.x * (kEncThreads / 32) + wid; c < (uint32_t)geo.nchunks; c += nw) {
    const uint32_t g = (uint32_t)geo.g0 + c;
    const uint32_t b = geo.fd_cpb.div(g), ci = g - b * cpb;
    const uint64_t blk_start = (uint64_t)b * geo.epb;
    const uint64_t blk_end = min(blk_start + geo.epb, geo.n_total);
    const uint64_t chunk_lo = blk_start + (uint64_t)ci * kChunk;
    const uint64_t lo = max(chunk_lo, geo.elem0), hi = min(blk_end, local_end);
    const uint64_t grp_lo = chunk_lo + (uint64_t)lane * kGroup;
    const bool full = chunk_lo >= geo.elem0 && chunk_lo + kChunk <= hi;  // warp-uniform
    T bv[kGroup], xv[kGroup];
    uint32_t code[kGroup];
    unsigned inc_mask = 0;
    const int64_t li = (int64_t)grp_lo - (int64_t)geo.elem0;
    constexpr int VN = EVec<T>::N;
    if (full && ptr_al && (li % VN) == 0) {
      load8<T>(base + li, bv);
      load8<T>(cur + li, xv);
#pragma unroll
      for (int e = 0; e < kGroup; ++e) {
        code[e] = cls(bv[e], xv[e]);
        inc_mask |= (code[e] == sentinel ? 1u : 0u) << e;
      }
      if constexpr (kRecon) {   // the decoder's values, written by the encoder
        using V = typename EVec<T>::V;
#pragma unroll
        for (int q = 0; q < kGroup / VN; ++q) {
          V w;
          T* t = reinterpret_cast<T*>(&w);
#pragma unroll
          for (int e = 0; e < VN; ++e) {
            const int ee = q * VN + e;
            t[e] = code[ee] == sentinel ? xv[ee] : rec_of(code[ee], bv[ee]);
          }
          reinterpret_cast<V*>(recon + li)[q] = w;
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < kGroup; ++e) {
        const uint64_t j = grp_lo + e;
        const bool in = j >= lo && j < hi;
        bv[e] = in ? __ldg(base + (li + e)) : T(0);
        xv[e] = in ? __ldg(cur + (li + e)) : T(0);
        code[e] = in ? cls(bv[e], xv[e]) : 0u;
        inc_mask |= (in && code[e] == sentinel ? 1u : 0u) << e;
        if constexpr (kRecon)
          if (in) recon[li + e] = code[e] == sentinel ? xv[e] : rec_of(code[e], bv[e]);
      }
    }
    chunk_finish<T, B>(geo, c, b, ci, blk_start, blk_end, code, inc_mask, [&](int e) { return xv[e]; }, scratch,
                       counts, my, packed);
  }
}

// The keyed chunk loop: codes from the keys; the snapshots are read only
// where a key cannot decide (slow), for the incompressible values, and for
// the fused reconstruction's base values.  Each warp keeps the keys of
// kKeyStagesE chunks in flight (TMA ring in shared memory).
#ifndef NMK_ENCK_STAGES
#define NMK_ENCK_STAGES 2   // stages of two chunks' keys (2 KB) per warp
#endif
constexpr int kKeyStagesE = NMK_ENCK_STAGES;
// a stage holds a chunk pair's keys plus 4 of slack: a pair whose first key
// is not 16-byte aligned (blocks of epb % 4 != 0 elements, e.g. B = 12) is
// copied from the aligned address below it
constexpr int kStageKeys = 2 * kChunk + 4;
// dynamic shared memory of k_encode_keyed: opc doubles, then 128-byte aligned key tiles
__host__ __device__ constexpr size_t keyed_ring_off(int k_cap) { return ((size_t)(k_cap + 2) + 15) & ~(size_t)15; }
__host__ __device__ constexpr size_t keyed_smem_bytes(int k_cap) {
  return keyed_ring_off(k_cap) * 8 + (size_t)(kEncThreads / 32) * kKeyStagesE * kStageKeys * 4;
}
// Lane keys 8 l + shift .. + 7 from a 16-byte aligned shared-memory row p
// (p = row + 8 l): three aligned vectors, then a warp-uniform shift.
__device__ __forceinline__ void shifted_keys(const float* p, uint32_t shift, float4& a, float4& b) {
  const float4 v0 = reinterpret_cast<const float4*>(p)[0], v1 = reinterpret_cast<const float4*>(p)[1],
               v2 = reinterpret_cast<const float4*>(p)[2];
  if (shift == 1) {
    a = make_float4(v0.y, v0.z, v0.w, v1.x);
    b = make_float4(v1.y, v1.z, v1.w, v2.x);
  } else if (shift == 2) {
    a = make_float4(v0.z, v0.w, v1.x, v1.y);
    b = make_float4(v1.z, v1.w, v2.x, v2.y);
  } else {
    a = make_float4(v0.w, v1.x, v1.y, v1.z);
    b = make_float4(v1.w, v2.x, v2.y, v2.z);
  }
}

template <typename T, int B, bool kRecon, bool kAligned, typename Slow, typename Rec>
__device__ __forceinline__ void encode_chunks_keyed(const float* __restrict__ keys, const T* __restrict__ base,
                                                    const T* __restrict__ cur, const EncodeGeom& geo,
                                                    uint8_t* __restrict__ packed, uint8_t* __restrict__ masks,
                                                    uint32_t* __restrict__ counts, uint8_t* my,
                                                    T* __restrict__ recon, const KeyedGrid& kg, float* kring,
                                                    unsigned long long* kbars, Slow&& slow, Rec&& rec_of) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t sentinel = (1u << B) - 1u;
  constexpr bool kT16 = B <= NMK_T16_MAXB;
  constexpr uint32_t kInc = 1u << kIncBit<kT16>;   // tags the sentinel in table codes
  const uint64_t local_end = geo.elem0 + geo.n_local;
  // keys are 16-byte aligned (nmk_encode_keyed_dev checks); vector access
  // to base / recon needs them aligned too
  const bool ptr_al = (((uintptr_t)base | (uintptr_t)recon) & 15) == 0;
  const uint32_t cpb = (uint32_t)geo.cpb;
  const uint32_t cpb_whole = (uint32_t)(geo.epb / kChunk);   // chunks per block that are never clipped
  constexpr int VN = EVec<T>::N;
  // this warp's contiguous run of chunks [cA, cB)
  const uint32_t nch = (uint32_t)geo.nchunks;
  const uint32_t nwarps = gridDim.x * (kEncThreads / 32);
  const uint32_t wg = blockIdx.x * (kEncThreads / 32) + wid;
  const uint32_t per = nch / nwarps, rem = nch % nwarps;
  const uint32_t cA = wg * per + min(wg, rem);
  const uint32_t cB = cA + per + (wg < rem ? 1u : 0u);
  const uint32_t cBf = min(cB, geo.c_last + 1u);   // whole chunks of this range end here
  // chunk cursor, advanced incrementally (no division in the loop).  `left`
  // counts the pairs still ahead in the current run of whole chunks (same
  // block, keys aligned), so the common step is a few adds.
  struct Cur {
    uint32_t c, b, ci, left;
    uint64_t lo;   // first element of the chunk
  };
  auto at = [&](uint32_t c) {
    Cur k;
    const uint32_t g = (uint32_t)geo.g0 + c;
    k.c = c;
    k.b = geo.fd_cpb.div(g);
    k.ci = g - k.b * cpb;
    k.lo = (uint64_t)k.b * geo.epb + (uint64_t)k.ci * kChunk;
    k.left = 0;
    return k;
  };
  auto next = [&](Cur& k) {   // one chunk
    ++k.c;
    if (++k.ci == cpb) {
      k.ci = 0;
      ++k.b;
      k.lo = (uint64_t)k.b * geo.epb;
    } else {
      k.lo += kChunk;
    }
  };
  auto next_pair = [&](Cur& k) {   // ci + 2 <= cpb_whole <= cpb
    k.c += 2;
    --k.left;
    k.ci += 2;
    k.lo += 2 * kChunk;
    if (k.ci == cpb) {
      k.ci = 0;
      ++k.b;
      k.lo = (uint64_t)k.b * geo.epb;
    }
  };
  // warp-uniform: a whole chunk of this range, inside its block
  auto fast_of = [&](const Cur& k) { return k.c >= geo.c_first && k.c <= geo.c_last && k.ci < cpb_whole; };
  // warp-uniform: the current item is a pair of whole chunks (starts a run
  // when needed).  A misaligned run's copies read up to 4 - shift keys past
  // the pair, so its last pair must leave them inside this range.
  auto pair_of = [&](Cur& k) {
    if (k.left == 0 && k.c + 1 < cBf && k.ci + 1 < cpb_whole && fast_of(k)) {
      uint32_t avail = min(cBf - k.c, cpb_whole - k.ci) & ~1u;
      const uint32_t sh = kAligned ? 0u : (uint32_t)(k.lo - geo.elem0) & 3u;
      if (sh && k.lo + (uint64_t)avail * kChunk + 4 - sh > local_end) avail -= 2;
      k.left = avail >> 1;
    }
    return k.left != 0;
  };
  // the rare keys: NaN (invalid -> sentinel), the f64 key test, the exact path
  auto redo = [&](uint32_t& code, int64_t j, float key) {   // key = keys[j] (already in registers)
    uint32_t v = key != key ? (sentinel | kInc) : classify_key64<kT16>(key, kg);
    if (v == kKeySlow) {
      v = slow(__ldg(base + j), __ldg(cur + j));
      v |= v == sentinel ? kInc : 0u;
    }
    code = v;
  };
  auto recon8 = [&](int64_t li, const uint32_t (&code)[kGroup]) {   // the decoder's values
    if (!ptr_al || (li & (VN - 1)) != 0) {
#pragma unroll
      for (int e = 0; e < kGroup; ++e)
        recon[li + e] = code[e] == sentinel ? __ldg(cur + li + e) : rec_of(code[e], __ldg(base + li + e));
      return;
    }
    T bv[kGroup];
    load8<T>(base + li, bv);
    using V = typename EVec<T>::V;
#pragma unroll
    for (int q = 0; q < kGroup / VN; ++q) {
      V w;
      T* t = reinterpret_cast<T*>(&w);
#pragma unroll
      for (int e = 0; e < VN; ++e) {
        const int ee = q * VN + e;
        t[e] = code[ee] == sentinel ? __ldg(cur + li + ee) : rec_of(code[ee], bv[ee]);
      }
      reinterpret_cast<V*>(recon + li)[q] = w;
    }
  };
  // a pair of whole chunks (16 keys per lane): one warp reduction decides
  // whether anything but table codes occurred
  auto run_pair = [&](const Cur& k, const float4& a0, const float4& a1, const float4& b0, const float4& b1) {
    uint32_t ca[kGroup], cb[kGroup];
    classify_key2<kT16>(a0.x, a0.y, kg, ca[0], ca[1]);
    classify_key2<kT16>(a0.z, a0.w, kg, ca[2], ca[3]);
    classify_key2<kT16>(a1.x, a1.y, kg, ca[4], ca[5]);
    classify_key2<kT16>(a1.z, a1.w, kg, ca[6], ca[7]);
    classify_key2<kT16>(b0.x, b0.y, kg, cb[0], cb[1]);
    classify_key2<kT16>(b0.z, b0.w, kg, cb[2], cb[3]);
    classify_key2<kT16>(b1.x, b1.y, kg, cb[4], cb[5]);
    classify_key2<kT16>(b1.z, b1.w, kg, cb[6], cb[7]);
    const int64_t li = (int64_t)(k.lo - geo.elem0) + lane * kGroup;   // chunk B: li + kChunk
    uint32_t any = 0;
#pragma unroll
    for (int e = 0; e < kGroup; ++e) any |= ca[e] | cb[e];
    const uint32_t flags = __reduce_or_sync(0xffffffffu, any & (kKeySlow | kInc));
    uint32_t tot = 0;
    if (flags) {
      if (flags & kKeySlow) {
        if (any & kKeySlow) {
          const float kva[kGroup] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
          const float kvb[kGroup] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
          for (int e = 0; e < kGroup; ++e) {
            if (ca[e] & kKeySlow) redo(ca[e], li + e, kva[e]);
            if (cb[e] & kKeySlow) redo(cb[e], li + kChunk + e, kvb[e]);
          }
        }
      }
      unsigned ma = 0, mb = 0;
#pragma unroll
      for (int e = 0; e < kGroup; ++e) {
        ma |= ((ca[e] >> kIncBit<kT16>) & 1u) << e;
        mb |= ((cb[e] >> kIncBit<kT16>) & 1u) << e;
        ca[e] &= ~kInc;
        cb[e] &= ~kInc;
      }
      // both chunks' counts in one reduction (each <= 256)
      tot = __reduce_add_sync(0xffffffffu, (unsigned)__popc(ma) | ((unsigned)__popc(mb) << 16));
      masks[(uint64_t)k.c * 32 + lane] = (uint8_t)ma;
      masks[(uint64_t)k.c * 32 + 32 + lane] = (uint8_t)mb;
    }
    if (lane < 2) counts[k.c + lane] = lane ? tot >> 16 : tot & 0xffffu;
    if constexpr (kRecon) {
      recon8(li, ca);
      recon8(li + kChunk, cb);
    }
    uint8_t* dst = packed + (uint64_t)(k.b - geo.b0) * geo.stride + (uint64_t)k.ci * (32 * B) + lane * B;
    pack8<B>(ca, dst);
    pack8<B>(cb, dst + 32 * B);
  };
  // a single chunk: whole (keys given) or clipped by its block / this range
  auto run = [&](const Cur& k, bool fast, const float4& k0, const float4& k1) {
    uint32_t code[kGroup];
    unsigned live = 0xffu;
    const uint64_t grp_lo = k.lo + (uint64_t)lane * kGroup;
    const int64_t li = (int64_t)grp_lo - (int64_t)geo.elem0;
    uint64_t blk_start = 0, blk_end = 0;
    if (fast) {
      classify_key2<kT16>(k0.x, k0.y, kg, code[0], code[1]);
      classify_key2<kT16>(k0.z, k0.w, kg, code[2], code[3]);
      classify_key2<kT16>(k1.x, k1.y, kg, code[4], code[5]);
      classify_key2<kT16>(k1.z, k1.w, kg, code[6], code[7]);
    } else {
      blk_start = (uint64_t)k.b * geo.epb;
      blk_end = min(blk_start + geo.epb, geo.n_total);
      const uint64_t lo = max(k.lo, geo.elem0), hi = min(blk_end, local_end);
      live = 0u;
#pragma unroll
      for (int e = 0; e < kGroup; ++e) {
        const uint64_t j = grp_lo + e;
        const bool in = j >= lo && j < hi;
        live |= (in ? 1u : 0u) << e;
        code[e] = in ? classify_key<kT16>(keys[li + e], kg) : 0u;
      }
    }
    uint32_t any = 0;
#pragma unroll
    for (int e = 0; e < kGroup; ++e) any |= code[e];
    const uint32_t flags = __reduce_or_sync(0xffffffffu, any & (kKeySlow | kInc));
    unsigned total = 0;
    if (flags) {
      if (any & kKeySlow) {
        const float kv[kGroup] = {k0.x, k0.y, k0.z, k0.w, k1.x, k1.y, k1.z, k1.w};
#pragma unroll
        for (int e = 0; e < kGroup; ++e)
          if (code[e] & kKeySlow) redo(code[e], li + e, fast ? kv[e] : __ldg(keys + li + e));
      }
      // incompressible elements: the chunk's count and its 256-bit position
      // mask (one byte per lane); k_enc_finalize gathers the values from cur
      unsigned inc_mask = 0;
#pragma unroll
      for (int e = 0; e < kGroup; ++e) {
        inc_mask |= ((code[e] >> kIncBit<kT16>) & 1u) << e;
        code[e] &= ~kInc;
      }
      inc_mask &= live;
      total = __reduce_add_sync(0xffffffffu, (unsigned)__popc(inc_mask));
      masks[(uint64_t)k.c * 32 + lane] = (uint8_t)inc_mask;
    }
    if (lane == 0) counts[k.c] = total;
    if constexpr (kRecon) {
      if (fast) {
        recon8(li, code);
      } else {
#pragma unroll
        for (int e = 0; e < kGroup; ++e)
          if (live >> e & 1u)
            recon[li + e] = code[e] == sentinel ? __ldg(cur + li + e) : rec_of(code[e], __ldg(base + li + e));
      }
    }
    if (fast) {   // whole chunk inside its block: each lane stores its B bytes
      pack8<B>(code, packed + (uint64_t)(k.b - geo.b0) * geo.stride + (uint64_t)k.ci * (32 * B) + lane * B);
    } else {
      chunk_pack<B>(geo, k.b, k.ci, blk_start, blk_end, code, my, packed);
    }
  };
  // per-warp ring of kKeyStagesE tiles, each the keys of two consecutive
  // chunks (2 KB), filled by TMA bulk copies.  A pair is staged when both
  // chunks are whole and in the same block; other chunks go one at a time
  // with their keys read directly.
  float* ring = kring + (size_t)wid * kKeyStagesE * kStageKeys;
  unsigned long long* bars = kbars + wid * kKeyStagesE;
  if (lane == 0) {
    for (int st = 0; st < kKeyStagesE; ++st) mbar_init(&bars[st], 1);
    mbar_fence_init();
  }
  __syncwarp();
  if (cA >= cB) return;
  Cur cp = at(cA), pf = cp;
  auto issue = [&](int st) {   // warp-uniform; lane 0 issues the copy of item pf
    if (pf.c >= cB) return;
    if (pair_of(pf)) {
      if (lane == 0) {
        const uint32_t sh = kAligned ? 0u : (uint32_t)(pf.lo - geo.elem0) & 3u;
        const unsigned bytes = sh ? kStageKeys * 4 : 2 * kChunk * 4;
        fence_proxy_async_smem();
        mbar_arrive_tx(&bars[st], bytes);
        tma_load_1d(ring + st * kStageKeys, keys + (pf.lo - geo.elem0 - sh), bytes, &bars[st]);
      }
      next_pair(pf);
    } else {
      next(pf);
    }
  };
#pragma unroll
  for (int st = 0; st < kKeyStagesE; ++st) issue(st);
  uint32_t ph = 0;   // per-stage mbarrier phase bits
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  int st = 0;
  while (cp.c < cB) {
    if (pair_of(cp)) {
      mbar_wait(&bars[st], (ph >> st) & 1u);
      ph ^= 1u << st;
      const uint32_t sh = kAligned ? 0u : (uint32_t)(cp.lo - geo.elem0) & 3u;   // warp-uniform
      float4 a0, a1, b0, b1;
      if (sh == 0) {
        const float4* src = reinterpret_cast<const float4*>(ring + st * kStageKeys) + lane * 2;
        a0 = src[0];
        a1 = src[1];
        b0 = src[64];
        b1 = src[65];
      } else {
        shifted_keys(ring + st * kStageKeys + lane * 8, sh, a0, a1);
        shifted_keys(ring + st * kStageKeys + kChunk + lane * 8, sh, b0, b1);
      }
      __syncwarp();
      issue(st);   // refill the stage just read
      run_pair(cp, a0, a1, b0, b1);
      next_pair(cp);
    } else {
      issue(st);
      const bool fast = fast_of(cp);
      float4 a0 = z4, a1 = z4;
      if (fast) {
        const float* kp = keys + (cp.lo - geo.elem0) + lane * 8;
        if (kAligned || ((cp.lo - geo.elem0) & 3) == 0) {
          a0 = __ldg(reinterpret_cast<const float4*>(kp));
          a1 = __ldg(reinterpret_cast<const float4*>(kp) + 1);
        } else {
          a0 = make_float4(__ldg(kp), __ldg(kp + 1), __ldg(kp + 2), __ldg(kp + 3));
          a1 = make_float4(__ldg(kp + 4), __ldg(kp + 5), __ldg(kp + 6), __ldg(kp + 7));
        }
      }
      run(cp, fast, a0, a1);
      next(cp);
    }
    st = st + 1 == kKeyStagesE ? 0 : st + 1;
  }
}

template <typename T, int B, bool kRecon>
__global__ void __launch_bounds__(kEncThreads, NMK_ENC_MINB)
k_encode(const T* __restrict__ base, const T* __restrict__ cur, EncodeGeom geo,
         const double* __restrict__ centers_g, const double* __restrict__ cuts_g, int k,
         double tol_bin, double tol, uint8_t* __restrict__ packed, T* __restrict__ scratch,
         uint32_t* __restrict__ counts, const nmk_model* __restrict__ model, bool smem_ok, T* __restrict__ recon,
         const uint32_t* __restrict__ done) {
  __shared__ __align__(16) uint8_t wbytes[kEncThreads / 32][32 * B + 16];
  __shared__ uint32_t lut32[kLutCells];   // cell -> center (direct mode) or, as u16, the cut grid
  uint16_t* lut = reinterpret_cast<uint16_t*>(lut32);
  __shared__ double s_lo, s_scale;
  __shared__ bool s_use;
  __shared__ int s_fail, s_span;
  __shared__ unsigned long long s_dmax;
  extern __shared__ __align__(16) double cutsp[];   // [-inf, cuts..., +inf, +inf] or centers

  pdl_enter();
  zero_list_run(geo.zl);
  if (done && *done) return;   // k_encode_keyed already encoded this range
  if (model) {   // sync-free path: the model scalars live on the device
    if (model->status != 0) {   // nothing to encode: leave empty chunks behind
      for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < (uint32_t)geo.nchunks; c += gridDim.x * blockDim.x)
        counts[c] = 0;
      return;
    }
    k = model->k;
    tol_bin = model->tol_bin;
  }
  const int ncuts = k - 1;
  const uint32_t sentinel = (1u << B) - 1u;
  uint8_t* my = wbytes[threadIdx.x >> 5];
  const bool cuts_in_smem = smem_ok && k <= kSmemCuts + 1;
  if (cuts_in_smem) {
    DirectGrid g;
    if (setup_direct(centers_g, k, tol_bin, lut32, cutsp, g, &s_fail, &s_dmax, &s_span)) {
      encode_chunks<T, B, kRecon>(
          base, cur, geo, packed, scratch, counts, my, recon,
          [&](T b, T x) -> uint32_t { return classify_direct<T>(b, x, g, tol, sentinel, cuts_g, ncuts, centers_g, tol_bin); },
          [&](uint32_t cd, T b) -> T { return narrow<T>(__dmul_rn(lds_f64(g.opc_s + 8 * cd), to_f64(b))); });
      return;
    }
    for (int i = threadIdx.x; i < ncuts; i += kEncThreads) cutsp[i + 1] = cuts_g[i];
    if (threadIdx.x == 0) {
      cutsp[0] = __longlong_as_double(0xfff0000000000000LL);
      cutsp[ncuts + 1] = __longlong_as_double(0x7ff0000000000000LL);
      cutsp[ncuts + 2] = cutsp[ncuts + 1];   // read (unused) when i == ncuts
    }
  }
  __syncthreads();
  if (cuts_in_smem) {
    double lo, sc;
    bool use;
    build_cut_lut(cutsp + 1, ncuts, lut, lo, sc, use);
    if (threadIdx.x == 0) { s_lo = lo; s_scale = sc; s_use = use; }
  } else if (threadIdx.x == 0) {
    s_lo = 0.0; s_scale = 0.0; s_use = false;
  }
  __syncthreads();
  if (s_use) {
    // O(1) search: the grid cell gives i = #cuts below the cell's left edge;
    // with at most one cut per cell the answer is i or i+1, settled by exact
    // compares against the three candidate cuts (padded with -inf/+inf).
    // Any other case (rounding at a cell edge, a crowded cell) walks exactly.
    const double lo = s_lo, scale = s_scale;
    auto find = [&](double r) -> uint32_t {
      int g = __double2int_rz((r - lo) * scale);   // saturating
      g = min(max(g, 0), kLutCells - 1);
      int i = lut[g];
      const double a = cutsp[i], m = cutsp[i + 1], z = cutsp[i + 2];
      const bool up = m < r;
      if (up ? (r <= z) : (a < r)) return (uint32_t)(i + up);
      while (i < ncuts && cutsp[i + 1] < r) ++i;
      while (i > 0 && cutsp[i] >= r) --i;
      return (uint32_t)i;
    };
    encode_chunks<T, B, kRecon>(
        base, cur, geo, packed, scratch, counts, my, recon,
        [&](T b, T x) -> uint32_t { return classify<T>(b, x, find, centers_g, tol_bin, tol, sentinel); },
        [&](uint32_t cd, T b) -> T { return apply_center<T>(__ldg(centers_g + cd), to_f64(b)); });
  } else {
    auto find = [&](double r) -> uint32_t {
      int a = 0, z = ncuts;
      while (a < z) {
        int mid = (a + z) >> 1;
        if (__ldg(cuts_g + mid) < r) a = mid + 1; else z = mid;
      }
      return (uint32_t)a;
    };
    encode_chunks<T, B, kRecon>(
        base, cur, geo, packed, scratch, counts, my, recon,
        [&](T b, T x) -> uint32_t { return classify<T>(b, x, find, centers_g, tol_bin, tol, sentinel); },
        [&](uint32_t cd, T b) -> T { return apply_center<T>(__ldg(centers_g + cd), to_f64(b)); });
  }
}

// K4 keyed mode as its own kernel (own register budget).  Every CTA runs the
// same set-up; when the mode does not apply (centers off the bin grid, span
// too wide, bound too loose) it writes done = 0 and returns, and k_encode,
// launched right after, does the work; otherwise done = 1 and k_encode exits.
#ifndef NMK_ENCK_MINB
#define NMK_ENCK_MINB 2
#endif
template <typename T, int B, bool kRecon>
__global__ void __launch_bounds__(kEncThreads, NMK_ENCK_MINB)
k_encode_keyed(const T* __restrict__ base, const T* __restrict__ cur, EncodeGeom geo,
               const double* __restrict__ centers_g, const double* __restrict__ cuts_g, double tol,
               uint8_t* __restrict__ packed, T* __restrict__ scratch, uint32_t* __restrict__ counts,
               const nmk_model* __restrict__ model, int k_cap, T* __restrict__ recon, EncodeKeys kx) {
  __shared__ __align__(16) uint8_t wbytes[kEncThreads / 32][32 * B + 16];
  __shared__ uint32_t tab[kLutCells];   // ordinal row -> code
  __shared__ int s_fail, s_q[2];
  __shared__ unsigned long long s_dmax;
  __shared__ double s_kd[3];
  __shared__ __align__(8) unsigned long long kbars[(kEncThreads / 32) * kKeyStagesE];
  extern __shared__ __align__(128) double opc[];   // RN(1 + c_i) [k_cap + 2], then the key ring
  float* kring = reinterpret_cast<float*>(opc + keyed_ring_off(k_cap));
  const uint32_t sentinel = (1u << B) - 1u;
  pdl_enter();
  zero_list_run(geo.zl);
  if (model->status != 0) {   // nothing to encode: leave empty chunks behind
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < (uint32_t)geo.nchunks; c += gridDim.x * blockDim.x)
      counts[c] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) *kx.done = 1u;
    return;
  }
  const int k = model->k;
  const double tol_bin = model->tol_bin;
  KeyedGrid kg;
  const bool ok = k <= k_cap && k <= kSmemCuts + 1 &&
                  setup_keyed<T, (B <= NMK_T16_MAXB)>(centers_g, k, kx.st, kx.width, tol, tol_bin, sentinel, tab, opc, kg, &s_fail,
                                 &s_dmax, s_q, s_kd);
  const bool exact_only = !ok && kx.only && k <= k_cap;
  if (blockIdx.x == 0 && threadIdx.x == 0) *kx.done = ok ? 1u : (exact_only ? 2u : 0u);
  if (exact_only) setup_keyed_exact_only<(B <= NMK_T16_MAXB)>(centers_g, k, sentinel, tab, opc, kg, s_kd);
  else if (!ok) return;
  const int ncuts = k - 1;
  auto slow = [&](T b, T x) -> uint32_t {
    return classify_exact<T>(b, x, cuts_g, ncuts, centers_g, tol_bin, tol, sentinel);
  };
  auto rec = [&](uint32_t cd, T b) -> T { return narrow<T>(__dmul_rn(lds_f64(kg.opc_s + 8 * cd), to_f64(b))); };
  // every chunk's keys 16-byte aligned (epb % 4 == 0): the shift logic compiles away
  if (geo.key_al)
    encode_chunks_keyed<T, B, kRecon, true>(kx.keys, base, cur, geo, packed, reinterpret_cast<uint8_t*>(scratch),
                                            counts, wbytes[threadIdx.x >> 5], recon, kg, kring, kbars, slow, rec);
  else
    encode_chunks_keyed<T, B, kRecon, false>(kx.keys, base, cur, geo, packed, reinterpret_cast<uint8_t*>(scratch),
                                             counts, wbytes[threadIdx.x >> 5], recon, kg, kring, kbars, slow, rec);
}

static int sm_count_e() { return sm_count(); }

template <typename T, int B, bool kRecon>
static void launch_encode_k(const void* base, const void* cur, const EncodeGeom& geo, const double* centers,
                            const double* cuts, int k, double tol_bin, double tol, uint8_t* packed, void* scratch,
                            uint32_t* counts, const nmk_model* model, int k_cap, void* recon, const EncodeKeys& kx,
                            cudaStream_t s) {
  const bool smem_ok = k_cap <= kSmemCuts + 1;
  const size_t smem = smem_ok ? (size_t)(k_cap + 2) * 8 : 0;
  ensure_dyn_smem(k_encode<T, B, kRecon>, smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_encode<T, B, kRecon>, kEncThreads, smem);
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = (uint64_t)sm_count_e() * per_sm;
  uint64_t need = (geo.nchunks + 7) / 8;
  if (grid > need) grid = need;
  const bool keyed = kx.keys && model && smem_ok;
  if (keyed) {
    const size_t smem_k = keyed_smem_bytes(k_cap);
    ensure_dyn_smem(k_encode_keyed<T, B, kRecon>, smem_k);
    int per_sm_k = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_k, k_encode_keyed<T, B, kRecon>, kEncThreads, smem_k);
    if (per_sm_k < 1) per_sm_k = 1;
    uint64_t grid_k = (uint64_t)sm_count_e() * per_sm_k;
    if (grid_k > need) grid_k = need;
    launch_chain(kPdlK4, k_encode_keyed<T, B, kRecon>, (unsigned)grid_k, kEncThreads, smem_k, s, (const T*)base, (const T*)cur,
                 geo, centers, cuts, tol, packed, (T*)scratch, counts, model, k_cap, (T*)recon, kx);
  }
  if (keyed && kx.only) return;   // hint: the keyed kernel applied last time (it still finishes alone if not)
  launch_chain(kPdlK4Fallback, k_encode<T, B, kRecon>, (unsigned)grid, kEncThreads, smem, s, (const T*)base, (const T*)cur, geo, centers,
               cuts, k, tol_bin, tol, packed, (T*)scratch, counts, model, smem_ok, (T*)recon,
               keyed ? kx.done : nullptr);
}

// the fused reconstruction is a separate instantiation: the plain encode
// keeps its register budget
template <typename T, int B>
void launch_encode(const void* base, const void* cur, const EncodeGeom& geo, const double* centers,
                          const double* cuts, int k, double tol_bin, double tol, uint8_t* packed, void* scratch,
                          uint32_t* counts, const nmk_model* model, int k_cap, void* recon, const EncodeKeys& kx,
                          cudaStream_t s) {
  if (recon)
    launch_encode_k<T, B, true>(base, cur, geo, centers, cuts, k, tol_bin, tol, packed, scratch, counts, model, k_cap,
                                recon, kx, s);
  else
    launch_encode_k<T, B, false>(base, cur, geo, centers, cuts, k, tol_bin, tol, packed, scratch, counts, model,
                                 k_cap, nullptr, kx, s);
}

}  // namespace nmk
