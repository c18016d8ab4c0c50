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

struct EncodeGeom {
  uint64_t n_local, elem0, n_total, epb, cpb, g0, nchunks, b0, stride;
  FastDiv fd_cpb;   // chunk id -> block
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

// The chunk loop, instantiated once per classification flavour.
template <typename T, int B, typename Cls>
__device__ __forceinline__ void encode_chunks(const T* __restrict__ base, const T* __restrict__ cur,
                                              const EncodeGeom& geo, uint8_t* __restrict__ packed,
                                              T* __restrict__ scratch, uint32_t* __restrict__ counts,
                                              uint8_t* my, Cls&& cls) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t sentinel = (1u << B) - 1u;
  const uint64_t local_end = geo.elem0 + geo.n_local;
  const bool ptr_al = (((uintptr_t)base | (uintptr_t)cur) & 15) == 0;
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
    } else {
#pragma unroll
      for (int e = 0; e < kGroup; ++e) {
        const uint64_t j = grp_lo + e;
        const bool in = j >= lo && j < hi;
        bv[e] = in ? __ldg(base + (li + e)) : T(0);
        xv[e] = in ? __ldg(cur + (li + e)) : T(0);
        code[e] = in ? cls(bv[e], xv[e]) : 0u;
        inc_mask |= (in && code[e] == sentinel ? 1u : 0u) << e;
      }
    }
    // warp-level compaction of the incompressible values into the chunk's
    // scratch window (element order); most chunks have none
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
      if (inc_mask) {
        T* w = scratch + (uint64_t)c * kChunk + (incl - cnt);
#pragma unroll
        for (int e = 0; e < kGroup; ++e)
          if (inc_mask >> e & 1u) *w++ = xv[e];   // raw bits (NaN payloads kept)
      }
    }
    if (lane == 0) counts[c] = total;
    // packed bytes: stage per warp, then 16-byte stores clipped to the block
    pack8<B>(code, my + lane * B);
    __syncwarp();
    const uint64_t blk_bytes = ((blk_end - blk_start) * B + 7) / 8;
    const uint64_t off = (uint64_t)ci * (32 * B);
    const uint32_t nbytes = (uint32_t)min(blk_bytes > off ? blk_bytes - off : 0, (uint64_t)(32 * B));
    uint8_t* dst = packed + (uint64_t)(b - geo.b0) * geo.stride + off;
    const uint32_t nvec = nbytes / 16;
    for (uint32_t i = lane; i < nvec; i += 32)
      reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(my)[i];
    for (uint32_t i = nvec * 16 + lane; i < nbytes; i += 32) dst[i] = my[i];
    __syncwarp();
  }
}

template <typename T, int B>
__global__ void __launch_bounds__(kEncThreads, 4)
k_encode(const T* __restrict__ base, const T* __restrict__ cur, EncodeGeom geo,
         const double* __restrict__ centers_g, const double* __restrict__ cuts_g, int k,
         double tol_bin, double tol, uint8_t* __restrict__ packed, T* __restrict__ scratch,
         uint32_t* __restrict__ counts, const nmk_model* __restrict__ model, bool smem_ok) {
  __shared__ __align__(16) uint8_t wbytes[kEncThreads / 32][32 * B + 16];
  __shared__ uint32_t lut32[kLutCells];   // cell -> center (direct mode) or, as u16, the cut grid
  uint16_t* lut = reinterpret_cast<uint16_t*>(lut32);
  __shared__ double s_lo, s_scale;
  __shared__ bool s_use;
  __shared__ int s_fail, s_span;
  __shared__ unsigned long long s_dmax;
  extern __shared__ __align__(16) double cutsp[];   // [-inf, cuts..., +inf, +inf] or centers

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
      encode_chunks<T, B>(base, cur, geo, packed, scratch, counts, my, [&](T b, T x) -> uint32_t {
        return classify_direct<T>(b, x, g, tol, sentinel, cuts_g, ncuts, centers_g, tol_bin);
      });
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
    encode_chunks<T, B>(base, cur, geo, packed, scratch, counts, my, [&](T b, T x) -> uint32_t {
      return classify<T>(b, x, find, centers_g, tol_bin, tol, sentinel);
    });
  } else {
    auto find = [&](double r) -> uint32_t {
      int a = 0, z = ncuts;
      while (a < z) {
        int mid = (a + z) >> 1;
        if (__ldg(cuts_g + mid) < r) a = mid + 1; else z = mid;
      }
      return (uint32_t)a;
    };
    encode_chunks<T, B>(base, cur, geo, packed, scratch, counts, my, [&](T b, T x) -> uint32_t {
      return classify<T>(b, x, find, centers_g, tol_bin, tol, sentinel);
    });
  }
}

// Finalize: chunk offsets -> compacted exact list + per-block prefix.
// One thread per chunk for the bookkeeping; chunks with more than a few
// incompressible values are copied by the whole warp, one chunk at a time.
template <typename T>
__global__ void __launch_bounds__(256)
k_enc_finalize(EncodeGeom geo, const uint32_t* __restrict__ counts, const unsigned long long* __restrict__ offsets,
               const T* __restrict__ scratch, T* __restrict__ exact, unsigned long long* __restrict__ prefix,
               unsigned long long* __restrict__ n_inc) {
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_inc = offsets[geo.nchunks];
  const uint32_t cpb = (uint32_t)geo.cpb;
  const uint32_t nthr = gridDim.x * blockDim.x;
  for (uint32_t c0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); c0 < (uint32_t)geo.nchunks; c0 += nthr) {
    const uint32_t c = c0 + lane;
    const bool in = c < (uint32_t)geo.nchunks;
    const unsigned n = in ? counts[c] : 0u;
    const unsigned long long off = in ? offsets[c] : 0ULL;
    if (in) {
      const uint32_t g = (uint32_t)geo.g0 + c;
      const uint32_t b = geo.fd_cpb.div(g);
      if (g == b * cpb && (uint64_t)b * geo.epb >= geo.elem0) prefix[b - geo.b0] = off;
      if (n <= 4)
        for (unsigned i = 0; i < n; ++i) exact[off + i] = scratch[(uint64_t)c * kChunk + i];
    }
    unsigned big = __ballot_sync(0xffffffffu, n > 4);
    while (big) {
      const int src = __ffs(big) - 1;
      big &= big - 1;
      const unsigned nn = __shfl_sync(0xffffffffu, n, src);
      const unsigned long long oo = __shfl_sync(0xffffffffu, off, src);
      const uint64_t cs = (uint64_t)(c0 + src) * kChunk;
      for (unsigned i = lane; i < nn; i += 32) exact[oo + i] = scratch[cs + i];
    }
  }
}

// ---- standalone pack/unpack (codec.pack_block / unpack_block) -------------
template <int B>
__device__ __forceinline__ void unpack8(const uint8_t* src, uint32_t (&code)[kGroup]) {
  unsigned long long acc = 0;
  int nacc = 0, bi = 0;
#pragma unroll
  for (int e = 0; e < kGroup; ++e) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (nacc < B) {
        acc = (acc << 8) | src[bi++];
        nacc += 8;
      }
    }
    code[e] = (uint32_t)(acc >> (nacc - B)) & ((1u << B) - 1u);
    nacc -= B;
  }
}

template <int B>
__global__ void k_pack(const uint32_t* __restrict__ codes, uint64_t n, uint8_t* __restrict__ out) {
  const uint64_t ngrp = (n + kGroup - 1) / kGroup;
  const uint64_t nbytes = (n * B + 7) / 8;
  for (uint64_t gi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < ngrp;
       gi += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t c[kGroup];
#pragma unroll
    for (int e = 0; e < kGroup; ++e) {
      uint64_t j = gi * kGroup + e;
      c[e] = j < n ? codes[j] : 0u;
    }
    uint8_t tmp[B + 16];
    uint8_t* al = reinterpret_cast<uint8_t*>(((uintptr_t)tmp + 15) & ~(uintptr_t)15);
    pack8<B>(c, al);
#pragma unroll
    for (int w = 0; w < B; ++w) {
      uint64_t o = gi * B + w;
      if (o < nbytes) out[o] = al[w];
    }
  }
}

template <int B>
__global__ void k_unpack(const uint8_t* __restrict__ in, uint64_t n, uint32_t* __restrict__ codes) {
  const uint64_t ngrp = (n + kGroup - 1) / kGroup;
  const uint64_t nbytes = (n * B + 7) / 8;
  for (uint64_t gi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < ngrp;
       gi += (uint64_t)gridDim.x * blockDim.x) {
    uint8_t tmp[B];
#pragma unroll
    for (int w = 0; w < B; ++w) {
      uint64_t o = gi * B + w;
      tmp[w] = o < nbytes ? in[o] : 0;
    }
    uint32_t c[kGroup];
    unpack8<B>(tmp, c);
#pragma unroll
    for (int e = 0; e < kGroup; ++e) {
      uint64_t j = gi * kGroup + e;
      if (j < n) codes[j] = c[e];
    }
  }
}

static int sm_count_e() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

struct EncodeChunks {
  uint64_t b0, cpb, g0, nchunks;
};

static EncodeChunks encode_chunks(uint64_t n_local, uint64_t elem0, uint64_t epb) {
  EncodeChunks et{};
  if (n_local == 0 || epb == 0) return et;
  et.cpb = (epb + kChunk - 1) / kChunk;
  uint64_t last = elem0 + n_local - 1;
  uint64_t b0 = elem0 / epb, b1 = last / epb;
  uint64_t c0 = (elem0 - b0 * epb) / kChunk, c1 = (last - b1 * epb) / kChunk;
  et.b0 = b0;
  et.g0 = b0 * et.cpb + c0;
  et.nchunks = (b1 * et.cpb + c1) - et.g0 + 1;
  return et;
}

static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

// workspace: counts u32[nchunks] | offsets u64[nchunks] | total | scan ws | scratch T[nchunks*256]
struct EncodeWs {
  size_t off_counts, off_offsets, off_total, off_scan, off_scratch, total;
};

static EncodeWs encode_ws_layout(uint64_t nchunks, int elem_bytes) {
  EncodeWs w{};
  w.off_counts = 0;
  w.off_offsets = al256(nchunks * 4);
  w.off_total = w.off_offsets + al256(nchunks * 8 + 8);   // offsets[nchunks] = total
  w.off_scan = w.off_total + 256;
  w.off_scratch = w.off_scan + al256(chunk_scan_ws_bytes(nchunks));
  w.total = w.off_scratch + al256(nchunks * kChunk * (size_t)elem_bytes);
  return w;
}

template <typename T, int B>
static void launch_encode(const void* base, const void* cur, const EncodeGeom& geo, const double* centers,
                          const double* cuts, int k, double tol_bin, double tol, uint8_t* packed, void* scratch,
                          uint32_t* counts, const nmk_model* model, int k_cap, cudaStream_t s) {
  const bool smem_ok = k_cap <= kSmemCuts + 1;
  const size_t smem = smem_ok ? (size_t)(k_cap + 2) * 8 : 0;
  static size_t attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(k_encode<T, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_encode<T, B>, kEncThreads, smem);
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = (uint64_t)sm_count_e() * per_sm;
  uint64_t need = (geo.nchunks + 7) / 8;
  if (grid > need) grid = need;
  k_encode<T, B><<<(unsigned)grid, kEncThreads, smem, s>>>((const T*)base, (const T*)cur, geo, centers, cuts, k,
                                                           tol_bin, tol, packed, (T*)scratch, counts, model, smem_ok);
}

template <typename T>
static int dispatch_encode(int bits, const void* base, const void* cur, const EncodeGeom& geo, const double* centers,
                           const double* cuts, int k, double tol_bin, double tol, uint8_t* packed, void* scratch,
                           uint32_t* counts, const nmk_model* model, int k_cap, cudaStream_t s) {
  switch (bits) {
#define NMK_ENC_CASE(BB)                                                                                           \
  case BB: launch_encode<T, BB>(base, cur, geo, centers, cuts, k, tol_bin, tol, packed, scratch, counts, model, \
                                k_cap, s); break;
    NMK_ENC_CASE(2) NMK_ENC_CASE(3) NMK_ENC_CASE(4) NMK_ENC_CASE(5) NMK_ENC_CASE(6) NMK_ENC_CASE(7)
    NMK_ENC_CASE(8) NMK_ENC_CASE(9) NMK_ENC_CASE(10) NMK_ENC_CASE(11) NMK_ENC_CASE(12) NMK_ENC_CASE(13)
    NMK_ENC_CASE(14) NMK_ENC_CASE(15) NMK_ENC_CASE(16) NMK_ENC_CASE(17) NMK_ENC_CASE(18) NMK_ENC_CASE(19)
    NMK_ENC_CASE(20) NMK_ENC_CASE(21) NMK_ENC_CASE(22) NMK_ENC_CASE(23) NMK_ENC_CASE(24) NMK_ENC_CASE(25)
    NMK_ENC_CASE(26) NMK_ENC_CASE(27) NMK_ENC_CASE(28) NMK_ENC_CASE(29) NMK_ENC_CASE(30)
#undef NMK_ENC_CASE
    default: return set_error(NMK_ERR_ARG, "nmk_encode: bits %d outside [2, 30]", bits);
  }
  return check_launch("k_encode");
}

// Shared body of nmk_encode / nmk_encode_dev.
static int encode_impl(const void* base, const void* cur, uint64_t n_local, uint64_t elem0, uint64_t n_total,
                       int dtype, const double* centers, const double* cuts, int k, const nmk_model* model,
                       int k_cap, int bits, double tol_bin, double tolerance, uint64_t epb, uint8_t* packed,
                       uint64_t block_stride, void* exact, unsigned long long* prefix, unsigned long long* n_inc,
                       void* ws, size_t ws_bytes, cudaStream_t s);

}  // namespace nmk

using namespace nmk;

extern "C" size_t nmk_encode_ws_bytes(uint64_t n_local, uint64_t elem0, uint64_t epb, int dtype) {
  EncodeChunks et = encode_chunks(n_local, elem0, epb);
  return encode_ws_layout(et.nchunks, dtype == NMK_F32 ? 4 : 8).total;
}

static int nmk::encode_impl(const void* base, const void* cur, uint64_t n_local, uint64_t elem0, uint64_t n_total,
                            int dtype, const double* centers, const double* cuts, int k, const nmk_model* model,
                            int k_cap, int bits, double tol_bin, double tolerance, uint64_t epb, uint8_t* packed,
                            uint64_t block_stride, void* exact, unsigned long long* prefix,
                            unsigned long long* n_inc, void* ws, size_t ws_bytes, cudaStream_t s) {
  if (n_local == 0) {
    cudaMemsetAsync(n_inc, 0, sizeof(unsigned long long), s);
    return check_launch("nmk_encode(empty)");
  }
  if (!base || !cur || !centers || !packed || !exact || !prefix || !n_inc || !ws || k < 1 || k_cap < k)
    return set_error(NMK_ERR_ARG, "nmk_encode: bad argument");
  if (dtype != NMK_F32 && dtype != NMK_F64) return set_error(NMK_ERR_ARG, "nmk_encode: bad dtype");
  if (k_cap > 1 && !cuts) return set_error(NMK_ERR_ARG, "nmk_encode: cuts required for k > 1");
  if (bits < 2 || bits > 30) return set_error(NMK_ERR_ARG, "nmk_encode: bits %d outside [2, 30]", bits);
  if ((uint64_t)k_cap > (1ULL << bits) - 1) return set_error(NMK_ERR_ARG, "nmk_encode: k %d exceeds 2^B-1", k_cap);
  if (epb == 0 || elem0 + n_local > n_total) return set_error(NMK_ERR_ARG, "nmk_encode: bad geometry");
  if (block_stride % 16 || block_stride < (epb * bits + 7) / 8)
    return set_error(NMK_ERR_ARG, "nmk_encode: block_stride must be >= ceil(epb*B/8) and a multiple of 16");
  if ((uintptr_t)packed & 15) return set_error(NMK_ERR_ARG, "nmk_encode: packed must be 16-byte aligned");
  const size_t need = nmk_encode_ws_bytes(n_local, elem0, epb, dtype);
  if (ws_bytes < need) return set_error(NMK_ERR_ARG, "nmk_encode: workspace too small");
  EncodeChunks et = encode_chunks(n_local, elem0, epb);
  if (epb >= (1ULL << 31) || (n_total + kChunk - 1) / kChunk >= (1ULL << 32))
    return set_error(NMK_ERR_ARG, "nmk_encode: block or stream too large for 32-bit chunk indexing");
  EncodeGeom geo{n_local, elem0, n_total, epb, et.cpb, et.g0, et.nchunks, et.b0, block_stride, FastDiv{}};
  geo.fd_cpb.init((uint32_t)et.cpb);
  EncodeWs w = encode_ws_layout(et.nchunks, dtype == NMK_F32 ? 4 : 8);
  char* wb = (char*)ws;
  uint32_t* counts = (uint32_t*)(wb + w.off_counts);
  unsigned long long* offsets = (unsigned long long*)(wb + w.off_offsets);
  void* scratch = wb + w.off_scratch;
  // A range starting inside a block: zero the packed bytes of the chunks in
  // front of it so they decode as non-sentinel codes and OR-merge neutrally.
  const uint64_t c0_in_blk = (elem0 - et.b0 * epb) / kChunk;
  if (c0_in_blk) cudaMemsetAsync(packed, 0, c0_in_blk * (uint64_t)(32 * bits), s);
  int rc = (dtype == NMK_F64)
               ? dispatch_encode<double>(bits, base, cur, geo, centers, cuts, k, tol_bin, tolerance, packed,
                                         scratch, counts, model, k_cap, s)
               : dispatch_encode<float>(bits, base, cur, geo, centers, cuts, k, tol_bin, tolerance, packed,
                                        scratch, counts, model, k_cap, s);
  if (rc) return rc;
  chunk_scan(counts, et.nchunks, offsets, wb + w.off_scan, s);
  unsigned grid = (unsigned)((et.nchunks + 255) / 256);
  if (grid > (unsigned)sm_count_e() * 8) grid = sm_count_e() * 8;
  if (dtype == NMK_F64)
    k_enc_finalize<double><<<grid, 256, 0, s>>>(geo, counts, offsets, (const double*)scratch, (double*)exact, prefix,
                                                n_inc);
  else
    k_enc_finalize<float><<<grid, 256, 0, s>>>(geo, counts, offsets, (const float*)scratch, (float*)exact, prefix,
                                               n_inc);
  return check_launch("k_enc_finalize");
}

extern "C" int nmk_encode(const void* base, const void* cur, uint64_t n_local, uint64_t elem0, uint64_t n_total,
                          int dtype, const double* centers, const double* cuts, int k, int bits, double tol_bin,
                          double tolerance, uint64_t epb, uint8_t* packed, uint64_t block_stride, void* exact,
                          unsigned long long* prefix, unsigned long long* n_inc, void* ws, size_t ws_bytes,
                          void* stream) {
  return encode_impl(base, cur, n_local, elem0, n_total, dtype, centers, cuts, k, nullptr, k, bits, tol_bin, tolerance,
                     epb, packed, block_stride, exact, prefix, n_inc, ws, ws_bytes, (cudaStream_t)stream);
}

extern "C" int nmk_encode_dev(const void* base, const void* cur, uint64_t n_local, uint64_t elem0, uint64_t n_total,
                              int dtype, const double* centers, const double* cuts, const nmk_model* model,
                              int k_cap, int bits, double tolerance, uint64_t epb, uint8_t* packed,
                              uint64_t block_stride, void* exact, unsigned long long* prefix,
                              unsigned long long* n_inc, void* ws, size_t ws_bytes, void* stream) {
  if (!model) return set_error(NMK_ERR_ARG, "nmk_encode_dev: model required");
  return encode_impl(base, cur, n_local, elem0, n_total, dtype, centers, cuts, 1, model, k_cap, bits, 0.0, tolerance,
                     epb, packed, block_stride, exact, prefix, n_inc, ws, ws_bytes, (cudaStream_t)stream);
}

template <int B>
static void launch_pack(const uint32_t* codes, uint64_t n, uint8_t* out, cudaStream_t s, bool unpack,
                        const uint8_t* in, uint32_t* codes_out) {
  uint64_t ngrp = (n + kGroup - 1) / kGroup;
  unsigned grid = (unsigned)((ngrp + 255) / 256);
  if (grid > 4096) grid = 4096;
  if (grid == 0) grid = 1;
  if (unpack) k_unpack<B><<<grid, 256, 0, s>>>(in, n, codes_out);
  else k_pack<B><<<grid, 256, 0, s>>>(codes, n, out);
}

static int dispatch_pack(int bits, bool unpack, const uint32_t* codes, uint64_t n, uint8_t* out, const uint8_t* in,
                         uint32_t* codes_out, cudaStream_t s) {
  switch (bits) {
#define NMK_PK_CASE(BB) case BB: launch_pack<BB>(codes, n, out, s, unpack, in, codes_out); break;
    NMK_PK_CASE(2) NMK_PK_CASE(3) NMK_PK_CASE(4) NMK_PK_CASE(5) NMK_PK_CASE(6) NMK_PK_CASE(7) NMK_PK_CASE(8)
    NMK_PK_CASE(9) NMK_PK_CASE(10) NMK_PK_CASE(11) NMK_PK_CASE(12) NMK_PK_CASE(13) NMK_PK_CASE(14)
    NMK_PK_CASE(15) NMK_PK_CASE(16) NMK_PK_CASE(17) NMK_PK_CASE(18) NMK_PK_CASE(19) NMK_PK_CASE(20)
    NMK_PK_CASE(21) NMK_PK_CASE(22) NMK_PK_CASE(23) NMK_PK_CASE(24) NMK_PK_CASE(25) NMK_PK_CASE(26)
    NMK_PK_CASE(27) NMK_PK_CASE(28) NMK_PK_CASE(29) NMK_PK_CASE(30)
#undef NMK_PK_CASE
    default: return set_error(NMK_ERR_ARG, "bits %d outside [2, 30]", bits);
  }
  return check_launch(unpack ? "k_unpack" : "k_pack");
}

extern "C" int nmk_pack(const uint32_t* codes, uint64_t n, int bits, uint8_t* out, void* stream) {
  if (n == 0) return NMK_OK;
  if (!codes || !out) return set_error(NMK_ERR_ARG, "nmk_pack: null pointer");
  return dispatch_pack(bits, false, codes, n, out, nullptr, nullptr, (cudaStream_t)stream);
}

extern "C" int nmk_unpack(const uint8_t* packed, uint64_t n, int bits, uint32_t* codes, void* stream) {
  if (n == 0) return NMK_OK;
  if (!packed || !codes) return set_error(NMK_ERR_ARG, "nmk_unpack: null pointer");
  return dispatch_pack(bits, true, nullptr, n, nullptr, packed, codes, (cudaStream_t)stream);
}
