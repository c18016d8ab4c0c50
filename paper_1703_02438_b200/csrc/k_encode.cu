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
// finalize pass (k_enc_finalize: tile scan with look-back + gather) turns the
// counts into positions, moves the (rare) values into the compacted list and
// fills the per-block prefix table.
#include "k_encode.cuh"
#include "nmk_scan.cuh"

namespace nmk {

// instantiated in k_encode_b*.cu
#define NMK_ENC_EXTERN(BB)                                                                                      \
  extern template void launch_encode<double, BB>(const void*, const void*, const EncodeGeom&, const double*,      \
                                                 const double*, int, double, double, uint8_t*, void*, uint32_t*, \
                                                 const nmk_model*, int, void*, const EncodeKeys&, cudaStream_t);                     \
  extern template void launch_encode<float, BB>(const void*, const void*, const EncodeGeom&, const double*,       \
                                                const double*, int, double, double, uint8_t*, void*, uint32_t*,  \
                                                const nmk_model*, int, void*, const EncodeKeys&, cudaStream_t);
NMK_ENC_EXTERN(2) NMK_ENC_EXTERN(3) NMK_ENC_EXTERN(4) NMK_ENC_EXTERN(5) NMK_ENC_EXTERN(6) NMK_ENC_EXTERN(7)
NMK_ENC_EXTERN(8) NMK_ENC_EXTERN(9) NMK_ENC_EXTERN(10) NMK_ENC_EXTERN(11) NMK_ENC_EXTERN(12) NMK_ENC_EXTERN(13)
NMK_ENC_EXTERN(14) NMK_ENC_EXTERN(15) NMK_ENC_EXTERN(16) NMK_ENC_EXTERN(17) NMK_ENC_EXTERN(18) NMK_ENC_EXTERN(19)
NMK_ENC_EXTERN(20) NMK_ENC_EXTERN(21) NMK_ENC_EXTERN(22) NMK_ENC_EXTERN(23) NMK_ENC_EXTERN(24) NMK_ENC_EXTERN(25)
NMK_ENC_EXTERN(26) NMK_ENC_EXTERN(27) NMK_ENC_EXTERN(28) NMK_ENC_EXTERN(29) NMK_ENC_EXTERN(30)
#undef NMK_ENC_EXTERN

#ifndef NMK_FIN_UNROLL
#define NMK_FIN_UNROLL 0
#endif
#ifndef NMK_FIN_GATHER_BIG
#define NMK_FIN_GATHER_BIG 4   // A/B (cfg5 B12 E1e-4, 30 values per chunk): 4 beats the per-thread loop (32)
#endif
// Finalize: chunk counts -> compacted exact list + per-block prefix, in one
// launch.  A CTA takes a tile of kFinTile consecutive chunks (lane = chunk,
// kFinRounds rounds per warp), scans their counts (warp shuffles + one CTA
// step), obtains the tile's exclusive prefix by decoupled look-back over the
// tile-status words (nmk_scan.cuh; cleared by the encode kernel in front) and
// then moves the values with the offsets still in registers -- no offsets
// array, no separate scan launch.  The values come either from the chunk's
// scratch window (k_encode: chunks with more than a few values are copied by
// the whole warp, one chunk at a time) or, after k_encode_keyed
// (*keyed_done), straight from `cur` at the positions of the chunk's 256-bit
// mask (one byte per lane of the encoding warp).
constexpr int kFinThreads = 256;
#ifndef NMK_FIN_ROUNDS
#define NMK_FIN_ROUNDS 2   // A/B on cfg2: 1 -> 1.121 ms step, 2 -> 1.115, 4 -> 1.123 (fewer, longer-lived threads)
#endif
constexpr int kFinRounds = NMK_FIN_ROUNDS;
constexpr int kFinTile = kFinThreads * kFinRounds;   // chunks per CTA

template <typename T>
__global__ void __launch_bounds__(kFinThreads)
k_enc_finalize(EncodeGeom geo, const uint32_t* __restrict__ counts, unsigned long long* __restrict__ status,
               const T* __restrict__ scratch, T* __restrict__ exact, unsigned long long* __restrict__ prefix,
               unsigned long long* __restrict__ n_inc, const T* __restrict__ cur,
               const uint32_t* __restrict__ keyed_done) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  pdl_enter();
  const uint32_t nch = (uint32_t)geo.nchunks;
  const uint32_t wc0 = blockIdx.x * (uint32_t)kFinTile + (uint32_t)wid * (32 * kFinRounds);   // the warp's first chunk
  // ---- scan of the tile's counts -----------------------------------------
  unsigned cnt[kFinRounds], ex[kFinRounds];
#pragma unroll
  for (int q = 0; q < kFinRounds; ++q) {
    const uint32_t c = wc0 + q * 32 + lane;
    cnt[q] = c < nch ? __ldcs(counts + c) : 0u;
  }
  unsigned wsum = 0;   // warp running total (uniform; a tile holds <= kFinTile * 256 values)
#pragma unroll
  for (int q = 0; q < kFinRounds; ++q) {
    unsigned incl = cnt[q];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    ex[q] = wsum + incl - cnt[q];
    wsum += __shfl_sync(0xffffffffu, incl, 31);
  }
  __shared__ unsigned s_warp[kFinThreads / 32];
  __shared__ unsigned long long s_prefix;
  if (lane == 0) s_warp[wid] = wsum;
  __syncthreads();
  unsigned wbase = 0, agg = 0;
#pragma unroll
  for (int w = 0; w < kFinThreads / 32; ++w) {
    const unsigned x = s_warp[w];
    wbase += w < wid ? x : 0u;
    agg += x;
  }
  if (wid == 0) {
    const unsigned long long p = scan_lookback(status, blockIdx.x, agg, lane);
    if (lane == 0) {
      s_prefix = p;
      if (blockIdx.x == gridDim.x - 1) *n_inc = p + agg;   // the last tile knows the total
    }
  }
  __syncthreads();
  const unsigned long long wstart = s_prefix + wbase;
  // ---- the values ------------------------------------------------------------
  const bool gather = keyed_done && *keyed_done;
  const uint8_t* masks = reinterpret_cast<const uint8_t*>(scratch);
  const uint32_t cpb = (uint32_t)geo.cpb;
  // local index of element 0 of lane l's group in chunk c: chunk_lo - elem0 + 8 l
  auto chunk_li = [&](uint32_t c) -> int64_t {
    const uint32_t g = (uint32_t)geo.g0 + c;
    const uint32_t b = geo.fd_cpb.div(g);
    return (int64_t)((uint64_t)b * geo.epb + (uint64_t)(g - b * cpb) * kChunk) - (int64_t)geo.elem0;
  };
  // chunks with more values than this go to the warp-cooperative copy (one
  // chunk per warp iteration, every lane's loads issued together)
  const unsigned big_at = gather ? (unsigned)NMK_FIN_GATHER_BIG : 4u;
#pragma unroll
  for (int q = 0; q < kFinRounds; ++q) {
    const uint32_t c0 = wc0 + q * 32;
    if (c0 >= nch) break;   // warp-uniform
    const uint32_t c = c0 + lane;
    const bool in = c < nch;
    const unsigned n = cnt[q];
    const unsigned long long off = wstart + ex[q];
    if (in) {
      const uint32_t g = (uint32_t)geo.g0 + c;
      const uint32_t b = geo.fd_cpb.div(g);
      if (g == b * cpb && (uint64_t)b * geo.epb >= geo.elem0) prefix[b - geo.b0] = off;
      if (n && n <= big_at) {
        if (gather) {
          const uint4* mp = reinterpret_cast<const uint4*>(masks + (uint64_t)c * 32);
          const uint4 m0 = mp[0], m1 = mp[1];
          const uint32_t mw[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
          const int64_t li = chunk_li(c);
          unsigned long long o = off;
#pragma unroll
          for (int w = 0; w < 8; ++w)
            for (uint32_t m = mw[w]; m; m &= m - 1u) {   // bit 8 l + e of the mask = element 8 l + e
              const int bit = __ffs(m) - 1;
              exact[o++] = cur[li + w * 32 + bit];
            }
        } else {
          for (unsigned i = 0; i < n; ++i) exact[off + i] = scratch[(uint64_t)c * kChunk + i];
        }
      }
    }
    unsigned big = __ballot_sync(0xffffffffu, n > big_at);
    while (big) {
      const int src = __ffs(big) - 1;
      big &= big - 1;
      const unsigned nn = __shfl_sync(0xffffffffu, n, src);
      const unsigned long long oo = __shfl_sync(0xffffffffu, off, src);
      const uint32_t cb = c0 + src;
      if (gather) {   // lane l handles its byte of the mask: warp scan for the output slot
        const unsigned m = masks[(uint64_t)cb * 32 + lane];
        const unsigned mc = __popc(m);
        unsigned incl = mc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        const int64_t li = chunk_li(cb) + lane * kGroup;
        unsigned long long o = oo + (incl - mc);
#if NMK_FIN_UNROLL
        T v[kGroup];
#pragma unroll
        for (int e = 0; e < kGroup; ++e)
          if (m >> e & 1u) v[e] = cur[li + e];   // independent loads, all in flight
#pragma unroll
        for (int e = 0; e < kGroup; ++e)
          if (m >> e & 1u) exact[o++] = v[e];
#else
        for (unsigned mm = m; mm; mm &= mm - 1u) exact[o++] = cur[li + __ffs(mm) - 1];
#endif
      } else {
        const uint64_t cs = (uint64_t)cb * kChunk;
        for (unsigned i = lane; i < nn; i += 32) exact[oo + i] = scratch[cs + i];
      }
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

// workspace: counts u32[nchunks] | flags | finalize tile status | scratch T[nchunks*256]
struct EncodeWs {
  size_t off_counts, off_total, off_scan, off_scratch, total;
};

static EncodeWs encode_ws_layout(uint64_t nchunks, int elem_bytes) {
  EncodeWs w{};
  w.off_counts = 0;
  w.off_total = al256(nchunks * 4);   // 256 bytes of flags (the keyed-mode word at + 128)
  w.off_scan = w.off_total + 256;
  w.off_scratch = w.off_scan + al256(((nchunks + kFinTile - 1) / kFinTile) * 8 + 256);   // finalize tile status
  w.total = w.off_scratch + al256(nchunks * kChunk * (size_t)elem_bytes);
  return w;
}

template <typename T>
static int dispatch_encode(int bits, const void* base, const void* cur, const EncodeGeom& geo, const double* centers,
                           const double* cuts, int k, double tol_bin, double tol, uint8_t* packed, void* scratch,
                           uint32_t* counts, const nmk_model* model, int k_cap, void* recon, const EncodeKeys& kx,
                           cudaStream_t s) {
  switch (bits) {
#define NMK_ENC_CASE(BB)                                                                                           \
  case BB: launch_encode<T, BB>(base, cur, geo, centers, cuts, k, tol_bin, tol, packed, scratch, counts, model, \
                                k_cap, recon, kx, s); break;
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
                       void* recon, const EncodeKeys& kx, void* ws, size_t ws_bytes, cudaStream_t s);

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
                            unsigned long long* n_inc, void* recon, const EncodeKeys& kx, void* ws, size_t ws_bytes,
                            cudaStream_t s) {
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
  EncodeGeom geo{n_local, elem0, n_total, epb, et.cpb, et.g0, et.nchunks, et.b0, block_stride, FastDiv{}, 0, 0, false,
                 ZeroList{}};
  geo.fd_cpb.init((uint32_t)et.cpb);
  {
    auto chunk_lo = [&](uint64_t c) {   // first element of local chunk c
      const uint64_t g = et.g0 + c, b = g / et.cpb;
      return b * epb + (g - b * et.cpb) * kChunk;
    };
    const uint64_t local_end = elem0 + n_local;
    geo.c_first = chunk_lo(0) == elem0 ? 0u : 1u;
    const uint64_t last = et.nchunks - 1;
    geo.c_last = (uint32_t)(chunk_lo(last) + kChunk <= local_end ? last : (last ? last - 1 : 0));
    if (et.nchunks == 1 && chunk_lo(0) + kChunk > local_end) geo.c_first = 1;   // no whole chunk
    geo.key_al = elem0 % 4 == 0 && epb % 4 == 0;
  }
  EncodeWs w = encode_ws_layout(et.nchunks, dtype == NMK_F32 ? 4 : 8);
  char* wb = (char*)ws;
  geo.zl.p[0] = (unsigned long long*)(wb + w.off_scan);   // the scan's tile status: zeroed by the encode kernels
  geo.zl.n[0] = (uint32_t)((et.nchunks + kFinTile - 1) / kFinTile);
  EncodeKeys kxw = kx;
  kxw.done = (uint32_t*)(wb + w.off_total + 128);   // keyed-mode flag (k_encode_keyed -> k_encode, finalize)
  const bool keyed = kx.keys && model && k_cap <= kSmemCuts + 1;   // launch_encode_k's condition
  uint32_t* counts = (uint32_t*)(wb + w.off_counts);
  void* scratch = wb + w.off_scratch;
  // A range starting inside a block: zero the packed bytes of the chunks in
  // front of it so they decode as non-sentinel codes and OR-merge neutrally.
  const uint64_t c0_in_blk = (elem0 - et.b0 * epb) / kChunk;
  if (c0_in_blk) cudaMemsetAsync(packed, 0, c0_in_blk * (uint64_t)(32 * bits), s);
  int rc = (dtype == NMK_F64)
               ? dispatch_encode<double>(bits, base, cur, geo, centers, cuts, k, tol_bin, tolerance, packed,
                                         scratch, counts, model, k_cap, recon, kxw, s)
               : dispatch_encode<float>(bits, base, cur, geo, centers, cuts, k, tol_bin, tolerance, packed,
                                        scratch, counts, model, k_cap, recon, kxw, s);
  if (rc) return rc;
  unsigned long long* status = (unsigned long long*)(wb + w.off_scan);
  const unsigned grid = (unsigned)((et.nchunks + kFinTile - 1) / kFinTile);
  if (dtype == NMK_F64)
    launch_chain(kPdlFinalize, k_enc_finalize<double>, grid, kFinThreads, 0, s, geo, counts, status, (const double*)scratch,
                 (double*)exact, prefix, n_inc, (const double*)cur, keyed ? kxw.done : nullptr);
  else
    launch_chain(kPdlFinalize, k_enc_finalize<float>, grid, kFinThreads, 0, s, geo, counts, status, (const float*)scratch,
                 (float*)exact, prefix, n_inc, (const float*)cur, keyed ? kxw.done : nullptr);
  return check_launch("k_enc_finalize");
}

extern "C" int nmk_encode(const void* base, const void* cur, uint64_t n_local, uint64_t elem0, uint64_t n_total,
                          int dtype, const double* centers, const double* cuts, int k, int bits, double tol_bin,
                          double tolerance, uint64_t epb, uint8_t* packed, uint64_t block_stride, void* exact,
                          unsigned long long* prefix, unsigned long long* n_inc, void* recon, void* ws,
                          size_t ws_bytes, void* stream) {
  return encode_impl(base, cur, n_local, elem0, n_total, dtype, centers, cuts, k, nullptr, k, bits, tol_bin, tolerance,
                     epb, packed, block_stride, exact, prefix, n_inc, recon, EncodeKeys{nullptr, nullptr, 0.0, nullptr, 0}, ws,
                     ws_bytes, (cudaStream_t)stream);
}

extern "C" int nmk_encode_dev(const void* base, const void* cur, uint64_t n_local, uint64_t elem0, uint64_t n_total,
                              int dtype, const double* centers, const double* cuts, const nmk_model* model,
                              int k_cap, int bits, double tolerance, uint64_t epb, uint8_t* packed,
                              uint64_t block_stride, void* exact, unsigned long long* prefix,
                              unsigned long long* n_inc, void* recon, void* ws, size_t ws_bytes, void* stream) {
  if (!model) return set_error(NMK_ERR_ARG, "nmk_encode_dev: model required");
  return encode_impl(base, cur, n_local, elem0, n_total, dtype, centers, cuts, 1, model, k_cap, bits, 0.0, tolerance,
                     epb, packed, block_stride, exact, prefix, n_inc, recon, EncodeKeys{nullptr, nullptr, 0.0, nullptr, 0}, ws,
                     ws_bytes, (cudaStream_t)stream);
}

extern "C" int nmk_encode_keyed_dev2(const float* keys, const nmk_stats* stats, double width, const void* base,
                                     const void* cur, uint64_t n_local, uint64_t elem0, uint64_t n_total, int dtype,
                                     const double* centers, const double* cuts, const nmk_model* model, int k_cap,
                                     int bits, double tolerance, uint64_t epb, uint8_t* packed, uint64_t block_stride,
                                     void* exact, unsigned long long* prefix, unsigned long long* n_inc, void* recon,
                                     int keyed_hint, void* ws, size_t ws_bytes, void* stream) {
  if (!model || !keys || !stats) return set_error(NMK_ERR_ARG, "nmk_encode_keyed_dev: model, keys and stats required");
  if ((uintptr_t)keys & 15) return set_error(NMK_ERR_ARG, "nmk_encode_keyed_dev: keys must be 16-byte aligned");
  return encode_impl(base, cur, n_local, elem0, n_total, dtype, centers, cuts, 1, model, k_cap, bits, 0.0, tolerance,
                     epb, packed, block_stride, exact, prefix, n_inc, recon,
                     EncodeKeys{keys, stats, width, nullptr, keyed_hint == 1 ? 1 : 0}, ws, ws_bytes, (cudaStream_t)stream);
}

extern "C" int nmk_encode_keyed_dev(const float* keys, const nmk_stats* stats, double width, const void* base,
                                    const void* cur, uint64_t n_local, uint64_t elem0, uint64_t n_total, int dtype,
                                    const double* centers, const double* cuts, const nmk_model* model, int k_cap,
                                    int bits, double tolerance, uint64_t epb, uint8_t* packed, uint64_t block_stride,
                                    void* exact, unsigned long long* prefix, unsigned long long* n_inc, void* recon,
                                    void* ws, size_t ws_bytes, void* stream) {
  return nmk_encode_keyed_dev2(keys, stats, width, base, cur, n_local, elem0, n_total, dtype, centers, cuts, model, k_cap,
                               bits, tolerance, epb, packed, block_stride, exact, prefix, n_inc, recon, 0, ws, ws_bytes,
                               stream);
}

extern "C" size_t nmk_encode_ws_mode_offset(uint64_t n_local, uint64_t elem0, uint64_t epb, int dtype) {
  EncodeChunks et = encode_chunks(n_local, elem0, epb);
  return encode_ws_layout(et.nchunks, dtype == NMK_F32 ? 4 : 8).off_total + 128;
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
