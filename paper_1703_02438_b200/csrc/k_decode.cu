// k_decode.cu — K5: fused unpack + sentinel scan + reconstruct, batched over
// element ranges ("segments").
//
// Replaces, for full and partial decompression, the per-block loop of
// codec._decode_range (pkg/src/nmk/codec.py:204-239): unpack_block
// (codec.py:95-105), the seek into the incompressible table
// (inc_before = prefix[first] + #sentinels ahead, codec.py:231-236) and
// core.reconstruct (core.py:158-208): sentinel -> next exact value (raw
// bits), otherwise T((1 + c[idx]) * f64(base)); ids in [k, sentinel) are an
// error, as is running out of exact values.
//
// Tiles are the encode tiles (2048 elements on the block grid).  A segment
// covers a run of consecutive tiles; its first tile is seeded with
// prefix_rel[block] + #sentinels between the block start and the tile (one
// small pre-count CTA per segment), and the running sentinel rank inside the
// segment is carried by a decoupled look-back, so no element is read twice.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "nmk_common.cuh"

namespace nmk {

template <int B>
__device__ __forceinline__ void unpack8d(const uint8_t* src, uint32_t (&code)[kGroup]) {
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

struct Seg {
  uint64_t start, count, out;   // global element range, output offset
  uint64_t tile0;               // first tile (linear, across segments)
  uint64_t gfirst;              // block-grid tile id of the first tile
};

struct DecodeGeom {
  uint64_t epb, tpb, n_total, first_block, stride, n_exact, total_tiles;
  int nseg, k;
};

template <typename T> struct DVec;
template <> struct DVec<double> { using V = double2; static constexpr int N = 2; };
template <> struct DVec<float>  { using V = float4;  static constexpr int N = 4; };

// pre-count: seed[s] = prefix_rel[block(start)] + #sentinels in
// [block start, first tile start) — one CTA per segment.
template <int B>
__global__ void __launch_bounds__(kTileThreads)
k_decode_seed(const uint8_t* __restrict__ packed, const Seg* __restrict__ segs, DecodeGeom geo,
              const unsigned long long* __restrict__ prefix_rel, unsigned long long* __restrict__ seed) {
  typedef cub::BlockReduce<unsigned long long, kTileThreads> BR;
  __shared__ typename BR::TempStorage tmp;
  const Seg sg = segs[blockIdx.x];
  const uint64_t b = sg.gfirst / geo.tpb, ti = sg.gfirst % geo.tpb;
  const uint32_t sentinel = (1u << B) - 1u;
  const uint8_t* blk = packed + (b - geo.first_block) * geo.stride;
  unsigned long long cnt = 0;
  const uint64_t ngrp = ti * kTileThreads;  // whole groups before the first tile
  for (uint64_t gi = threadIdx.x; gi < ngrp; gi += kTileThreads) {
    uint32_t c[kGroup];
    unpack8d<B>(blk + gi * B, c);
#pragma unroll
    for (int e = 0; e < kGroup; ++e) cnt += (c[e] == sentinel);
  }
  unsigned long long tot = BR(tmp).Sum(cnt);
  if (threadIdx.x == 0) seed[blockIdx.x] = prefix_rel[b - geo.first_block] + tot;
}

template <typename T, int B>
__global__ void __launch_bounds__(kTileThreads)
k_decode(const uint8_t* __restrict__ packed, DecodeGeom geo, const Seg* __restrict__ segs,
         const unsigned long long* __restrict__ seed, const double* __restrict__ centers_g,
         const T* __restrict__ exact, const T* __restrict__ base, T* __restrict__ out,
         nmk_segment_info* __restrict__ info, nmk_decode_err* __restrict__ err,
         unsigned long long* __restrict__ status, unsigned int* __restrict__ ticket) {
  typedef cub::BlockScan<unsigned, kTileThreads> BScan;
  typedef cub::BlockReduce<unsigned, kTileThreads> BRed;
  __shared__ union {
    typename BScan::TempStorage scan;
    typename BRed::TempStorage red;
  } tmp;
  __shared__ __align__(16) uint8_t tile_bytes[kTileThreads * B + 16];
  __shared__ unsigned long long s_tile, s_excl;
  extern __shared__ double smc[];

  const int tid = threadIdx.x;
  const int k = geo.k;
  const double* C = centers_g;
  if (k <= 4096) {
    for (int i = tid; i < k; i += kTileThreads) smc[i] = centers_g[i];
    C = smc;
  }
  const uint32_t sentinel = (1u << B) - 1u;

  for (;;) {
    if (tid == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint64_t t = s_tile;
    if (t >= geo.total_tiles) break;
    // segment lookup (segments are few; binary search over tile0)
    int lo_s = 0, hi_s = geo.nseg - 1;
    while (lo_s < hi_s) {
      int mid = (lo_s + hi_s + 1) >> 1;
      if (segs[mid].tile0 <= t) lo_s = mid; else hi_s = mid - 1;
    }
    const Seg sg = segs[lo_s];
    const uint64_t lt = t - sg.tile0;
    const uint64_t g = sg.gfirst + lt;
    const uint64_t b = g / geo.tpb, ti = g % geo.tpb;
    const uint64_t blk_start = b * geo.epb;
    uint64_t blk_end = blk_start + geo.epb;
    if (blk_end > geo.n_total) blk_end = geo.n_total;
    const uint64_t tile_lo = blk_start + ti * kTile;
    uint64_t tile_hi = tile_lo + kTile;
    if (tile_hi > blk_end) tile_hi = blk_end;
    const uint64_t seg_lo = sg.start, seg_hi = sg.start + sg.count;

    // stage this tile's packed bytes
    {
      const uint64_t blk_bytes = ((blk_end - blk_start) * B + 7) / 8;
      const uint64_t off = ti * (uint64_t)(kTileThreads * B);
      uint64_t nbytes = blk_bytes > off ? blk_bytes - off : 0;
      if (nbytes > (uint64_t)kTileThreads * B) nbytes = (uint64_t)kTileThreads * B;
      const uint8_t* src = packed + (b - geo.first_block) * geo.stride + off;
      const uint32_t nvec = (uint32_t)(nbytes / 16);
      for (uint32_t i = tid; i < nvec; i += kTileThreads)
        reinterpret_cast<uint4*>(tile_bytes)[i] = __ldg(reinterpret_cast<const uint4*>(src) + i);
      for (uint32_t i = nvec * 16 + tid; i < (uint32_t)kTileThreads * B; i += kTileThreads)
        tile_bytes[i] = (i < nbytes) ? src[i] : 0;
    }
    __syncthreads();
    uint32_t code[kGroup];
    unpack8d<B>(tile_bytes + tid * B, code);
    const uint64_t grp_lo = tile_lo + (uint64_t)tid * kGroup;
    unsigned smask = 0, inmask = 0;
#pragma unroll
    for (int e = 0; e < kGroup; ++e) {
      uint64_t j = grp_lo + e;
      if (j < tile_hi && code[e] == sentinel) smask |= 1u << e;
      // the last group of a block may run past the block end: those lanes
      // belong to the next block's tile
      if (j >= seg_lo && j < seg_hi && j < tile_hi) inmask |= 1u << e;
    }
    unsigned cnt = __popc(smask), ex, agg;
    BScan(tmp.scan).ExclusiveSum(cnt, ex, agg);
    if (tid == 0) {
      if (lt == 0) st_relaxed(status + t, kFlagInc | (seed[lo_s] + agg));
      else st_relaxed(status + t, kFlagAgg | agg);
    }
    // compressible outputs do not need the look-back: do them first
    const bool full_tile = tile_lo >= seg_lo && tile_hi <= seg_hi;
    const bool full_grp = (inmask == 0xffu);
    T bv[kGroup], ov[kGroup];
    const uint64_t oi = sg.out + (grp_lo - seg_lo);  // valid when grp_lo >= seg_lo
    constexpr int VN = DVec<T>::N;
    const bool vec = full_grp && (oi % VN == 0) && ((((uintptr_t)base | (uintptr_t)out) & 15) == 0);
    if (vec) {
      using V = typename DVec<T>::V;
#pragma unroll
      for (int q = 0; q < kGroup / VN; ++q) {
        V w = __ldg(reinterpret_cast<const V*>(base + oi) + q);
        const T* tw = reinterpret_cast<const T*>(&w);
#pragma unroll
        for (int e = 0; e < VN; ++e) bv[q * VN + e] = tw[e];
      }
    } else {
#pragma unroll
      for (int e = 0; e < kGroup; ++e)
        bv[e] = (inmask >> e & 1u) ? __ldg(base + sg.out + (grp_lo + e - seg_lo)) : T(0);
    }
    unsigned bad = 0, maxbad = 0;
#pragma unroll
    for (int e = 0; e < kGroup; ++e) {
      ov[e] = T(0);
      if (!(inmask >> e & 1u) || (smask >> e & 1u)) continue;
      if (code[e] >= (uint32_t)k) {
        bad = 1;
        maxbad = code[e] > maxbad ? code[e] : maxbad;
        continue;
      }
      ov[e] = apply_center<T>(C[code[e]], to_f64(bv[e]));
    }
    if (bad) {
      atomicOr(&err->bad_index, 1u);
      atomicMax(&err->max_bad_index, maxbad);
    }
    // running sentinel rank
    if (tid < 32) {
      unsigned long long excl = (lt == 0) ? seed[lo_s] : lookback(status, (long long)t, (long long)sg.tile0);
      if (tid == 0) {
        if (lt != 0) st_relaxed(status + t, kFlagInc | (excl + agg));
        s_excl = excl;
      }
    }
    __syncthreads();
    const unsigned long long excl = s_excl;
    unsigned long long pos = excl + ex;
    bool exhausted = false;
#pragma unroll
    for (int e = 0; e < kGroup; ++e) {
      if (smask >> e & 1u) {
        if (inmask >> e & 1u) {
          if (pos < geo.n_exact) ov[e] = exact[pos];
          else exhausted = true;
        }
        ++pos;
      }
    }
    if (exhausted) atomicOr(&err->exhausted, 1u);
    if (vec) {
      using V = typename DVec<T>::V;
#pragma unroll
      for (int q = 0; q < kGroup / VN; ++q) reinterpret_cast<V*>(out + oi)[q] = *reinterpret_cast<const V*>(&ov[q * VN]);
    } else {
#pragma unroll
      for (int e = 0; e < kGroup; ++e)
        if (inmask >> e & 1u) out[sg.out + (grp_lo + e - seg_lo)] = ov[e];
    }
    // segment bookkeeping: sentinels inside the segment, and ahead of it
    if (full_tile) {
      if (tid == 0) atomicAdd(&info[lo_s].n_sentinel, (unsigned long long)agg);
    } else {
      unsigned in_cnt = __popc(smask & inmask);
      unsigned ahead = 0;
#pragma unroll
      for (int e = 0; e < kGroup; ++e)
        if ((smask >> e & 1u) && grp_lo + e < seg_lo) ++ahead;
      __syncthreads();
      unsigned tot_in = BRed(tmp.red).Sum(in_cnt);
      __syncthreads();
      unsigned tot_ahead = BRed(tmp.red).Sum(ahead);
      if (tid == 0) {
        if (tot_in) atomicAdd(&info[lo_s].n_sentinel, (unsigned long long)tot_in);
        if (lt == 0) info[lo_s].inc_before = excl + tot_ahead;
      }
    }
    if (full_tile && lt == 0 && tid == 0) info[lo_s].inc_before = excl;
    __syncthreads();
  }
}

static int sm_count_d() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

struct DecodePlan {
  uint64_t total_tiles;
  size_t off_status, off_segs, off_seed, total;
};

static uint64_t seg_first_tile(uint64_t start, uint64_t epb, uint64_t tpb) {
  uint64_t b = start / epb;
  return b * tpb + (start - b * epb) / kTile;
}

static DecodePlan decode_plan(const uint64_t* st, const uint64_t* ct, int nseg, uint64_t epb) {
  DecodePlan p{};
  uint64_t tpb = (epb + kTile - 1) / kTile;
  uint64_t tiles = 0;
  for (int s = 0; s < nseg; ++s) {
    if (ct[s] == 0) continue;
    uint64_t a = seg_first_tile(st[s], epb, tpb), z = seg_first_tile(st[s] + ct[s] - 1, epb, tpb);
    tiles += z - a + 1;
  }
  p.total_tiles = tiles;
  p.off_status = 256;
  p.off_segs = p.off_status + al256((tiles + 1) * 8);
  p.off_seed = p.off_segs + al256((size_t)(nseg + 1) * sizeof(Seg));
  p.total = p.off_seed + al256((size_t)(nseg + 1) * 8);
  return p;
}

template <typename T, int B>
static void launch_decode(const uint8_t* packed, const DecodeGeom& geo, const Seg* segs, unsigned long long* seed,
                          const unsigned long long* prefix_rel, const double* centers, const void* exact,
                          const void* base, void* out, nmk_segment_info* info, nmk_decode_err* err,
                          unsigned long long* status, unsigned* ticket, cudaStream_t s) {
  k_decode_seed<B><<<geo.nseg, kTileThreads, 0, s>>>(packed, segs, geo, prefix_rel, seed);
  size_t smem = (geo.k <= 4096) ? 4096 * sizeof(double) : 0;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_decode<T, B>, kTileThreads, smem);
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = (uint64_t)sm_count_d() * per_sm;
  if (grid > geo.total_tiles) grid = geo.total_tiles;
  k_decode<T, B><<<(unsigned)grid, kTileThreads, smem, s>>>(packed, geo, segs, seed, centers, (const T*)exact,
                                                            (const T*)base, (T*)out, info, err, status, ticket);
}

template <typename T>
static int dispatch_decode(int bits, const uint8_t* packed, const DecodeGeom& geo, const Seg* segs,
                           unsigned long long* seed, const unsigned long long* prefix_rel, const double* centers,
                           const void* exact, const void* base, void* out, nmk_segment_info* info,
                           nmk_decode_err* err, unsigned long long* status, unsigned* ticket, cudaStream_t s) {
  switch (bits) {
#define NMK_DEC_CASE(BB) \
  case BB: launch_decode<T, BB>(packed, geo, segs, seed, prefix_rel, centers, exact, base, out, info, err, status, ticket, s); break;
    NMK_DEC_CASE(2) NMK_DEC_CASE(3) NMK_DEC_CASE(4) NMK_DEC_CASE(5) NMK_DEC_CASE(6) NMK_DEC_CASE(7)
    NMK_DEC_CASE(8) NMK_DEC_CASE(9) NMK_DEC_CASE(10) NMK_DEC_CASE(11) NMK_DEC_CASE(12) NMK_DEC_CASE(13)
    NMK_DEC_CASE(14) NMK_DEC_CASE(15) NMK_DEC_CASE(16) NMK_DEC_CASE(17) NMK_DEC_CASE(18) NMK_DEC_CASE(19)
    NMK_DEC_CASE(20) NMK_DEC_CASE(21) NMK_DEC_CASE(22) NMK_DEC_CASE(23) NMK_DEC_CASE(24) NMK_DEC_CASE(25)
    NMK_DEC_CASE(26) NMK_DEC_CASE(27) NMK_DEC_CASE(28) NMK_DEC_CASE(29) NMK_DEC_CASE(30)
#undef NMK_DEC_CASE
    default: return set_error(NMK_ERR_ARG, "nmk_decode: bits %d outside [2, 30]", bits);
  }
  return check_launch("k_decode");
}

}  // namespace nmk

using namespace nmk;

extern "C" size_t nmk_decode_ws_bytes(const uint64_t* h_seg_start, const uint64_t* h_seg_count, int nseg,
                                      uint64_t epb) {
  if (nseg < 0 || epb == 0) return 0;
  return decode_plan(h_seg_start, h_seg_count, nseg, epb).total;
}

extern "C" int nmk_decode(const uint8_t* packed, uint64_t block_stride, uint64_t first_block, int bits,
                          uint64_t epb, uint64_t n_total, const unsigned long long* prefix_rel,
                          const double* centers, int k, const void* exact, uint64_t n_exact, const void* base,
                          void* out, int dtype, const uint64_t* h_seg_start, const uint64_t* h_seg_count,
                          const uint64_t* h_seg_out, int nseg, nmk_segment_info* seg_info,
                          nmk_decode_err* err, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (nseg < 1 || !h_seg_start || !h_seg_count || !h_seg_out || !seg_info || !err || !ws)
    return set_error(NMK_ERR_ARG, "nmk_decode: bad argument");
  if (bits < 2 || bits > 30 || epb == 0 || k < 1) return set_error(NMK_ERR_ARG, "nmk_decode: bad geometry");
  if (block_stride % 16 || ((uintptr_t)packed & 15)) return set_error(NMK_ERR_ARG, "nmk_decode: packed alignment");
  DecodePlan p = decode_plan(h_seg_start, h_seg_count, nseg, epb);
  if (ws_bytes < p.total) return set_error(NMK_ERR_ARG, "nmk_decode: workspace too small");
  const uint64_t tpb = (epb + kTile - 1) / kTile;
  // host-side segment table (only non-empty segments get tiles)
  Seg* hs = (Seg*)malloc(sizeof(Seg) * (size_t)nseg);
  int ns = 0;
  uint64_t tile0 = 0;
  for (int i = 0; i < nseg; ++i) {
    uint64_t st = h_seg_start[i], ct = h_seg_count[i];
    if (st + ct > n_total) { free(hs); return set_error(NMK_ERR_ARG, "nmk_decode: segment out of range"); }
    if (ct == 0) continue;
    if (st / epb < first_block) { free(hs); return set_error(NMK_ERR_ARG, "nmk_decode: segment before first block"); }
    Seg sg;
    sg.start = st; sg.count = ct; sg.out = h_seg_out[i];
    sg.gfirst = seg_first_tile(st, epb, tpb);
    sg.tile0 = tile0;
    tile0 += seg_first_tile(st + ct - 1, epb, tpb) - sg.gfirst + 1;
    hs[ns++] = sg;
  }
  cudaMemsetAsync(seg_info, 0, sizeof(nmk_segment_info) * (size_t)nseg, s);
  cudaMemsetAsync(err, 0, sizeof(nmk_decode_err), s);
  if (ns == 0) { free(hs); return check_launch("nmk_decode(empty)"); }
  if (!packed || !centers || !base || !out || !prefix_rel) { free(hs); return set_error(NMK_ERR_ARG, "nmk_decode: null pointer"); }
  if (ns != nseg) {  // empty segments are skipped: info indices follow non-empty order
    free(hs);
    return set_error(NMK_ERR_ARG, "nmk_decode: empty segments must be filtered by the caller");
  }
  char* w = (char*)ws;
  unsigned* ticket = (unsigned*)w;
  unsigned long long* status = (unsigned long long*)(w + p.off_status);
  Seg* dsegs = (Seg*)(w + p.off_segs);
  unsigned long long* seed = (unsigned long long*)(w + p.off_seed);
  cudaMemsetAsync(w, 0, p.off_segs, s);
  cudaMemcpyAsync(dsegs, hs, sizeof(Seg) * (size_t)ns, cudaMemcpyHostToDevice, s);
  // a pageable H2D cudaMemcpyAsync returns after staging the source, so the
  // host table can be released immediately (no stream synchronisation)
  free(hs);
  DecodeGeom geo{epb, tpb, n_total, first_block, block_stride, n_exact, p.total_tiles, ns, k};
  if (dtype == NMK_F64)
    return dispatch_decode<double>(bits, packed, geo, dsegs, seed, prefix_rel, centers, exact, base, out, seg_info, err,
                                   status, ticket, s);
  if (dtype == NMK_F32)
    return dispatch_decode<float>(bits, packed, geo, dsegs, seed, prefix_rel, centers, exact, base, out, seg_info, err,
                                  status, ticket, s);
  return set_error(NMK_ERR_ARG, "nmk_decode: bad dtype");
}
