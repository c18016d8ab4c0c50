// k_scan.cu — exclusive scan of per-chunk u32 counts into u64 offsets.
//
// Used by K4 (incompressible counts per 256-element chunk -> positions in the
// compacted exact-value list and the per-block prefix table, pipeline.py:257-
// 276) and by K5 (sentinel counts per chunk -> rank of every sentinel in the
// exact list, codec.py:231-236).  One single-pass decoupled look-back scan
// over n + 1 items (the last one reads as 0, so offsets[n] is the total):
// 4 bytes read and 8 written per 256 elements.  Tiles of 8192 items go to
// CTAs in blockIdx order; each CTA publishes its tile aggregate, then looks
// back over its predecessors' (flag, value) words until it meets an
// inclusive prefix.  The tile-status words are zeroed in front of the kernel
// (by the counting kernel that precedes it on the stream, or a memset node),
// so no state survives between launches.
#include "nmk_common.cuh"
#include "nmk_scan.cuh"

namespace nmk {

constexpr int kScanThreads = 256;
#ifndef NMK_SCAN_ROUNDS
#define NMK_SCAN_ROUNDS 8   // A/B: 2 and 4 (more, smaller tiles) no faster on cfg2
#endif
constexpr int kScanRounds = NMK_SCAN_ROUNDS;                      // uint4 per lane
constexpr int kScanWarpItems = 32 * 4 * kScanRounds;              // 1024 contiguous counts per warp
constexpr int kScanTile = (kScanThreads / 32) * kScanWarpItems;   // 8192 per CTA (few tiles: short look-back)
// Each warp owns 1024 contiguous items; in round q lane l holds items
// w0 + 128 q + 4 l .. + 3 (coalesced 512-byte loads, 1 KB stores).
__global__ void __launch_bounds__(kScanThreads)
k_chunk_scan(const uint32_t* __restrict__ counts, uint64_t n, unsigned long long* __restrict__ offsets,
             unsigned long long* __restrict__ status) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  pdl_enter();
  const uint64_t tile = blockIdx.x;
  const uint64_t w0 = tile * kScanTile + (uint64_t)wid * kScanWarpItems;
  const bool vec = ((reinterpret_cast<uintptr_t>(counts) & 15) == 0);
  uint4 v[kScanRounds];
  uint32_t ex[kScanRounds];        // lane's exclusive offset inside the round
  unsigned long long wsum = 0;     // warp running total (uniform)
  unsigned long long rbase[kScanRounds];
#pragma unroll
  for (int q = 0; q < kScanRounds; ++q) {
    const uint64_t i = w0 + (uint64_t)q * 128 + (uint64_t)lane * 4;
    if (vec && i + 4 <= n) {
      v[q] = __ldcs(reinterpret_cast<const uint4*>(counts + i));
    } else {   // item n (and beyond) reads 0
      v[q].x = i < n ? counts[i] : 0u;
      v[q].y = i + 1 < n ? counts[i + 1] : 0u;
      v[q].z = i + 2 < n ? counts[i + 2] : 0u;
      v[q].w = i + 3 < n ? counts[i + 3] : 0u;
    }
  }
#pragma unroll
  for (int q = 0; q < kScanRounds; ++q) {
    const uint32_t sq = v[q].x + v[q].y + v[q].z + v[q].w;   // < 2^32: counts are <= 256 each
    uint32_t incl = sq;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    ex[q] = incl - sq;
    rbase[q] = wsum;
    wsum += __shfl_sync(0xffffffffu, incl, 31);
  }
  __shared__ unsigned long long s_warp[kScanThreads / 32];
  __shared__ unsigned long long s_prefix;
  if (lane == 0) s_warp[wid] = wsum;
  __syncthreads();
  unsigned long long wbase = 0, agg = 0;
#pragma unroll
  for (int w = 0; w < kScanThreads / 32; ++w) {
    const unsigned long long x = s_warp[w];
    wbase += w < wid ? x : 0ULL;
    agg += x;
  }
  if (wid == 0) {   // look-back (nmk_scan.cuh)
    const unsigned long long prefix = scan_lookback(status, tile, agg, lane);
    if (lane == 0) s_prefix = prefix;
  }
  __syncthreads();
  const unsigned long long wstart = s_prefix + wbase;
#pragma unroll
  for (int q = 0; q < kScanRounds; ++q) {
    const uint64_t i = w0 + (uint64_t)q * 128 + (uint64_t)lane * 4;
    const unsigned long long o0 = wstart + rbase[q] + ex[q];
    const unsigned long long o1 = o0 + v[q].x, o2 = o1 + v[q].y, o3 = o2 + v[q].z;
    if (i + 4 <= n + 1) {   // offsets holds n + 1 entries
      if ((i & 1) == 0) {
        reinterpret_cast<ulonglong2*>(offsets + i)[0] = make_ulonglong2(o0, o1);
        reinterpret_cast<ulonglong2*>(offsets + i)[1] = make_ulonglong2(o2, o3);
      } else {
        offsets[i] = o0; offsets[i + 1] = o1; offsets[i + 2] = o2; offsets[i + 3] = o3;
      }
    } else {
      if (i <= n) offsets[i] = o0;
      if (i + 1 <= n) offsets[i + 1] = o1;
      if (i + 2 <= n) offsets[i + 2] = o2;
    }
  }
}

size_t chunk_scan_ws_bytes(uint64_t n) { return ((n + 1 + kScanTile - 1) / kScanTile) * 8 + 256; }

uint32_t chunk_scan_tiles(uint64_t n) { return (uint32_t)((n + 1 + kScanTile - 1) / kScanTile); }

void chunk_scan(const uint32_t* counts, uint64_t n, unsigned long long* offsets, void* ws, cudaStream_t s,
                bool status_zeroed) {
  const uint64_t ntiles = chunk_scan_tiles(n);
  unsigned long long* status = reinterpret_cast<unsigned long long*>(ws);
  if (!status_zeroed) cudaMemsetAsync(status, 0, ntiles * 8, s);
  launch_chain(kPdlScan, k_chunk_scan, (unsigned)ntiles, kScanThreads, 0, s, counts, n, offsets, status);
}

}  // namespace nmk
