// k_scan.cu — exclusive scan of per-chunk u32 counts into u64 offsets.
//
// Used by K4 (incompressible counts per 256-element chunk -> positions in the
// compacted exact-value list and the per-block prefix table, pipeline.py:257-
// 276) and by K5 (sentinel counts per chunk -> rank of every sentinel in the
// exact list, codec.py:231-236).  Three small launches over 4 bytes per 256
// elements: per-CTA sums, one-CTA scan of the sums, per-CTA rescan.
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "nmk_common.cuh"
#include "nmk_scan.cuh"

namespace nmk {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;

__global__ void __launch_bounds__(kScanThreads)
k_scan_reduce(const uint32_t* __restrict__ counts, uint64_t n, unsigned long long* __restrict__ partial) {
  typedef cub::BlockReduce<unsigned long long, kScanThreads> BR;
  __shared__ typename BR::TempStorage tmp;
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  unsigned long long s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    uint64_t j = base + (uint64_t)i * kScanThreads + threadIdx.x;
    if (j < n) s += counts[j];
  }
  unsigned long long t = BR(tmp).Sum(s);
  if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

__global__ void __launch_bounds__(1024)
k_scan_top(unsigned long long* __restrict__ partial, uint64_t np, unsigned long long* __restrict__ total) {
  typedef cub::BlockScan<unsigned long long, 1024> BS;
  __shared__ typename BS::TempStorage tmp;
  unsigned long long run = 0;
  for (uint64_t c0 = 0; c0 < np; c0 += 1024) {
    uint64_t j = c0 + threadIdx.x;
    unsigned long long v = j < np ? partial[j] : 0ULL, ex, agg;
    BS(tmp).ExclusiveSum(v, ex, agg);
    __syncthreads();
    if (j < np) partial[j] = run + ex;
    run += agg;
  }
  if (threadIdx.x == 0 && total) *total = run;
}

__global__ void __launch_bounds__(kScanThreads)
k_scan_apply(const uint32_t* __restrict__ counts, uint64_t n, const unsigned long long* __restrict__ partial,
             unsigned long long* __restrict__ offsets) {
  typedef cub::BlockScan<unsigned long long, kScanThreads> BS;
  __shared__ typename BS::TempStorage tmp;
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  unsigned long long v[kScanItems], s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = (base + i < n) ? counts[base + i] : 0u;
    s += v[i];
  }
  unsigned long long ex;
  BS(tmp).ExclusiveSum(s, ex);
  unsigned long long run = partial[blockIdx.x] + ex;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < n) offsets[base + i] = run;
    run += v[i];
  }
}

size_t chunk_scan_ws_bytes(uint64_t n) { return ((n + kScanTile - 1) / kScanTile + 1) * 8 + 256; }

void chunk_scan(const uint32_t* counts, uint64_t n, unsigned long long* offsets, unsigned long long* total,
                void* ws, cudaStream_t s) {
  if (n == 0) return;
  const uint64_t np = (n + kScanTile - 1) / kScanTile;
  unsigned long long* partial = (unsigned long long*)ws;
  k_scan_reduce<<<(unsigned)np, kScanThreads, 0, s>>>(counts, n, partial);
  k_scan_top<<<1, 1024, 0, s>>>(partial, np, total);
  k_scan_apply<<<(unsigned)np, kScanThreads, 0, s>>>(counts, n, partial, offsets);
}

}  // namespace nmk
