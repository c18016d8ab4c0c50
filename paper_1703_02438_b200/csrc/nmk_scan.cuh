// nmk_scan.cuh — host launcher of the chunk-count scan (k_scan.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace nmk {
// offsets[i] = sum(counts[0..i)) for i = 0..n (offsets holds n + 1 entries;
// offsets[n] is the total).
size_t chunk_scan_ws_bytes(uint64_t n);
// tile-status words at the front of the scan workspace; they must be zero when
// the scan starts: either chunk_scan's memset node, or (status_zeroed) the
// kernel in front of it on the stream ran zero_list_run over them
uint32_t chunk_scan_tiles(uint64_t n);
void chunk_scan(const uint32_t* counts, uint64_t n, unsigned long long* offsets, void* ws, cudaStream_t s,
                bool status_zeroed = false);

// Small device buffers (8-byte words) a kernel zeroes for its successors on the
// stream instead of memset nodes between the chained launches.
struct ZeroList {
  unsigned long long* p[3];
  uint32_t n[3];
};
#ifdef __CUDACC__
__device__ __forceinline__ void zero_list_run(const ZeroList& z) {
  if (blockIdx.x != 0) return;
#pragma unroll
  for (int k = 0; k < 3; ++k)
    for (uint32_t i = threadIdx.x; i < z.n[k]; i += blockDim.x) z.p[k][i] = 0ULL;
}
#endif
}  // namespace nmk
