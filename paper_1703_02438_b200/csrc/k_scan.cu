// k_scan.cu — exclusive scan of per-chunk u32 counts into u64 offsets.
//
// Used by K4 (incompressible counts per 256-element chunk -> positions in the
// compacted exact-value list and the per-block prefix table, pipeline.py:257-
// 276) and by K5 (sentinel counts per chunk -> rank of every sentinel in the
// exact list, codec.py:231-236).  One single-pass decoupled look-back scan
// (CUB) over n + 1 items, the last one reading as 0, so offsets[n] is the
// total: 4 bytes read and 8 written per 256 elements, no second pass.
#include <cub/device/device_scan.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include "nmk_common.cuh"
#include "nmk_scan.cuh"

namespace nmk {

struct CountAt {
  const uint32_t* counts;
  uint64_t n;
  __host__ __device__ unsigned long long operator()(uint64_t i) const {
    return i < n ? (unsigned long long)counts[i] : 0ULL;
  }
};

using CountIter = thrust::transform_iterator<CountAt, thrust::counting_iterator<uint64_t>>;

static size_t scan_temp_bytes(uint64_t n) {
  size_t bytes = 0;
  CountIter it(thrust::counting_iterator<uint64_t>(0), CountAt{nullptr, n});
  cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, (unsigned long long*)nullptr, (int64_t)(n + 1));
  return bytes;
}

size_t chunk_scan_ws_bytes(uint64_t n) { return scan_temp_bytes(n) + 256; }

void chunk_scan(const uint32_t* counts, uint64_t n, unsigned long long* offsets, void* ws, cudaStream_t s) {
  if (n == 0) {
    cudaMemsetAsync(offsets, 0, sizeof(unsigned long long), s);
    return;
  }
  size_t bytes = scan_temp_bytes(n);
  CountIter it(thrust::counting_iterator<uint64_t>(0), CountAt{counts, n});
  cub::DeviceScan::ExclusiveSum(ws, bytes, it, offsets, (int64_t)(n + 1), s);
}

}  // namespace nmk
