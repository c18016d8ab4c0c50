// nmk_scan.cuh — host launcher of the chunk-count scan (k_scan.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace nmk {
// offsets[i] = sum(counts[0..i)) for i = 0..n (offsets holds n + 1 entries;
// offsets[n] is the total).
size_t chunk_scan_ws_bytes(uint64_t n);
void chunk_scan(const uint32_t* counts, uint64_t n, unsigned long long* offsets, void* ws, cudaStream_t s);
}  // namespace nmk
