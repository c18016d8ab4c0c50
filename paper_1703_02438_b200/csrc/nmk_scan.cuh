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
// ---- decoupled look-back over tile-status words (k_scan.cu, k_encode.cu) ----
constexpr unsigned long long kFlagAgg = 1ULL << 62;    // tile aggregate published
constexpr unsigned long long kFlagPre = 2ULL << 62;    // inclusive prefix published
constexpr unsigned long long kValMask = (1ULL << 62) - 1;

__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_status(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// One whole warp of tile `tile` (tiles take CTAs in blockIdx order; status
// words zero at kernel start): publishes the tile aggregate, sums its
// predecessors' (flag, value) words back to the nearest inclusive prefix,
// publishes its own inclusive prefix and returns the exclusive one.
__device__ __forceinline__ unsigned long long scan_lookback(unsigned long long* status, uint64_t tile,
                                                            unsigned long long agg, int lane) {
  unsigned long long prefix = 0;
  if (tile == 0) {
    if (lane == 0) st_status(status, kFlagPre | agg);
    return 0ULL;
  }
  if (lane == 0) st_status(status + tile, kFlagAgg | agg);
  int64_t base = (int64_t)tile - 1;
  while (true) {   // lane j inspects tile - 1 - j - 32 r
    const int64_t t = base - lane;
    unsigned long long s = t >= 0 ? ld_status(status + t) : kFlagPre;   // before tile 0: prefix 0
    // wait until every inspected predecessor has published something
    while (__any_sync(0xffffffffu, s == 0)) {
      if (s == 0) s = ld_status(status + t);
    }
    const unsigned pre = __ballot_sync(0xffffffffu, (s & kFlagPre) != 0);
    const int stop = pre ? __ffs(pre) - 1 : 32;   // first (nearest) inclusive prefix
    unsigned long long part = (lane <= stop && t >= 0) ? (s & kValMask) : 0ULL;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    prefix += part;
    if (pre) break;
    base -= 32;
  }
  if (lane == 0) st_status(status + tile, kFlagPre | (prefix + agg));
  return prefix;
}

__device__ __forceinline__ void zero_list_run(const ZeroList& z) {
  if (blockIdx.x != 0) return;
#pragma unroll
  for (int k = 0; k < 3; ++k)
    for (uint32_t i = threadIdx.x; i < z.n[k]; i += blockDim.x) z.p[k][i] = 0ULL;
}
#endif
}  // namespace nmk
