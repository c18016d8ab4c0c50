// nmk_block.cuh — CTA-wide reduce and exclusive sum (warp shuffles + one
// shared-memory step), used by K3 (k_select.cu) and the run-length kernels of
// the sparse histogram (k_hist.cu).  `scratch` is caller-provided shared
// memory; a __syncthreads() must separate two uses of the same scratch.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace nmk {

template <typename T>
__device__ __forceinline__ T shfl_down_any(const T& v, int o) {
  static_assert(sizeof(T) % 4 == 0, "whole 32-bit words");
  T r;
  const uint32_t* p = reinterpret_cast<const uint32_t*>(&v);
  uint32_t* q = reinterpret_cast<uint32_t*>(&r);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(T) / 4); ++i) q[i] = __shfl_down_sync(0xffffffffu, p[i], o);
  return r;
}

// op-reduction over the CTA's threads in thread order; the result is valid in
// thread 0 only.  scratch: T[THREADS / 32].
template <int THREADS, typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, Op op, T* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = shfl_down_any(v, o);
    if (lane + o < 32) v = op(v, y);
  }
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int w = 1; w < THREADS / 32; ++w) v = op(v, scratch[w]);
  }
  return v;
}

struct SumOp {
  template <typename T>
  __device__ __forceinline__ T operator()(const T& a, const T& b) const { return a + b; }
};

// exclusive prefix sum of one unsigned per thread (thread order) and the CTA
// total, both valid in every thread (THREADS <= 1024).  scratch: unsigned[THREADS / 32].
template <int THREADS>
__device__ __forceinline__ unsigned block_exclusive_sum(unsigned v, unsigned& total, unsigned* scratch) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) scratch[wid] = incl;
  __syncthreads();
  // every warp scans the warp totals itself (no second barrier)
  constexpr int NW = THREADS / 32;
  const unsigned x = lane < NW ? scratch[lane] : 0u;
  unsigned xi = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xffffffffu, xi, o);
    if (lane >= o) xi += y;
  }
  const unsigned base = __shfl_sync(0xffffffffu, xi - x, wid), tot = __shfl_sync(0xffffffffu, xi, NW - 1);
  total = tot;
  return base + incl - v;
}

}  // namespace nmk
