// nmk_common.cuh — shared device helpers for the NUMARCK sm_100a kernels.
//
// Exactness rules (restating pkg/src/nmk/core.py:115-137,
// binning.py:50-51,113,287-301, pipeline.py:143-160, core.py:202-205):
//  * every fp64 op is an explicit round-to-nearest intrinsic (__dadd_rn,
//    __dsub_rn, __dmul_rn, __ddiv_rn) so no FMA contraction can change a bit;
//    the library is additionally built with -fmad=false;
//  * f64 -> f32 narrowing is __double2float_rn (IEEE, denormals kept: -ftz=false).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/nmk_b200.h"

namespace nmk {

constexpr int kTileThreads = 256;             // threads per encode/decode CTA
constexpr int kGroup = 8;                     // elements per thread (B bytes out)
constexpr int kTile = kTileThreads * kGroup;  // elements per tile (2048)

// ---- element types --------------------------------------------------------
template <typename T> struct Bits;
template <> struct Bits<float>  { using U = uint32_t; };
template <> struct Bits<double> { using U = unsigned long long; };

__device__ __forceinline__ double to_f64(float v) { return (double)v; }
__device__ __forceinline__ double to_f64(double v) { return v; }

template <typename T> __device__ __forceinline__ T narrow(double v);
template <> __device__ __forceinline__ float narrow<float>(double v) { return __double2float_rn(v); }
template <> __device__ __forceinline__ double narrow<double>(double v) { return v; }

__device__ __forceinline__ bool finite64(double v) {
  // exponent field not all-ones
  return (__double_as_longlong(v) & 0x7ff0000000000000ULL) != 0x7ff0000000000000ULL;
}

// ---- Eq. 1 with the zero / non-finite rules (core.py:115-137) --------------
// r = RN(RN(x - b) / b); valid = finite(r) & finite(b) & finite(x);
// b == 0 && x == 0 -> r = +0, valid; invalid -> r = +0.
__device__ __forceinline__ double change_ratio(double b, double x, bool& valid) {
  double r = __ddiv_rn(__dsub_rn(x, b), b);
  bool ok = finite64(r) && finite64(b) && finite64(x);
  if (b == 0.0 && x == 0.0) { r = 0.0; ok = true; }
  valid = ok;
  return ok ? r : 0.0;
}

// floor(RN(RN(r - origin) / width)), canonicalised so -0.0 -> +0.0
// (binning.py:113; np.unique merges the two zeros).
__device__ __forceinline__ double bin_ordinal(double r, double origin, double width) {
  double q = floor(__ddiv_rn(__dsub_rn(r, origin), width));
  return __dadd_rn(q, 0.0);
}

// origin + (q + 0.5) * width, add -> mul -> add (binning.py:50-51).
__device__ __forceinline__ double bin_center(double q, double origin, double width) {
  return __dadd_rn(origin, __dmul_rn(__dadd_rn(q, 0.5), width));
}

// Decoder arithmetic: T((1 + c) * f64(b)) (core.py:202-205, pipeline.py:158).
template <typename T>
__device__ __forceinline__ T apply_center(double c, double b) {
  return narrow<T>(__dmul_rn(__dadd_rn(1.0, c), b));
}

// Round-trip filter: |f64(T((1+c)*b)) - x| <= E*|b| (pipeline.py:143-160).
template <typename T>
__device__ __forceinline__ bool roundtrip_ok(double c, double b, double x, double tol) {
  double rec = to_f64(apply_center<T>(c, b));
  return fabs(__dsub_rn(rec, x)) <= __dmul_rn(tol, fabs(b));
}

// #cuts strictly below r == np.searchsorted(cuts, r, 'left') (binning.py:300).
__device__ __forceinline__ uint32_t lower_bound_cuts(const double* cuts, int ncuts, double r) {
  int lo = 0, hi = ncuts;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (cuts[mid] < r) lo = mid + 1; else hi = mid;
  }
  return (uint32_t)lo;
}

// ---- relaxed 64-bit status words for decoupled look-back ------------------
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// status word: [63:62] flag (0 none, 1 aggregate, 2 inclusive), [61:0] value
constexpr unsigned long long kFlagAgg = 1ULL << 62;
constexpr unsigned long long kFlagInc = 2ULL << 62;
constexpr unsigned long long kValMask = (1ULL << 62) - 1;

// Warp-0 decoupled look-back: returns the exclusive prefix of `tile`
// (tiles < tile_first are not consulted; tile_first seeds its own INCL).
// Must be called by all 32 lanes of one warp.
__device__ __forceinline__ unsigned long long lookback(const unsigned long long* status,
                                                       long long tile, long long tile_first) {
  const int lane = threadIdx.x & 31;
  unsigned long long excl = 0;
  long long base = tile - 1;
  while (base >= tile_first) {
    long long t = base - lane;
    unsigned long long s = kFlagInc;  // lanes before tile_first act as INCL 0
    if (t >= tile_first) {
      do { s = ld_relaxed(status + t); } while ((s >> 62) == 0);
    }
    unsigned inc_mask = __ballot_sync(0xffffffffu, (s >> 62) == 2);
    unsigned long long v = (s & kValMask);
    int stop = inc_mask ? (__ffs(inc_mask) - 1) : 32;  // nearest inclusive lane
    if (lane > stop) v = 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += v;
    if (inc_mask) break;
    base -= 32;
  }
  return excl;
}

}  // namespace nmk

// ---- host-side error plumbing (defined in abi.cu) --------------------------
namespace nmk {
int set_error(int code, const char* fmt, ...);
int check_launch(const char* what);
}  // namespace nmk
