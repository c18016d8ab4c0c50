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

constexpr int kGroup = 8;   // consecutive elements per lane: 8 codes = B whole bytes

// ---- element types --------------------------------------------------------
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

// ---- division-free fast path with a rigorous error bound -------------------
// ra approximates r = RN((x - b) / b) through a reciprocal seed refined by two
// Newton steps (relative error <= 2^-50 even from a 2^-13 seed), so
//     |ra - r| <= ea = |ra| * 2^-44        (a >= 16x safety margin).
// Callers decide from ra whenever every decision threshold is farther than
// the bound and fall back to the IEEE path otherwise, so results stay
// bit-identical.  Applies to normal b in [2^-900, 2^900] with a finite,
// non-tiny quotient; returns false otherwise (IEEE path, incl. all invalid).
__device__ __forceinline__ double rcp_approx(double b) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(b));
  return y;
}

__device__ __forceinline__ bool fast_ratio(double b, double x, double& ra, double& ea) {
  const int eb = (__double2hiint(b) >> 20) & 0x7ff;
  const double d = __dsub_rn(x, b);
  if (eb < 1023 - 900 || eb > 1023 + 900) return false;
  double y = rcp_approx(b);
  double e = __fma_rn(-b, y, 1.0);
  y = __fma_rn(y, e, y);
  e = __fma_rn(-b, y, 1.0);
  y = __fma_rn(y, e, y);
  ra = __dmul_rn(d, y);
  const double a = fabs(ra);
  ea = a * 0x1p-44;
  // finite, and either exactly zero or far from the subnormal range
  return (a <= 0x1p+900) && (a >= 0x1p-900 || ra == 0.0);
}

// Bin ordinal of the element's ratio (binning.py:113) or false if invalid.
// Fast path: t = (ra - origin) * inv_w is within et of RN(RN(r - origin)/w);
// floor(t) is the exact ordinal unless an integer lies within et of t.
__device__ __forceinline__ bool element_ordinal(double b, double x, double origin, double width, double inv_w,
                                                double& q) {
  double ra, ea;
  if (fast_ratio(b, x, ra, ea)) {
    const double s = __dsub_rn(ra, origin);
    const double t = __dmul_rn(s, inv_w);
    const double et = __dadd_rn(__dmul_rn(__dadd_rn(ea, fabs(s) * 0x1p-48), inv_w * 1.0000001),
                                fabs(t) * 0x1p-46);
    const double fl = floor(t);
    if (t < 0x1p+50 && __dsub_rn(t, fl) > et && __dsub_rn(__dadd_rn(fl, 1.0), t) > et) {
      q = __dadd_rn(fl, 0.0);
      return true;
    }
  }
  bool valid;
  const double r = change_ratio(b, x, valid);
  if (!valid) return false;
  q = bin_ordinal(r, origin, width);
  return true;
}

// ---- f32 ratio keys (K1 -> K2) -----------------------------------------------
// K1 stores, per element, key = RN_f32(r) (from ra or the exact r) so the
// histogram pass reads 4 bytes instead of both snapshots.  |key - r| <=
// |key| * 2^-23 whenever key is a normal float in [2^-100, 2^100] or exactly
// zero; other magnitudes are stored as +inf ("use the exact path"), invalid
// elements as NaN.
__device__ __forceinline__ float ratio_key(double r) {
  const double a = fabs(r);
  if (r == 0.0) return (float)r;
  if (a < 0x1p-100 || a > 0x1p+100) return __int_as_float(0x7f800000);
  return __double2float_rn(r);
}

// Safe range for a finite key (K4 keyed mode, k_encode.cuh): |b| in
// [2^-900, 2^901) and |x| < 2^901 for f64 inputs, [2^-100, 2^101) and
// < 2^101 for f32, so the decoder's product (1 + c) b neither overflows nor
// loses relative accuracy to subnormal rounding.
template <typename T>
__device__ __forceinline__ bool key_safe(double b, double x) {
  constexpr int lo = sizeof(T) == 4 ? 1023 - 100 : 1023 - 900;
  constexpr int hi = sizeof(T) == 4 ? 1023 + 100 : 1023 + 900;
  const int eb = (__double2hiint(b) >> 20) & 0x7ff, ex = (__double2hiint(x) >> 20) & 0x7ff;
  return eb >= lo && eb <= hi && ex <= hi;
}

// One bound for a whole launch: the per-element bound of key_ordinal is
// monotone in |key|, |s| and |t|, all of which are bounded by the global
// (gmin, gmax), so et_c below dominates it for every valid element.
__device__ __forceinline__ double key_bound(double gmin, double gmax, double inv_w) {
  const double amax = fmax(fabs(gmin), fabs(gmax)) * (1.0 + 0x1p-20);
  const double smax = (gmax - gmin) * (1.0 + 0x1p-20) + amax * 0x1p-20;
  const double tmax = smax * inv_w * (1.0 + 0x1p-20) + 1.0;
  return (amax * 0x1p-22 + smax * 0x1p-48) * inv_w * 1.0000001 + tmax * 0x1p-46;
}

__device__ __forceinline__ bool key_ordinal_c(float key, double origin, double inv_w, double et_c, double& q) {
  const double t = __dmul_rn(__dsub_rn((double)key, origin), inv_w);
  const double fl = floor(t);
  const double fr = __dsub_rn(t, fl);
  if (t < 0x1p+50 && fr > et_c && fr < 1.0 - et_c) {
    q = __dadd_rn(fl, 0.0);
    return true;
  }
  return false;
}

// ---- all-f32 ordinal from a key (the K2 common case) -------------------------
// th = RN32(key * iw32 + c32) (one FMA) with iw32 = RN32(1/w) and
// c32 = RN32(-gmin/w - 0.5) estimates u - 1/2, u = (r - gmin)/w.  With
// A >= |key|, |gmin|; T >= |u| + 1 (every valid r lies in [gmin, gmax]):
//   |th - (u - 1/2)| <= |key - r| iw + |key| |iw32 - 1/w| + |c32 - c| + |th| 2^-24
//                    <= A iw (2^-23 + 2^-24) + (|gmin| iw + 1/2) 2^-24 + T 2^-24
// and the f64 reference t* = RN(RN(r - gmin)/w) is within T 2^-50 of u; e
// below is the sum, x1.05.  fl = RN_int(th) comes from the 1.5*2^23 magic
// add (exact for |th| < 2^22) and d = th - fl is exact, so |d| < 1/2 - e
// proves floor(t*) = fl.  The ordinal is the integer in m's mantissa.  NaN
// keys (invalid) and +inf keys (exact path) fail the test; when the bound
// is too loose the grid is switched off (hi < 0: every key fails).
struct KeyGrid32 {
  float iw32, c32, hi;
  uint32_t nbins;
};

__device__ __forceinline__ KeyGrid32 key_grid32(double gmin, double gmax, double inv_w, uint32_t nbins) {
  KeyGrid32 g;
  const double A = fmax(fabs(gmin), fabs(gmax)) * (1.0 + 0x1p-20);
  const double T = (gmax - gmin) * inv_w * (1.0 + 0x1p-20) + 2.0;
  const double G = fabs(gmin) * inv_w;
  const double e = (A * inv_w * (0x1p-23 + 0x1p-24) + (G + 0.5) * (0x1p-24 + 0x1p-48) + T * (0x1p-24 + 0x1p-50) +
                    0x1p-40) * 1.05;
  const bool on = e < 0.05 && T < 0x1p+21 && G < 0x1p+21 && A < 0x1p+100 && inv_w < 0x1p+100;
  g.iw32 = __double2float_rn(inv_w);
  g.c32 = __double2float_rn(-gmin * inv_w - 0.5);
  g.hi = on ? __double2float_rz(0.5 - e) : -1.0f;
  g.nbins = nbins;
  return g;
}

// true (and qi = the exact ordinal, < nbins) when the f32 arithmetic decides
// (nbins must be the dense span of the same gmin, gmax, width)
__device__ __forceinline__ bool key_ordinal32(float key, const KeyGrid32& g, uint32_t& qi) {
  constexpr float kMagic = 12582912.0f;   // 1.5 * 2^23
  const float th = __fmaf_rn(key, g.iw32, g.c32);
  const float m = __fadd_rn(th, kMagic);
  const float d = __fsub_rn(th, __fsub_rn(m, kMagic));
  qi = (uint32_t)(__float_as_int(m) - 0x4B400000);
  // decided => qi = floor(t*) <= floor(RN((gmax - gmin)/w)) = nbins - 1
  return fabsf(d) < g.hi;
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

// ---- O(1) nearest-center search -------------------------------------------
// A uniform grid of kLutCells cells over [cuts[0], cuts[ncuts-1]] stores, per
// cell, #cuts below the cell's left edge.  The cell of r gives a candidate i;
// exact compares against cuts i-1, i, i+1 settle #cuts < r (k_encode.cu), with
// an exact walk when the cell edge rounding or a crowded cell defeats it, so
// the grid only makes the search O(1), never inexact.
constexpr int kLutCells = 8192;

// Build the grid over `ncuts` cuts already in shared memory (all threads).
__device__ __forceinline__ void build_cut_lut(const double* cuts, int ncuts, uint16_t* lut, double& lo,
                                              double& scale, bool& use) {
  use = false;
  lo = 0.0;
  scale = 0.0;
  if (ncuts >= 2 && ncuts < 65535) {
    double a = cuts[0], z = cuts[ncuts - 1];
    double sc = (double)kLutCells / (z - a);
    if (z > a && finite64(a) && finite64(z) && finite64(sc) && sc > 0.0) {
      use = true;
      lo = a;
      scale = sc;
      for (int g = threadIdx.x; g < kLutCells; g += blockDim.x) {
        double edge = a + (double)g / sc;
        lut[g] = (uint16_t)lower_bound_cuts(cuts, ncuts, edge);
      }
    }
  }
}

// ---- TMA bulk copies + mbarriers (sm_90+/sm_100a) --------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// arrive once and expect `bytes` of async-proxy transactions on the phase
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// 1-D TMA: global -> shared, completion counted on `bar` (16-byte aligned,
// size a multiple of 16)
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// order this thread's (and, after __syncwarp, its warp's) generic shared
// accesses before subsequent async-proxy writes to the same buffer
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- programmatic dependent launch (sm_90+) -------------------------------
// The sync-free step is a fixed chain of kernels on one stream.  Launched with
// the programmatic-stream-serialization attribute (launch_chain below), a
// kernel's CTAs may become resident while the previous kernel drains; every
// chained kernel therefore runs pdl_enter() before its first global access:
// griddepcontrol.wait returns when the previous grid has completed and its
// writes are visible, then launch_dependents lets the next kernel in.  Both
// are no-ops for a plain launch.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---- division by a run-time invariant (Granlund-Montgomery) ---------------
// q = n / d for any 32-bit n with one mul-hi, an add and two shifts.
struct FastDiv {
  uint32_t d, m;
  int s1, s2;
  void init(uint32_t dd) {
    d = dd;
    int l = 0;
    while ((1ull << l) < dd) ++l;
    m = (uint32_t)(((1ull << 32) * ((1ull << l) - dd)) / dd + 1);
    s1 = l > 0 ? 1 : 0;
    s2 = l > 0 ? l - 1 : 0;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    const uint32_t t = __umulhi(m, n);
    return (t + ((n - t) >> s1)) >> s2;
  }
};

}  // namespace nmk

// ---- host-side error plumbing (defined in abi.cu) --------------------------
namespace nmk {
int set_error(int code, const char* fmt, ...);
int check_launch(const char* what);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) for the current device if
// `bytes` exceeds what was set there before (the attribute is per device, so
// one process driving several GPUs sets it once per device); defined in abi.cu.
void ensure_dyn_smem(const void* func, size_t bytes);
template <typename F>
inline void ensure_dyn_smem(F* func, size_t bytes) { ensure_dyn_smem(reinterpret_cast<const void*>(func), bytes); }
// multiprocessor count of the current device (cached per device)
int sm_count();
// programmatic dependent launch of the chained kernels: env NMK_PDL = 1 (every
// kernel), 0 / unset (none) or a hex mask 0x.. of chain ids (PdlId)
unsigned pdl_mask();
enum PdlId { kPdlK1 = 0, kPdlPrep, kPdlK2, kPdlK3, kPdlK4, kPdlK4Fallback, kPdlFinalize, kPdlCount, kPdlScan, kPdlDecode };
// <<<grid, block, smem, s>>> with the programmatic-stream-serialization
// attribute; the kernel must call pdl_enter() before touching global memory
template <typename... KA, typename... A>
inline void launch_chain(int id, void (*kernel)(KA...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                         A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = (pdl_mask() >> id) & 1u;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, KA(args)...);
}
}  // namespace nmk
