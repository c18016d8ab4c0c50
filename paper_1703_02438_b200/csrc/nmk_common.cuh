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

// Ordinal from a key (K2): true with the exact ordinal when decidable, false
// when the exact path (IEEE ratio + IEEE bin division) must run.
__device__ __forceinline__ bool key_ordinal(float key, double origin, double inv_w, double& q) {
  const double kd = (double)key;
  const double s = __dsub_rn(kd, origin);
  const double t = __dmul_rn(s, inv_w);
  const double et = __dadd_rn(__dmul_rn(__dadd_rn(fabs(kd) * 0x1p-22, fabs(s) * 0x1p-48), inv_w * 1.0000001),
                              fabs(t) * 0x1p-46);
  const double fl = floor(t);
  if (t < 0x1p+50 && __dsub_rn(t, fl) > et && __dsub_rn(__dadd_rn(fl, 1.0), t) > et) {
    q = __dadd_rn(fl, 0.0);
    return true;
  }
  return false;
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
// cell, #cuts below the cell's left edge.  The cell of r gives a starting
// guess; two exact compare loops then land on #cuts < r.  The answer is
// exact whatever the rounding of the cell computation (monotone cuts), the
// grid only makes it O(1) on average.
constexpr int kLutCells = 8192;

struct CutLut {
  const double* cuts;      // shared memory
  const uint16_t* lut;     // shared memory, kLutCells entries
  int ncuts;
  double lo, scale;
  bool use_lut;

  __device__ __forceinline__ uint32_t find(double r) const {
    if (!use_lut) return lower_bound_cuts(cuts, ncuts, r);
    double f = (r - lo) * scale;
    f = fmin(fmax(f, 0.0), (double)(kLutCells - 1));
    int i = lut[(int)f];
    while (i < ncuts && cuts[i] < r) ++i;
    while (i > 0 && cuts[i - 1] >= r) --i;
    return (uint32_t)i;
  }
};

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

// ---- cp.async (LDGSTS) helpers ---------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
// 4/8-byte copy with zero fill when !valid (src-size 0 reads nothing)
template <int N>
__device__ __forceinline__ void cp_async_zfill(void* s, const void* g, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(smem_u32(s)), "l"(g), "n"(N),
               "r"(valid ? N : 0) : "memory");
}
// 4-byte slot filled with the first `have` (0..4) source bytes, rest zero
__device__ __forceinline__ void cp_async_bytes4(void* s, const void* g, int have) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(s)), "l"(g), "r"(have) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// ---- TMA bulk copies + mbarriers (sm_90+/sm_100a) --------------------------
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

// Element stage: thread t's 8 consecutive elements at t*kRow(T) bytes, a row
// padded by 16 bytes so 128-bit shared loads of 8 threads hit distinct banks.
template <typename T> struct Stage {
  static constexpr int kRow = kGroup * (int)sizeof(T) + 16;        // 80 (f64) / 48 (f32)
  static constexpr int kBytes = kTileThreads * kRow;               // one array of a tile
  __device__ __forceinline__ static int off(int e) {               // element e of the tile
    return (e / kGroup) * kRow + (e % kGroup) * (int)sizeof(T);
  }
};

// Issue the loads of `src[li0 .. li0 + cnt)` (tile elements e0 .. e0 + cnt)
// into a Stage array.  Fast path: whole tile, 16-byte aligned.
template <typename T>
__device__ __forceinline__ void stage_tile(unsigned char* stage, const T* __restrict__ src, int64_t li_first,
                                           int e0, int cnt) {
  constexpr int VN = 16 / (int)sizeof(T);
  const T* g = src + li_first;  // element e of the tile lives at g[e]
  if (e0 == 0 && cnt == kTile && (((uintptr_t)g) & 15) == 0) {
#pragma unroll
    for (int m = 0; m < kTile / VN / kTileThreads; ++m) {
      int c = threadIdx.x + m * kTileThreads;   // 16-byte chunk
      cp_async16(stage + Stage<T>::off(c * VN), g + c * VN);
    }
  } else {
    for (int e = threadIdx.x; e < kTile; e += kTileThreads) {
      bool ok = e >= e0 && e < e0 + cnt;
      cp_async_zfill<(int)sizeof(T)>(stage + Stage<T>::off(e), ok ? (const void*)(g + e) : (const void*)src, ok);
    }
  }
}

template <typename T>
__device__ __forceinline__ void unstage_group(const unsigned char* stage, T (&v)[kGroup]) {
  const unsigned char* row = stage + threadIdx.x * Stage<T>::kRow;
#pragma unroll
  for (int q = 0; q < (int)(kGroup * sizeof(T)) / 16; ++q) {
    uint4 w = *reinterpret_cast<const uint4*>(row + 16 * q);
    const T* tw = reinterpret_cast<const T*>(&w);
#pragma unroll
    for (int e = 0; e < 16 / (int)sizeof(T); ++e) v[q * (16 / (int)sizeof(T)) + e] = tw[e];
  }
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
