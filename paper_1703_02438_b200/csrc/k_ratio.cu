// k_ratio.cu — K1: fused change ratio + min/max + valid count.
//
// Restates phase 1 of compress_pair (pkg/src/nmk/pipeline.py:190-212) with
// core.ratio_arrays (core.py:115-137) computed on the fly: the ratio field is
// never materialised, each pass recomputes it from the two snapshots.
// Streaming kernel: 16-byte vector loads of both snapshots, 4 vectors in
// flight per thread, warp-shuffle + smem CTA reduction, last-CTA grid
// reduction (no second launch).
#include <algorithm>
#include <cfloat>

#include "nmk_common.cuh"

namespace nmk {

constexpr int kMinmaxThreads = 256;
#ifndef NMK_MM_UNROLL
#define NMK_MM_UNROLL 3   // A/B: 3 removes the 44-byte spill at 64 registers (cfg2 K1 0.449 -> 0.439 ms); (256, 3) is slower
#endif
#ifndef NMK_MM_MINB
#define NMK_MM_MINB 4
#endif
#ifndef NMK_MM_CTAS
#define NMK_MM_CTAS 8
#endif
constexpr int kMinmaxUnroll = NMK_MM_UNROLL;
#ifndef NMK_MM_CTAS32
#define NMK_MM_CTAS32 4   // A/B on cfg3: 4 beats 8 (K1 86 -> 82 us) and 2
#endif
#ifndef NMK_MM_UNROLL32
#define NMK_MM_UNROLL32 2   // f32: 2 x 16-byte vectors of each snapshot per thread in flight
#endif

struct MinMax {
  double lo, hi;
  unsigned long long nv;
};

// One element into the running (min, max, count) over valid ratios
// (core.py:115-137, pipeline.py:194-197).  The IEEE quotient is only formed
// when the fast approximation cannot rule the element out as a new extreme.
// Returns the element's f32 ratio key for K2 and K4 (ratio_key in
// nmk_common.cuh): finite only when b = x = 0 or b lies in the safe range of
// key_safe<T> (K4's keyed round-trip proof needs it), else +inf ("decide
// exactly") for a valid element and NaN for an invalid one.
template <typename T>
__device__ __forceinline__ float mm_visit(MinMax& a, double b, double x) {
  double ra, ea;
  if (fast_ratio(b, x, ra, ea)) {
    a.nv += 1;                                          // finite quotient: valid
    if (!(__dsub_rn(ra, ea) > a.lo && __dadd_rn(ra, ea) < a.hi)) {
      const double r = __ddiv_rn(__dsub_rn(x, b), b);
      a.lo = r < a.lo ? r : a.lo;
      a.hi = r > a.hi ? r : a.hi;
    }
    return key_safe<T>(b, x) ? ratio_key(ra) : __int_as_float(0x7f800000);
  }
  bool v;
  const double r = change_ratio(b, x, v);
  if (v) {
    a.nv += 1;
    a.lo = r < a.lo ? r : a.lo;
    a.hi = r > a.hi ? r : a.hi;
    return (key_safe<T>(b, x) || (b == 0.0 && x == 0.0)) ? ratio_key(r) : __int_as_float(0x7f800000);
  }
  return __int_as_float(0x7fc00000);   // invalid: quiet NaN
}

// f32 inputs: the common element is decided in f32 arithmetic.  When |b| is
// in [2^-60, 2^60) and the computed d = RN32(x - b) has |d| < |b| / 4, the
// exact difference is below |b| / 4 (1 + 2^-24), so x / b is in (0.74, 1.26),
// x - b is exact (Sterbenz) and r = RN64(d / b) is finite: the element is
// valid and key_safe holds.  The key is d / b by a reciprocal seed (max rel.
// error 2^-22 assumed for rcp.approx) and one FMA Newton correction of the
// quotient: before the last rounding the relative error is below
// (2^-22 + 2^-24)^2 < 2^-43, so |key - r| <= |key| (2^-24 + 2^-43 + 2^-52)
// < |key| 2^-23 -- the key contract of ratio_key (nmk_common.cuh).  No
// intermediate is subnormal in this range (a nonzero |d| is >= 2^-25 |b| >= 2^-85).
// The element can only be a new extreme if [key -+ |key| 2^-22] (rounded
// f32, still containing r) reaches the running extremes, kept as
// lo32 >= RU32(lo) and hi32 <= RD32(hi) (shared across the warp between
// iterations: an element above some lane's minimum is never the global one);
// then the exact f64 quotient is formed.  Everything else takes the f64 path.
__device__ __forceinline__ float mm_visit32(MinMax& a, float& lo32, float& hi32, float b, float x) {
  const float ab = fabsf(b);
  const float d = __fsub_rn(x, b);
  if (ab >= 0x1p-60f && ab < 0x1p+60f && fabsf(d) < 0.25f * ab) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(b));
    const float q0 = __fmul_rn(d, y);
    const float key = __fmaf_rn(__fmaf_rn(-b, q0, d), y, q0);
    a.nv += 1;
    const float m = fabsf(key) * 0x1p-22f;
    if (!(__fsub_rn(key, m) > lo32 && __fadd_rn(key, m) < hi32)) {
      const double r = __ddiv_rn((double)d, (double)b);
      if (r < a.lo) {
        a.lo = r;
        lo32 = fminf(lo32, __double2float_ru(r));
      }
      if (r > a.hi) {
        a.hi = r;
        hi32 = fmaxf(hi32, __double2float_rd(r));
      }
    }
    return key;
  }
  const float key = mm_visit<float>(a, (double)b, (double)x);
  lo32 = fminf(lo32, __double2float_ru(a.lo));
  hi32 = fmaxf(hi32, __double2float_rd(a.hi));
  return key;
}

__device__ __forceinline__ MinMax mm_merge(MinMax a, const MinMax& b) {
  a.lo = b.lo < a.lo ? b.lo : a.lo;
  a.hi = b.hi > a.hi ? b.hi : a.hi;
  a.nv += b.nv;
  return a;
}

#ifndef NMK_MM_LDCS
#define NMK_MM_LDCS 0   // A/B: evict-first snapshot loads (to keep K1's keys in L2 for K2) cost K1 0.439 -> 0.450 ms on cfg2
#endif
#if NMK_MM_LDCS
#define MM_LD(p) __ldcs(p)
#else
#define MM_LD(p) __ldg(p)
#endif

template <int VN>
__device__ __forceinline__ void store_keys(float* p, const float (&kv)[VN]) {
  if constexpr (VN == 2) *reinterpret_cast<float2*>(p) = make_float2(kv[0], kv[1]);
  else *reinterpret_cast<float4*>(p) = make_float4(kv[0], kv[1], kv[2], kv[3]);
}

template <typename T> struct Vec;
template <> struct Vec<double> { using V = double2; static constexpr int N = 2; };
template <> struct Vec<float>  { using V = float4;  static constexpr int N = 4; };

__device__ __forceinline__ void vec_get(const double2& v, double* o) { o[0] = v.x; o[1] = v.y; }
__device__ __forceinline__ void vec_get(const float4& v, double* o) {
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}

// nmk_minmax_prep: K1 also does k_hist_prep's work (single-rank pipelines,
// where the stats need no exchange before the span is decided)
struct HistPrep {
  unsigned long long* counts;   // null: plain nmk_minmax
  double width;
  uint64_t cap_bins, zero_words;
};

template <typename T>
__global__ void __launch_bounds__(kMinmaxThreads, NMK_MM_MINB)
k_minmax(const T* __restrict__ base, const T* __restrict__ cur, uint64_t n,
         MinMax* __restrict__ partials, unsigned int* __restrict__ ticket,
         nmk_stats* __restrict__ out, bool vec_ok, float* __restrict__ keys, HistPrep hp) {
  using V = typename Vec<T>::V;
  constexpr int VN = Vec<T>::N;
  pdl_enter();
  // fused k_hist_prep, part 1: every CTA clears its share of the histogram's
  // first zero_words slots (the span is not known yet; see the last CTA)
  if (hp.counts)
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hp.zero_words;
         i += (uint64_t)gridDim.x * blockDim.x)
      hp.counts[i] = 0ULL;
  MinMax acc;
  acc.nv = 0;
  acc.lo = __longlong_as_double(0x7ff0000000000000LL);   // +inf
  acc.hi = __longlong_as_double(0xfff0000000000000LL);   // -inf
  float lo32 = __int_as_float(0x7f800000), hi32 = __int_as_float(0xff800000);   // f32 path: RU(lo), RD(hi)
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  uint64_t done = 0;
  if (vec_ok) {
    const uint64_t nvec = n / VN;
    const V* bv = reinterpret_cast<const V*>(base);
    const V* cv = reinterpret_cast<const V*>(cur);
    uint64_t i = tid;
    constexpr int U = VN == 4 ? NMK_MM_UNROLL32 : kMinmaxUnroll;
    // warp-uniform trip count (the f32 thresholds are shared by shuffles):
    // a warp iterates while its last lane is in range, the rest is the tail
    const uint64_t lane_hi = 31 - (threadIdx.x & 31);
    for (; i + lane_hi + (U - 1) * nthr < nvec; i += U * nthr) {
      V b[U], c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        b[u] = MM_LD(bv + i + u * nthr);
        c[u] = MM_LD(cv + i + u * nthr);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        float kv[VN];
        if constexpr (VN == 4) {   // f32
          const float bf[4] = {b[u].x, b[u].y, b[u].z, b[u].w}, cf[4] = {c[u].x, c[u].y, c[u].z, c[u].w};
#pragma unroll
          for (int e = 0; e < VN; ++e) kv[e] = mm_visit32(acc, lo32, hi32, bf[e], cf[e]);
        } else {
          double bb[VN], cc[VN];
          vec_get(b[u], bb);
          vec_get(c[u], cc);
#pragma unroll
          for (int e = 0; e < VN; ++e) kv[e] = mm_visit<T>(acc, bb[e], cc[e]);
        }
        if (keys) store_keys<VN>(keys + (i + u * nthr) * VN, kv);
      }
      if constexpr (VN == 4) {   // share the f32 thresholds across the warp
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          lo32 = fminf(lo32, __shfl_xor_sync(0xffffffffu, lo32, o));
          hi32 = fmaxf(hi32, __shfl_xor_sync(0xffffffffu, hi32, o));
        }
      }
    }
    for (; i < nvec; i += nthr) {
      double bb[VN], cc[VN];
      vec_get(__ldg(bv + i), bb);
      vec_get(__ldg(cv + i), cc);
      float kv[VN];
#pragma unroll
      for (int e = 0; e < VN; ++e) kv[e] = mm_visit<T>(acc, bb[e], cc[e]);
      if (keys) store_keys<VN>(keys + i * VN, kv);
    }
    done = nvec * VN;
  }
  for (uint64_t j = done + tid; j < n; j += nthr) {
    const float kv = mm_visit<T>(acc, to_f64(base[j]), to_f64(cur[j]));
    if (keys) keys[j] = kv;
  }
  // warp reduce
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    MinMax other;
    other.lo = __shfl_xor_sync(0xffffffffu, acc.lo, o);
    other.hi = __shfl_xor_sync(0xffffffffu, acc.hi, o);
    other.nv = __shfl_xor_sync(0xffffffffu, acc.nv, o);
    acc = mm_merge(acc, other);
  }
  __shared__ MinMax warp_mm[kMinmaxThreads / 32];
  __shared__ bool is_last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) warp_mm[wid] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    MinMax m = warp_mm[0];
    for (int w = 1; w < kMinmaxThreads / 32; ++w) m = mm_merge(m, warp_mm[w]);
    partials[blockIdx.x] = m;
    __threadfence();
    unsigned prev = atomicAdd(ticket, 1u);
    is_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return;
  // last CTA: reduce all partials (memory ordering via the fence above)
  __threadfence();
  MinMax m;
  m.lo = __longlong_as_double(0x7ff0000000000000LL);
  m.hi = __longlong_as_double(0xfff0000000000000LL);
  m.nv = 0;
  for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
    MinMax p;
    p.lo = __ldcg(&partials[i].lo);
    p.hi = __ldcg(&partials[i].hi);
    p.nv = __ldcg(&partials[i].nv);
    m = mm_merge(m, p);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    MinMax other;
    other.lo = __shfl_xor_sync(0xffffffffu, m.lo, o);
    other.hi = __shfl_xor_sync(0xffffffffu, m.hi, o);
    other.nv = __shfl_xor_sync(0xffffffffu, m.nv, o);
    m = mm_merge(m, other);
  }
  __syncthreads();
  if (lane == 0) warp_mm[wid] = m;
  __syncthreads();
  __shared__ unsigned long long s_nb;
  if (threadIdx.x == 0) {
    MinMax f = warp_mm[0];
    for (int w = 1; w < kMinmaxThreads / 32; ++w) f = mm_merge(f, warp_mm[w]);
    out->gmin = f.lo;
    out->gmax = f.hi;
    out->nvalid = f.nv;
    // fused k_hist_prep, part 2: the dense span (k_hist.cu, same f64 expression)
    unsigned long long nb = 0;
    if (hp.counts && f.nv) {
      const double span = __ddiv_rn(__dsub_rn(f.hi, f.lo), hp.width);
      nb = (finite64(span) && span < (double)hp.cap_bins) ? (unsigned long long)floor(span) + 1ULL : NMK_SPAN_SPARSE;
    }
    out->reserved = nb;
    s_nb = nb;
    *ticket = 0;  // self-reset for the next launch
  }
  if (!hp.counts) return;
  __syncthreads();
  // a span beyond the slots cleared up front (rare): the last CTA clears the rest
  const unsigned long long nb = s_nb;
  if (nb != NMK_SPAN_SPARSE)
    for (uint64_t i = hp.zero_words + threadIdx.x; i <= nb; i += blockDim.x) hp.counts[i] = 0ULL;
}

template <typename T>
__global__ void k_ratio(const T* __restrict__ base, const T* __restrict__ cur, uint64_t n,
                        double* __restrict__ ratios, uint8_t* __restrict__ valid) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x) {
    bool v;
    double r = change_ratio(to_f64(base[j]), to_f64(cur[j]), v);
    ratios[j] = r;
    valid[j] = v ? 1 : 0;
  }
}

static unsigned minmax_grid(uint64_t n, int dtype = NMK_F64) {
  uint64_t want = (n + 4095) / 4096;  // >= 4096 elements per CTA
  // f32: fewer, longer-lived threads -- each thread's first elements are all
  // extreme candidates (exact f64 division), so more elements per thread pay
  uint64_t cap = (uint64_t)sm_count() * (dtype == NMK_F32 ? NMK_MM_CTAS32 : NMK_MM_CTAS);
  if (want < 1) want = 1;
  return (unsigned)(want < cap ? want : cap);
}

}  // namespace nmk

using namespace nmk;

extern "C" size_t nmk_minmax_ws_bytes(uint64_t n) {
  const unsigned g = std::max(minmax_grid(n, NMK_F64), minmax_grid(n, NMK_F32));
  return 256 + (size_t)g * sizeof(MinMax);
}

static int minmax_impl(const void* base, const void* cur, uint64_t n, int dtype, nmk_stats* stats, float* keys,
                       void* ws, size_t ws_bytes, const HistPrep& hp, void* stream) {
  if (n == 0 || !base || !cur || !stats || !ws) return set_error(NMK_ERR_ARG, "nmk_minmax: bad argument");
  if (ws_bytes < nmk_minmax_ws_bytes(n)) return set_error(NMK_ERR_ARG, "nmk_minmax: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  unsigned grid = minmax_grid(n, dtype);
  unsigned* ticket = (unsigned*)ws;
  MinMax* partials = (MinMax*)((char*)ws + 256);
  // The ticket word must be zero on entry: callers zero a fresh workspace
  // once and the kernel's last CTA resets it after every launch.
  bool aligned = (((uintptr_t)base | (uintptr_t)cur | (uintptr_t)keys) & 15) == 0;
  if (dtype == NMK_F64)
    launch_chain(kPdlK1, k_minmax<double>, grid, kMinmaxThreads, 0, s, (const double*)base, (const double*)cur, n, partials,
                 ticket, stats, aligned, keys, hp);
  else if (dtype == NMK_F32)
    launch_chain(kPdlK1, k_minmax<float>, grid, kMinmaxThreads, 0, s, (const float*)base, (const float*)cur, n, partials,
                 ticket, stats, aligned, keys, hp);
  else
    return set_error(NMK_ERR_ARG, "nmk_minmax: bad dtype %d", dtype);
  return check_launch("k_minmax");
}

extern "C" int nmk_minmax(const void* base, const void* cur, uint64_t n, int dtype,
                          nmk_stats* stats, float* keys, void* ws, size_t ws_bytes, void* stream) {
  return minmax_impl(base, cur, n, dtype, stats, keys, ws, ws_bytes, HistPrep{nullptr, 0.0, 0, 0}, stream);
}

extern "C" int nmk_minmax_prep(const void* base, const void* cur, uint64_t n, int dtype, nmk_stats* stats,
                               float* keys, double width, uint64_t cap_bins, unsigned long long* counts,
                               void* ws, size_t ws_bytes, void* stream) {
  if (!counts || cap_bins == 0 || !(width > 0.0)) return set_error(NMK_ERR_ARG, "nmk_minmax_prep: bad argument");
  // slots cleared by all CTAs before the span is known; a wider span's rest
  // is cleared by the last CTA
  const uint64_t zero_words = cap_bins + 1 < 65537 ? cap_bins + 1 : 65537;
  return minmax_impl(base, cur, n, dtype, stats, keys, ws, ws_bytes, HistPrep{counts, width, cap_bins, zero_words},
                     stream);
}

extern "C" int nmk_ratio(const void* base, const void* cur, uint64_t n, int dtype,
                         double* ratios, uint8_t* valid, void* stream) {
  if (n == 0) return NMK_OK;
  if (!base || !cur || !ratios || !valid) return set_error(NMK_ERR_ARG, "nmk_ratio: null pointer");
  cudaStream_t s = (cudaStream_t)stream;
  unsigned grid = minmax_grid(n);
  if (dtype == NMK_F64)
    k_ratio<double><<<grid, 256, 0, s>>>((const double*)base, (const double*)cur, n, ratios, valid);
  else if (dtype == NMK_F32)
    k_ratio<float><<<grid, 256, 0, s>>>((const float*)base, (const float*)cur, n, ratios, valid);
  else
    return set_error(NMK_ERR_ARG, "nmk_ratio: bad dtype %d", dtype);
  return check_launch("k_ratio");
}
