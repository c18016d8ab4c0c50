// k_hist.cu — K2: histogram of bin ordinals floor((r - gmin) / 2E) over the
// valid change ratios (binning.py:110-116, merged per pipeline.py:214-224).
//
// Three forms, chosen by the host from the dense span nbins = q(gmax) + 1:
//  * smem   (nbins <= kSmemBins): per-warp-replica u32 counters in shared
//           memory, per-thread run-length coalescing of equal consecutive
//           ordinals (skewed fields put >90 % of elements in one bin), one
//           u64 global atomic per nonzero bin per CTA at the end;
//  * global (nbins <= kGlobalBins): run-length coalesced u64 atomics into an
//           L2-resident dense array;
//  * sparse (wider spans, e.g. 5e8 bins with 2e3 nonempty in the reference's
//           planted-outlier test): emit the canonical bit pattern of the
//           non-negative double ordinal (invalid -> UINT64_MAX), radix sort,
//           run-length encode.  Output = np.unique(ords, return_counts=True).
#include <algorithm>


#include "nmk_common.cuh"
#include "nmk_block.cuh"
#include "nmk_sort.cuh"

namespace nmk {

constexpr uint64_t kSmemBins = 48 * 1024;       // 192 KB of u32 counters max
constexpr uint64_t kGlobalBins = 1ULL << 22;    // 32 MB of u64 counters max

template <typename T> struct HVec;
template <> struct HVec<double> { using V = double2; static constexpr int N = 2; };
template <> struct HVec<float>  { using V = float4;  static constexpr int N = 4; };
__device__ __forceinline__ void hv_get(const double2& v, double* o) { o[0] = v.x; o[1] = v.y; }
__device__ __forceinline__ void hv_get(const float4& v, double* o) {
  o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}

// Visit every element's (base, current) pair with 16-byte loads when aligned.
template <typename T, int UNROLL, typename F>
__device__ __forceinline__ void for_each_pair(const T* __restrict__ base, const T* __restrict__ cur,
                                               uint64_t n, bool vec_ok, F&& f) {
  using V = typename HVec<T>::V;
  constexpr int VN = HVec<T>::N;
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  uint64_t done = 0;
  if (vec_ok) {
    const uint64_t nvec = n / VN;
    const V* bv = reinterpret_cast<const V*>(base);
    const V* cv = reinterpret_cast<const V*>(cur);
    uint64_t i = tid;
    for (; i + (UNROLL - 1) * nthr < nvec; i += UNROLL * nthr) {
      V b[UNROLL], c[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        b[u] = __ldg(bv + i + u * nthr);
        c[u] = __ldg(cv + i + u * nthr);
      }
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) {
        double bb[VN], cc[VN];
        hv_get(b[u], bb);
        hv_get(c[u], cc);
#pragma unroll
        for (int e = 0; e < VN; ++e) f(bb[e], cc[e], (i + u * nthr) * VN + e);
      }
    }
    for (; i < nvec; i += nthr) {
      double bb[VN], cc[VN];
      hv_get(__ldg(bv + i), bb);
      hv_get(__ldg(cv + i), cc);
#pragma unroll
      for (int e = 0; e < VN; ++e) f(bb[e], cc[e], i * VN + e);
    }
    done = nvec * VN;
  }
  for (uint64_t j = done + tid; j < n; j += nthr) f(to_f64(base[j]), to_f64(cur[j]), j);
}

// Visit the ordinal of every valid element from its f32 ratio key (K1), with
// the (base, current) pair re-read only when the key cannot decide it.
template <typename T, int UNROLL, typename F>
__device__ __forceinline__ void for_each_key_ordinal(const float* __restrict__ keys, const T* __restrict__ base,
                                                     const T* __restrict__ cur, uint64_t n, double gmin, double gmax,
                                                     double width, double inv_w, uint32_t nbins, F&& f) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nthr = (uint64_t)gridDim.x * blockDim.x;
  const double et_c = key_bound(gmin, gmax, inv_w);
  const KeyGrid32 g32 = key_grid32(gmin, gmax, inv_w, nbins);
  auto one = [&](float key, uint64_t j) {
    uint32_t qi;
    if (key_ordinal32(key, g32, qi)) {                       // all-f32 common case
      f(qi);
      return;
    }
    if (key != key) return;                                  // invalid element
    double q;
    if (!key_ordinal_c(key, gmin, inv_w, et_c, q) &&
        !element_ordinal(to_f64(base[j]), to_f64(cur[j]), gmin, width, inv_w, q))
      return;
    f(q);
  };
  const uint64_t nvec = n / 4;
  const float4* kv = reinterpret_cast<const float4*>(keys);
  uint64_t i = tid;
  for (; i + (UNROLL - 1) * nthr < nvec; i += UNROLL * nthr) {
    float4 w[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) w[u] = __ldcs(kv + i + u * nthr);   // streamed once
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const uint64_t j = (i + u * nthr) * 4;
      one(w[u].x, j);
      one(w[u].y, j + 1);
      one(w[u].z, j + 2);
      one(w[u].w, j + 3);
    }
  }
  for (; i < nvec; i += nthr) {
    const float4 w = __ldcs(kv + i);
    one(w.x, i * 4);
    one(w.y, i * 4 + 1);
    one(w.z, i * 4 + 2);
    one(w.w, i * 4 + 3);
  }
  for (uint64_t j = nvec * 4 + tid; j < n; j += nthr) one(keys[j], j);
}

// counts[nbins] is an out-of-range tripwire (must stay 0).
constexpr int kHistThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kHistThreads, 4)
k_hist_smem(const T* __restrict__ base, const T* __restrict__ cur, uint64_t n,
            const nmk_stats* __restrict__ st, double width, uint32_t nbins, int reps,
            unsigned long long* __restrict__ counts, bool vec_ok) {
  extern __shared__ uint32_t h[];
  for (uint32_t i = threadIdx.x; i < nbins * (uint32_t)reps; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const double gmin = st->gmin;
  uint32_t* my = h + (uint32_t)((threadIdx.x >> 5) % reps) * nbins;
  uint32_t last = 0xffffffffu, run = 0;
  const double inv_w = 1.0 / width;
  for_each_pair<T, 4>(base, cur, n, vec_ok, [&](double b, double x, uint64_t) {
    double q;
    if (!element_ordinal(b, x, gmin, width, inv_w, q)) return;
    uint32_t qi = (q < (double)nbins) ? (uint32_t)q : nbins;  // nbins = tripwire
    if (qi == last) {
      ++run;
    } else {
      if (run) {
        if (last < nbins) atomicAdd(&my[last], run);
        else atomicAdd(&counts[nbins], (unsigned long long)run);
      }
      last = qi;
      run = 1;
    }
  });
  if (run) {
    if (last < nbins) atomicAdd(&my[last], run);
    else atomicAdd(&counts[nbins], (unsigned long long)run);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < nbins; i += blockDim.x) {
    uint32_t s = 0;
    for (int r = 0; r < reps; ++r) s += h[r * nbins + i];
    if (s) atomicAdd(&counts[i], (unsigned long long)s);
  }
}

template <typename T>
__global__ void __launch_bounds__(256)
k_hist_global(const T* __restrict__ base, const T* __restrict__ cur, uint64_t n,
              const nmk_stats* __restrict__ st, double width, uint64_t nbins,
              unsigned long long* __restrict__ counts, bool vec_ok) {
  const double gmin = st->gmin;
  uint64_t last = ~0ULL;
  unsigned long long run = 0;
  const double inv_w = 1.0 / width;
  for_each_pair<T, 2>(base, cur, n, vec_ok, [&](double b, double x, uint64_t) {
    double q;
    if (!element_ordinal(b, x, gmin, width, inv_w, q)) return;
    uint64_t qi = (q < (double)nbins) ? (uint64_t)q : nbins;
    if (qi == last) {
      ++run;
    } else {
      if (run) atomicAdd(&counts[last], run);
      last = qi;
      run = 1;
    }
  });
  if (run) atomicAdd(&counts[last], run);
}

template <typename T>
__global__ void __launch_bounds__(256)
k_hist_keys(const T* __restrict__ base, const T* __restrict__ cur, uint64_t n,
            const nmk_stats* __restrict__ st, double width,
            unsigned long long* __restrict__ keys, bool vec_ok) {
  const double gmin = st->gmin;
  const double inv_w = 1.0 / width;
  for_each_pair<T, 2>(base, cur, n, vec_ok, [&](double b, double x, uint64_t j) {
    double q;
    keys[j] = element_ordinal(b, x, gmin, width, inv_w, q) ? (unsigned long long)__double_as_longlong(q) : ~0ULL;
  });
}

// ---- run-length / reduce-by-key over sorted keys ---------------------------
constexpr int kRleThreads = 256;
constexpr int kRleItems = 16;
constexpr int kRleChunk = kRleThreads * kRleItems;

__global__ void __launch_bounds__(kRleThreads)
k_rle_count(const unsigned long long* __restrict__ keys, uint64_t n, unsigned long long* __restrict__ chunk_heads) {
  uint64_t c0 = (uint64_t)blockIdx.x * kRleChunk;
  unsigned cnt = 0;
  for (int it = 0; it < kRleItems; ++it) {
    uint64_t i = c0 + (uint64_t)it * kRleThreads + threadIdx.x;
    if (i < n && keys[i] != ~0ULL && (i == 0 || keys[i] != keys[i - 1])) ++cnt;
  }
  __shared__ unsigned tmp[kRleThreads / 32];
  unsigned tot = block_reduce<kRleThreads>(cnt, SumOp(), tmp);
  if (threadIdx.x == 0) chunk_heads[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kRleThreads)
k_rle_scatter(const unsigned long long* __restrict__ keys, uint64_t n,
              const unsigned long long* __restrict__ chunk_off,
              unsigned long long* __restrict__ run_key, unsigned long long* __restrict__ run_start,
              unsigned long long* __restrict__ nruns, unsigned long long nchunks) {
  __shared__ unsigned tmp[kRleThreads / 32 + 1];
  uint64_t c0 = (uint64_t)blockIdx.x * kRleChunk;
  // thread-contiguous items so ranks follow element order
  uint64_t i0 = c0 + (uint64_t)threadIdx.x * kRleItems;
  unsigned flags = 0, cnt = 0;
  for (int it = 0; it < kRleItems; ++it) {
    uint64_t i = i0 + it;
    bool hd = i < n && keys[i] != ~0ULL && (i == 0 || keys[i] != keys[i - 1]);
    flags |= (hd ? 1u : 0u) << it;
    cnt += hd;
  }
  unsigned tot_unused;
  const unsigned ex = block_exclusive_sum<kRleThreads>(cnt, tot_unused, tmp);
  unsigned long long pos = chunk_off[blockIdx.x] + ex;
  for (int it = 0; it < kRleItems; ++it) {
    if (flags >> it & 1u) {
      run_key[pos] = keys[i0 + it];
      run_start[pos] = i0 + it;
      ++pos;
    }
  }
  if (blockIdx.x == nchunks - 1 && threadIdx.x == kRleThreads - 1) *nruns = pos;
}

__global__ void k_set_u64(unsigned long long* p, unsigned long long v) { *p = v; }

// first index whose key is UINT64_MAX (keys sorted ascending), else n
__global__ void k_valid_end(const unsigned long long* __restrict__ keys, uint64_t n,
                            unsigned long long* __restrict__ out) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    bool here = keys[i] == ~0ULL && (i == 0 || keys[i - 1] != ~0ULL);
    if (here) *out = i;
  }
}

// ---- ratio-array histograms (binning.histogram_of / merge_histograms) -----
// Keys are an order-preserving u64 image of the f64 ordinal, so negative,
// infinite and NaN ordinals (a Histogram built against any origin) sort like
// np.unique: -inf < ... < -0 == +0 < ... < +inf < NaN (one NaN bin).
// ~0ULL stays the "excluded" marker (no canonical value maps to it).
__device__ __forceinline__ unsigned long long ord_key(double q) {
  q = __dadd_rn(q, 0.0);                                   // -0 -> +0
  unsigned long long b = (unsigned long long)__double_as_longlong(q);
  if (q != q) b = 0x7ff8000000000000ULL;                   // one canonical NaN
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double key_ord(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffULL) : ~k;
  return __longlong_as_double((long long)b);
}

// floor(RN(RN(r - origin) / width)) per element (binning.py:113); elements
// with valid[j] == 0 are excluded (build_histogram's valid_ratios, core.py:99)
__global__ void __launch_bounds__(256)
k_ratio_keys(const double* __restrict__ ratios, const uint8_t* __restrict__ valid, uint64_t n, double origin,
             double width, unsigned long long* __restrict__ keys) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
    if (valid && !valid[j]) { keys[j] = ~0ULL; continue; }
    keys[j] = ord_key(floor(__ddiv_rn(__dsub_rn(ratios[j], origin), width)));
  }
}

// in place: each element's f64 ordinal is replaced by its key
__global__ void k_ords_to_keys(unsigned long long* keys, uint64_t n) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x)
    keys[j] = ord_key(__longlong_as_double((long long)keys[j]));
}

__global__ void k_keys_to_ords(unsigned long long* __restrict__ keys, const unsigned long long* __restrict__ nruns) {
  const uint64_t nr = *nruns;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nr; j += (uint64_t)gridDim.x * blockDim.x)
    reinterpret_cast<double*>(keys)[j] = key_ord(keys[j]);
}

static int sm_count_h() { return sm_count(); }

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// Workspace layout shared by the sparse histogram and the merge.
struct RleWs {
  unsigned long long* keys_a;     // n
  unsigned long long* keys_b;     // n
  unsigned long long* run_start;  // n
  unsigned long long* chunk;      // nchunks
  unsigned long long* chunk_off;  // nchunks
  unsigned long long* scal;       // 4 scalars
  unsigned long long* vals_b;     // n (merge only)
  unsigned long long* incl;       // n (merge only)
  void* cub_tmp;      // scratch of the sort / prefix sums (k_sort.cu)
  size_t cub_bytes;
  size_t total;
};

static RleWs rle_layout(uint64_t n, bool with_vals, void* base) {
  RleWs w{};
  uint64_t nchunks = (n + kRleChunk - 1) / kRleChunk;
  // scratch of the sort and of the two prefix sums (used one after the other)
  size_t cub_bytes = sort64_ws_bytes(n, with_vals);
  const size_t scan_bytes = scan64_ws_bytes(nchunks ? nchunks : 1);
  const size_t scan2 = with_vals ? scan64_ws_bytes(n) : 0;
  if (scan_bytes > cub_bytes) cub_bytes = scan_bytes;
  if (scan2 > cub_bytes) cub_bytes = scan2;
  char* p = (char*)base;
  size_t off = 0;
  auto take = [&](size_t bytes) { char* q = p ? p + off : nullptr; off += align256(bytes); return q; };
  w.keys_a = (unsigned long long*)take(n * 8);
  w.keys_b = (unsigned long long*)take(n * 8);
  w.run_start = (unsigned long long*)take(n * 8);
  w.chunk = (unsigned long long*)take((nchunks + 1) * 8);
  w.chunk_off = (unsigned long long*)take((nchunks + 1) * 8);
  w.scal = (unsigned long long*)take(4 * 8);
  if (with_vals) {
    w.vals_b = (unsigned long long*)take(n * 8);
    w.incl = (unsigned long long*)take(n * 8);
  }
  w.cub_tmp = take(cub_bytes);
  w.cub_bytes = cub_bytes;
  w.total = off;
  return w;
}

// Shared tail: sorted keys in w.keys_b (and values in w.vals_b for merge)
// -> run keys + counts written to out_keys/out_counts, *nruns.
static int rle_tail(RleWs& w, uint64_t n, bool with_vals, unsigned long long* out_keys,
                    unsigned long long* out_counts, unsigned long long* nruns, cudaStream_t s) {
  uint64_t nchunks = (n + kRleChunk - 1) / kRleChunk;
  k_rle_count<<<(unsigned)nchunks, kRleThreads, 0, s>>>(w.keys_b, n, w.chunk);
  scan64(w.chunk, w.chunk_off, nchunks, false, w.cub_tmp, s);
  k_rle_scatter<<<(unsigned)nchunks, kRleThreads, 0, s>>>(w.keys_b, n, w.chunk_off, out_keys,
                                                         w.run_start, nruns, nchunks);
  k_set_u64<<<1, 1, 0, s>>>(w.scal, n);  // default end = n (no invalid key)
  unsigned grid = (unsigned)((n + 255) / 256);
  if (grid > (unsigned)sm_count_h() * 8) grid = sm_count_h() * 8;
  k_valid_end<<<grid, 256, 0, s>>>(w.keys_b, n, w.scal);
  if (with_vals) scan64(w.vals_b, w.incl, n, true, w.cub_tmp, s);
  return 0;
}

__global__ void k_rle_lengths_dev(const unsigned long long* __restrict__ run_start,
                                  const unsigned long long* __restrict__ nruns_p,
                                  const unsigned long long* __restrict__ valid_end_p,
                                  const unsigned long long* __restrict__ incl,
                                  unsigned long long* __restrict__ out_counts) {
  uint64_t nr = *nruns_p;
  uint64_t vend = *valid_end_p;
  for (uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nr;
       p += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t s = run_start[p];
    uint64_t e = (p + 1 < nr) ? run_start[p + 1] : vend;
    out_counts[p] = incl ? (incl[e - 1] - (s ? incl[s - 1] : 0ULL)) : (e - s);
  }
}

}  // namespace nmk

using namespace nmk;

extern "C" int nmk_hist_dense(const void* base, const void* cur, uint64_t n, int dtype,
                              const nmk_stats* stats, double width, uint64_t nbins,
                              unsigned long long* counts, void* stream) {
  if (!base || !cur || !stats || !counts || n == 0 || nbins == 0)
    return set_error(NMK_ERR_ARG, "nmk_hist_dense: bad argument");
  if (nbins > kGlobalBins) return set_error(NMK_ERR_ARG, "nmk_hist_dense: nbins %llu too large", (unsigned long long)nbins);
  if (dtype != NMK_F32 && dtype != NMK_F64) return set_error(NMK_ERR_ARG, "nmk_hist_dense: bad dtype");
  cudaStream_t s = (cudaStream_t)stream;
  cudaMemsetAsync(counts, 0, (nbins + 1) * sizeof(unsigned long long), s);
  bool aligned = (((uintptr_t)base | (uintptr_t)cur) & 15) == 0;
  int sms = sm_count_h();
  if (nbins <= kSmemBins) {
    // replicas: one private copy per warp when it fits in ~48 KB, at least 1
    size_t one = nbins * 4;
    int reps = (int)((48 * 1024) / one);
    if (reps > kHistThreads / 32) reps = kHistThreads / 32;
    if (reps < 1) reps = 1;
    size_t smem = one * reps;
    int per_sm = (int)((220 * 1024) / (smem + 1024));
    if (per_sm > 4) per_sm = 4;
    if (per_sm < 1) per_sm = 1;
    uint64_t want = (n + 8191) / 8192;
    uint64_t grid = (uint64_t)sms * per_sm;
    if (want < grid) grid = want ? want : 1;
    if (dtype == NMK_F64) {
      if (smem > 48 * 1024) cudaFuncSetAttribute(k_hist_smem<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_hist_smem<double><<<(unsigned)grid, kHistThreads, smem, s>>>((const double*)base, (const double*)cur, n, stats,
                                                             width, (uint32_t)nbins, reps, counts, aligned);
    } else {
      if (smem > 48 * 1024) cudaFuncSetAttribute(k_hist_smem<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_hist_smem<float><<<(unsigned)grid, kHistThreads, smem, s>>>((const float*)base, (const float*)cur, n, stats,
                                                           width, (uint32_t)nbins, reps, counts, aligned);
    }
    return check_launch("k_hist_smem");
  }
  uint64_t want = (n + 4095) / 4096;
  uint64_t grid = (uint64_t)sms * 8;
  if (want < grid) grid = want ? want : 1;
  if (dtype == NMK_F64)
    k_hist_global<double><<<(unsigned)grid, 256, 0, s>>>((const double*)base, (const double*)cur, n, stats,
                                                         width, nbins, counts, aligned);
  else
    k_hist_global<float><<<(unsigned)grid, 256, 0, s>>>((const float*)base, (const float*)cur, n, stats,
                                                        width, nbins, counts, aligned);
  return check_launch("k_hist_global");
}

extern "C" size_t nmk_hist_sparse_ws_bytes(uint64_t n) { return rle_layout(n, false, nullptr).total; }
extern "C" size_t nmk_hist_merge_ws_bytes(uint64_t n_in) { return rle_layout(n_in, true, nullptr).total; }

extern "C" int nmk_hist_sparse(const void* base, const void* cur, uint64_t n, int dtype,
                               const nmk_stats* stats, double width, unsigned long long* keys,
                               unsigned long long* counts, unsigned long long* nruns, void* ws,
                               size_t ws_bytes, void* stream) {
  if (!base || !cur || !stats || !keys || !counts || !nruns || !ws || n == 0)
    return set_error(NMK_ERR_ARG, "nmk_hist_sparse: bad argument");
  if (dtype != NMK_F32 && dtype != NMK_F64) return set_error(NMK_ERR_ARG, "nmk_hist_sparse: bad dtype");
  RleWs w = rle_layout(n, false, ws);
  if (ws_bytes < w.total) return set_error(NMK_ERR_ARG, "nmk_hist_sparse: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  bool aligned = (((uintptr_t)base | (uintptr_t)cur) & 15) == 0;
  uint64_t want = (n + 4095) / 4096;
  uint64_t grid = (uint64_t)sm_count_h() * 8;
  if (want < grid) grid = want ? want : 1;
  if (dtype == NMK_F64)
    k_hist_keys<double><<<(unsigned)grid, 256, 0, s>>>((const double*)base, (const double*)cur, n, stats, width,
                                                       w.keys_a, aligned);
  else
    k_hist_keys<float><<<(unsigned)grid, 256, 0, s>>>((const float*)base, (const float*)cur, n, stats, width,
                                                      w.keys_a, aligned);
  sort64(w.keys_a, w.keys_b, nullptr, nullptr, n, w.cub_tmp, s);
  rle_tail(w, n, false, keys, counts, nruns, s);
  unsigned g2 = (unsigned)((n + 255) / 256);
  if (g2 > (unsigned)sm_count_h() * 8) g2 = sm_count_h() * 8;
  k_rle_lengths_dev<<<g2, 256, 0, s>>>(w.run_start, nruns, w.scal, nullptr, counts);
  return check_launch("nmk_hist_sparse");
}

extern "C" int nmk_hist_merge(unsigned long long* keys, unsigned long long* counts, uint64_t n_in,
                              unsigned long long* nruns, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n_in == 0) {
    cudaMemsetAsync(nruns, 0, 8, s);
    return check_launch("nmk_hist_merge");
  }
  if (!keys || !counts || !nruns || !ws) return set_error(NMK_ERR_ARG, "nmk_hist_merge: bad argument");
  RleWs w = rle_layout(n_in, true, ws);
  if (ws_bytes < w.total) return set_error(NMK_ERR_ARG, "nmk_hist_merge: workspace too small");
  sort64(keys, w.keys_b, counts, w.vals_b, n_in, w.cub_tmp, s);
  rle_tail(w, n_in, true, keys, counts, nruns, s);
  unsigned g2 = (unsigned)((n_in + 255) / 256);
  if (g2 > (unsigned)sm_count_h() * 8) g2 = sm_count_h() * 8;
  k_rle_lengths_dev<<<g2, 256, 0, s>>>(w.run_start, nruns, w.scal, w.incl, counts);
  return check_launch("nmk_hist_merge");
}

extern "C" size_t nmk_hist_values_ws_bytes(uint64_t n) { return rle_layout(n, false, nullptr).total; }

extern "C" int nmk_hist_values(const double* ratios, const uint8_t* valid, uint64_t n, double origin, double width,
                               double* ordinals, unsigned long long* counts, unsigned long long* nruns, void* ws,
                               size_t ws_bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!ordinals || !counts || !nruns) return set_error(NMK_ERR_ARG, "nmk_hist_values: bad argument");
  if (n == 0) {
    cudaMemsetAsync(nruns, 0, 8, s);
    return check_launch("nmk_hist_values");
  }
  if (!ratios || !ws) return set_error(NMK_ERR_ARG, "nmk_hist_values: bad argument");
  RleWs w = rle_layout(n, false, ws);
  if (ws_bytes < w.total) return set_error(NMK_ERR_ARG, "nmk_hist_values: workspace too small");
  unsigned grid = (unsigned)((n + 255) / 256);
  if (grid > (unsigned)sm_count_h() * 8) grid = sm_count_h() * 8;
  k_ratio_keys<<<grid, 256, 0, s>>>(ratios, valid, n, origin, width, w.keys_a);
  sort64(w.keys_a, w.keys_b, nullptr, nullptr, n, w.cub_tmp, s);
  unsigned long long* out_keys = reinterpret_cast<unsigned long long*>(ordinals);
  rle_tail(w, n, false, out_keys, counts, nruns, s);
  k_rle_lengths_dev<<<grid, 256, 0, s>>>(w.run_start, nruns, w.scal, nullptr, counts);
  k_keys_to_ords<<<grid, 256, 0, s>>>(out_keys, nruns);
  return check_launch("nmk_hist_values");
}

extern "C" int nmk_hist_merge_values(double* ordinals, unsigned long long* counts, uint64_t n_in,
                                     unsigned long long* nruns, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!nruns) return set_error(NMK_ERR_ARG, "nmk_hist_merge_values: bad argument");
  if (n_in == 0) {
    cudaMemsetAsync(nruns, 0, 8, s);
    return check_launch("nmk_hist_merge_values");
  }
  if (!ordinals || !counts || !ws) return set_error(NMK_ERR_ARG, "nmk_hist_merge_values: bad argument");
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(ordinals);
  unsigned grid = (unsigned)((n_in + 255) / 256);
  if (grid > (unsigned)sm_count_h() * 8) grid = sm_count_h() * 8;
  k_ords_to_keys<<<grid, 256, 0, s>>>(keys, n_in);
  const int rc = nmk_hist_merge(keys, counts, n_in, nruns, ws, ws_bytes, stream);
  if (rc) return rc;
  k_keys_to_ords<<<grid, 256, 0, s>>>(keys, nruns);
  return check_launch("nmk_hist_merge_values");
}

// ---- sync-free dense histogram: the span is decided on the device ---------
// k_hist_prep turns the (all-reduced) stats into the dense span
//   nbins = floor(RN(RN(gmax - gmin) / width)) + 1
// (the same f64 expression the host would evaluate), stores it in
// stats->reserved (0: no valid ratio, NMK_SPAN_SPARSE: too wide to densify)
// and zeroes counts[0 .. nbins] (the tripwire slot included).  k_hist_dev
// then bins with shared-memory replicas when the span fits a fixed 48 KB
// budget and with global atomics otherwise; no host round trip is needed.
namespace nmk {

constexpr uint32_t kDevSmemBins = 12 * 1024;   // 48 KB of u32 counters per CTA

__global__ void k_hist_prep(nmk_stats* __restrict__ st, double width, uint64_t cap_bins,
                            unsigned long long* __restrict__ counts) {
  __shared__ unsigned long long s_nb;
  pdl_enter();
  if (threadIdx.x == 0) {
    unsigned long long nb = 0;
    if (st->nvalid) {
      const double span = __ddiv_rn(__dsub_rn(st->gmax, st->gmin), width);
      nb = (finite64(span) && span < (double)cap_bins) ? (unsigned long long)floor(span) + 1ULL : NMK_SPAN_SPARSE;
    }
    s_nb = nb;
    if (blockIdx.x == 0) st->reserved = nb;
  }
  __syncthreads();
  const unsigned long long nb = s_nb;
  if (nb == 0 || nb == NMK_SPAN_SPARSE) return;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= nb; i += (uint64_t)gridDim.x * blockDim.x)
    counts[i] = 0;
}

// ---- key histogram with warp-held hot bins -----------------------------------
// Ratio fields are heavy-headed (most elements fall in one or two bins), so
// each warp holds two "hot" bins whose counts live in per-lane registers
// (a compare and a predicated add each).  Every key that is not a sure hit
// -- an f32-undecided key or a different bin -- is deferred: its bit is set
// in a per-lane mask and, after the tile, re-read from the shared-memory
// stage and counted through the full ordinal (f32 -> f64 key -> exact
// (base, cur)) with one shared-memory atomic into the warp's replica (slot
// nbins = out-of-range tripwire).  When more than 1/8 of a tile misses the
// hot pair the warp promotes the last missing ordinal (the evicted bin's
// count is reduced across the warp and flushed).  (A predicated in-loop
// atomic for the misses measured 5 % slower than the deferral.)
// Keys stream through a
// per-warp ring of TMA bulk copies (kKeyStages x 1 KB), so loads for later
// tiles are in flight while a tile is counted.
constexpr uint32_t kNoBin = 0xffffffffu;
// tile t of a warp's schedule -> tile in memory (ntiles in scope)
#if NMK_HIST_REVERSE
#define TILE_AT(t) (ntiles - 1 - (t))
#else
#define TILE_AT(t) (t)
#endif
#ifndef NMK_PRIV_ATOM
#define NMK_PRIV_ATOM 1   // A/B: atomicAdd beats the plain read-modify-write by 8 % (cfg4)
#endif
#ifndef NMK_HIST_REVERSE
#define NMK_HIST_REVERSE 1   // K2 walks the key tiles last-to-first: K1 wrote them first-to-last, so the tail is still
                             // in L2 (A/B: cfg2 K2 0.112 -> 0.110 ms, step 1.111 -> 1.107; cfg3 / cfg5 unchanged)
#endif
#ifndef NMK_HIST_DIRECT
#define NMK_HIST_DIRECT 1   // out-of-line direct tiles for spread fields (hist_tile_direct)
#endif
#ifndef NMK_HIST_PRIV
#define NMK_HIST_PRIV 1     // lane-private counters for spans <= 63 bins
#endif
#ifndef NMK_KEY_TILE
#define NMK_KEY_TILE 512   // measured: 512 x 2 stages beats 256 x 4 by 15 % (K2)
#endif
#ifndef NMK_KEY_STAGES
#define NMK_KEY_STAGES 2
#endif
constexpr int kKeyTile = NMK_KEY_TILE;     // keys per warp tile
constexpr int kKeyPerLane = kKeyTile / 32;
constexpr int kKeyStages = NMK_KEY_STAGES;
#ifndef NMK_KEY_BINS
#define NMK_KEY_BINS 8192
#endif
constexpr uint32_t kKeySmemBins = NMK_KEY_BINS;   // replicas of nbins + 1 counters (32 KB)

template <typename T>
__device__ __noinline__ uint32_t key_ordinal_slow(float key, const T* __restrict__ base, const T* __restrict__ cur,
                                                  uint64_t j, double gmin, double width, double inv_w,
                                                  double et_c, uint32_t nbins) {
  if (key != key) return kNoBin;   // invalid element
  double q;
  if (!key_ordinal_c(key, gmin, inv_w, et_c, q) &&
      !element_ordinal(to_f64(base[j]), to_f64(cur[j]), gmin, width, inv_w, q))
    return kNoBin;
  return q < (double)nbins ? (uint32_t)q : nbins;   // nbins = tripwire
}

// Hot-bin test in f32 without the magic rounding: th = RN32(key*iw32 + c32)
// with the origin moved to the bin of r = 0 (q_ref), c32 = RN32(c'),
// c' = -gmin/w - 1/2 - q_ref, estimates t* - 1/2 - q_ref (t* = the
// reference's RN(RN(r - gmin)/w)) within
//   e(th, key) = |th| 2^-24 + |key| iw 2^-22 + |c'| 2^-24 + |t*| 2^-52.
// For hot bin h the test |th - (h - q_ref)| < hi_h, with e bounded over bin
// h (|th| <= |h - q_ref| + 1/2, |key| <= max |r| over the bin, + slack),
// proves floor(t*) = h.  The difference th - (h - q_ref) is exact when below
// 1/2 (Sterbenz) and rounds monotonically otherwise.
struct HotGrid {
  double gmin, w, iw, qref, cabs, G;
  float iw32, c32;
};

__device__ __forceinline__ HotGrid hot_grid(double gmin, double width, double inv_w) {
  HotGrid g;
  g.gmin = gmin;
  g.w = width;
  g.iw = inv_w;
  g.G = fabs(gmin) * inv_w;
  const double cd = -gmin * inv_w - 0.5;
  g.qref = rint(cd);
  const double cp = cd - g.qref;   // exact (Sterbenz)
  g.cabs = fabs(cp);
  g.iw32 = __double2float_rn(inv_w);
  g.c32 = __double2float_rn(cp);
  return g;
}

// (h - q_ref as f32, threshold); threshold -1 never matches
__device__ __forceinline__ void hot_params(uint32_t h, uint32_t nbins, const HotGrid& g, float& hc, float& hi) {
  hc = 0.0f;
  hi = -1.0f;
  if (h >= nbins || !(g.G < 0x1p+30) || !(g.iw < 0x1p+100)) return;
  const double hcd = (double)h - g.qref;
  if (fabs(hcd) >= 0x1p+22) return;
  const double rlo = g.gmin + (double)h * g.w, rhi = g.gmin + ((double)h + 1.0) * g.w;
  const double K = fmax(fabs(rlo), fabs(rhi)) * (1.0 + 0x1p-20) + g.w * 0x1p-10;
  const double e = (fabs(hcd) + 0.5) * (0x1p-24 + 0x1p-52) * (1.0 + 0x1p-20) + K * g.iw * 0x1p-22 +
                   g.cabs * 0x1p-24 + g.G * 0x1p-50 + 0x1p-40;
  const double t = 0.5 - e - 0x1p-24;
  if (!(K < 0x1p+100) || !(t > 0.25)) return;
  hc = (float)hcd;   // exact
  hi = __double2float_rz(t);
}

// One tile of a spread field, out of line (hist_keys_hot calls it for tiles
// that follow a tile which missed its hot pair on > 1/4 of the keys):
// every key takes its f32 ordinal (undecided ones the full ordinal); hits on
// the warp's hot pair are counted and returned, other bins go straight to the
// warp's replica.  The deferral loop of the hot path would instead run at the
// pace of the lane with the most misses (cfg5: ~70 % of keys).
struct DirectTile {
  uint32_t c1, c2, miss, last;
};

template <typename T>
__device__ __noinline__ DirectTile hist_tile_direct(const float* sk, const T* __restrict__ base,
                                                    const T* __restrict__ cur, uint64_t j0, double gmin,
                                                    double et_c, double width, double inv_w, uint32_t nbins,
                                                    uint32_t* my, uint32_t hot1, uint32_t hot2, KeyGrid32 g32) {
  const int lane = threadIdx.x & 31;
  DirectTile r{0u, 0u, 0u, kNoBin};
  auto count = [&](uint32_t qi) {
    if (qi == hot1) {
      ++r.c1;
    } else if (qi == hot2) {
      ++r.c2;
    } else {
      atomicAdd(&my[qi], 1u);   // qi <= nbins
      ++r.miss;
      r.last = qi;
    }
  };
  uint32_t defer = 0;
#pragma unroll
  for (int u = 0; u < kKeyPerLane / 4; ++u) {
    const float4 w = reinterpret_cast<const float4*>(sk)[u * 32 + lane];
    const float kv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t qi;
      if (key_ordinal32(kv[e], g32, qi)) count(qi);
      else defer |= 1u << (4 * u + e);
    }
  }
  if (defer) {
    while (defer) {
      const int e = __ffs(defer) - 1;
      defer &= defer - 1;
      const int idx = ((e >> 2) * 32 + lane) * 4 + (e & 3);
      const uint32_t qi = key_ordinal_slow<T>(sk[idx], base, cur, j0 + idx, gmin, width, inv_w, et_c, nbins);
      if (qi != kNoBin) count(qi);
    }
  }
  return r;
}

// kSpread: the spread policy -- every tile takes the direct loop and the hot
// pair is never promoted (fields whose keys are spread over hundreds of bins,
// e.g. cfg5's bimodal mixture, where a promotion would be paid per tile)
template <typename T, bool kSpread>
__device__ __forceinline__ void hist_keys_hot(const float* __restrict__ keys, const T* __restrict__ base,
                                              const T* __restrict__ cur, uint64_t n, double gmin, double gmax,
                                              double width, double inv_w, uint32_t nbins, uint32_t* my,
                                              float* stage, unsigned long long* bars) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const double et_c = key_bound(gmin, gmax, inv_w);
  const KeyGrid32 g32 = key_grid32(gmin, gmax, inv_w, nbins);
  const HotGrid hg = hot_grid(gmin, width, inv_w);
  const unsigned long long iw2 = ((unsigned long long)__float_as_uint(hg.iw32) << 32) | __float_as_uint(hg.iw32);
  const unsigned long long c2c = ((unsigned long long)__float_as_uint(hg.c32) << 32) | __float_as_uint(hg.c32);
  uint32_t hot1 = kNoBin - 1, hot2 = kNoBin - 2;   // never real ordinals
  float h1c = 0.f, h2c = 0.f, hi1 = -1.f, hi2 = -1.f;
  unsigned long long n1c2 = 0, n2c2 = 0;            // (-h1c, -h1c), (-h2c, -h2c) as f32x2
  auto set_hot = [&]() {
    hot_params(hot1, nbins, hg, h1c, hi1);
    hot_params(hot2, nbins, hg, h2c, hi2);
    n1c2 = ((unsigned long long)__float_as_uint(-h1c) << 32) | __float_as_uint(-h1c);
    n2c2 = ((unsigned long long)__float_as_uint(-h2c) << 32) | __float_as_uint(-h2c);
  };
  uint32_t c2 = 0, miss = 0, last_miss = kNoBin;
  bool spread = false;   // warp-uniform: the last tile missed the hot pair on > 1/4 of its keys
  // hot-pair counts: c2 = hot2 hits of the f32 test; hot1 hits are derived,
  // c1 = tested - ndef - c2 + c1x; c1x / c2x: deferred keys resolving to hot1 / hot2
  uint32_t tested = 0, ndef = 0, c1x = 0, c2x = 0;
  // full ordinal of one key (f32 -> f64 key -> exact pair)
  auto ord = [&](float key, uint64_t j) -> uint32_t {
    uint32_t qi;
    if (key_ordinal32(key, g32, qi)) return qi;
    double q;
    if (key == key && key_ordinal_c(key, gmin, inv_w, et_c, q)) return q < (double)nbins ? (uint32_t)q : nbins;
    return key_ordinal_slow<T>(key, base, cur, j, gmin, width, inv_w, et_c, nbins);
  };
  auto visit = [&](uint32_t qi) {
    if (qi == hot1) {
      ++c1x;
    } else if (qi == hot2) {
      ++c2x;
    } else if (qi != kNoBin) {
      atomicAdd(&my[qi], 1u);   // qi <= nbins
      ++miss;
      last_miss = qi;
    }
  };
  auto flush = [&](uint32_t hot, uint32_t c) {
    const uint32_t tot = __reduce_add_sync(FULL, c);
    if (lane == 0 && tot && hot <= nbins) atomicAdd(&my[hot], tot);
  };
  // two keys against the hot pair.  Per key: a hot2 hit is counted, a key in
  // neither hot bin sets its defer bit; hot1 hits are not counted one by one
  // but derived at flush time: c1 = tested - deferred - c2 + c1x (c1x: deferred
  // keys whose full ordinal turned out to be hot1).
  auto hot2keys = [&](float ka, float kb, int e, uint32_t& defer) {
    const unsigned long long k2 = ((unsigned long long)__float_as_uint(kb) << 32) | __float_as_uint(ka);
    unsigned long long th, a, b;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(th) : "l"(k2), "l"(iw2), "l"(c2c));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(a) : "l"(th), "l"(n1c2));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(b) : "l"(th), "l"(n2c2));
    asm("{\n\t.reg .pred p1, p2, q1, q2;\n\t"
        "setp.lt.f32 p1, %3, %5;\n\t"       // key a in hot2
        "setp.lt.f32 q1, %2, %4;\n\t"       // key a in hot1
        "or.pred q1, q1, p1;\n\t"
        "@p1 add.u32 %0, %0, 1;\n\t"
        "@!q1 or.b32 %1, %1, %8;\n\t"
        "setp.lt.f32 p2, %7, %5;\n\t"       // key b in hot2
        "setp.lt.f32 q2, %6, %4;\n\t"       // key b in hot1
        "or.pred q2, q2, p2;\n\t"
        "@p2 add.u32 %0, %0, 1;\n\t"
        "@!q2 or.b32 %1, %1, %9;\n\t"
        "}"
        : "+r"(c2), "+r"(defer)
        : "f"(fabsf(__uint_as_float((uint32_t)a))), "f"(fabsf(__uint_as_float((uint32_t)b))), "f"(hi1), "f"(hi2),
          "f"(fabsf(__uint_as_float((uint32_t)(a >> 32)))), "f"(fabsf(__uint_as_float((uint32_t)(b >> 32)))),
          "r"(1u << e), "r"(2u << e));
  };
  const uint64_t ntiles = n / kKeyTile;
  const uint64_t wg = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  if (lane == 0) {
    for (int st = 0; st < kKeyStages; ++st) mbar_init(&bars[st], 1);
    mbar_fence_init();
  }
  __syncwarp();
  auto issue = [&](int st, uint64_t t) {   // lane 0 only
    mbar_arrive_tx(&bars[st], kKeyTile * 4);
    tma_load_1d(stage + st * kKeyTile, keys + TILE_AT(t) * kKeyTile, kKeyTile * 4, &bars[st]);
  };
  if (lane == 0)
    for (int st = 0; st < kKeyStages; ++st)
      if (wg + st * nw < ntiles) issue(st, wg + st * nw);
  if constexpr (kSpread) {
    // spread policy: every decided key is one shared-memory add into the
    // warp's replica (no hot pair, no per-tile bookkeeping)
    for (uint64_t kk = 0;; ++kk) {   // warp-uniform
      const uint64_t t = wg + kk * nw;
      if (t >= ntiles) break;
      const int st = (int)(kk % kKeyStages);
      mbar_wait(&bars[st], (unsigned)((kk / kKeyStages) & 1));
      const float* sk = stage + st * kKeyTile;
      uint32_t defer = 0;
#pragma unroll
      for (int u = 0; u < kKeyPerLane / 4; ++u) {
        const float4 w = reinterpret_cast<const float4*>(sk)[u * 32 + lane];
        const float kv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          uint32_t qi;
          const bool ok = key_ordinal32(kv[e], g32, qi);
          if (ok) atomicAdd(&my[qi], 1u);
          defer |= ok ? 0u : 1u << (4 * u + e);
        }
      }
      while (defer) {
        const int e = __ffs(defer) - 1;
        defer &= defer - 1;
        const int idx = ((e >> 2) * 32 + lane) * 4 + (e & 3);
        const uint32_t qi = ord(sk[idx], TILE_AT(t) * kKeyTile + idx);
        if (qi != kNoBin) atomicAdd(&my[qi], 1u);
      }
      __syncwarp();
      if (lane == 0) {
        fence_proxy_async_smem();
        const uint64_t nx = t + (uint64_t)kKeyStages * nw;
        if (nx < ntiles) issue(st, nx);
      }
    }
    for (uint64_t j = ntiles * kKeyTile + wg * 32 + lane; j < n; j += nw * 32) {
      const uint32_t qi = ord(keys[j], j);
      if (qi != kNoBin) atomicAdd(&my[qi], 1u);
    }
  } else {
  for (uint64_t kk = 0;; ++kk) {   // warp-uniform
    const uint64_t t = wg + kk * nw;
    if (t >= ntiles) break;
    const int st = (int)(kk % kKeyStages);
    mbar_wait(&bars[st], (unsigned)((kk / kKeyStages) & 1));
    const float* sk = stage + st * kKeyTile;
    uint32_t defer = 0;
    // the previous tile missed the hot pair on > 1/4 of its keys: this one
    // runs the direct loop (A/B: also sampling the tile's own concentration
    // with __match_any_sync before choosing cost cfg2 more than it saved)
    const bool direct = NMK_HIST_DIRECT && (kSpread || spread);
    if (direct) {
      const DirectTile r = hist_tile_direct<T>(sk, base, cur, TILE_AT(t) * kKeyTile, gmin, et_c, width, inv_w, nbins, my,
                                               hot1, hot2, g32);
      c1x += r.c1;
      c2x += r.c2;
      miss += r.miss;
      if (r.miss) last_miss = r.last;
    } else {
#pragma unroll
      for (int u = 0; u < kKeyPerLane / 4; ++u) {
        const float4 w = reinterpret_cast<const float4*>(sk)[u * 32 + lane];
        hot2keys(w.x, w.y, 4 * u, defer);
        hot2keys(w.z, w.w, 4 * u + 2, defer);
      }
      tested += kKeyPerLane;
      ndef += __popc(defer);
    }
    while (defer) {   // this lane's non-hit keys, re-read from the stage
      const int e = __ffs(defer) - 1;
      defer &= defer - 1;
      const int idx = ((e >> 2) * 32 + lane) * 4 + (e & 3);
      visit(ord(sk[idx], TILE_AT(t) * kKeyTile + idx));
    }
    // adapt: promote the most recent miss when the hot pair covers too little
    // (the spread policy never promotes: every tile is direct)
    const unsigned tile_miss = __reduce_add_sync(FULL, miss);
    spread = tile_miss > (unsigned)(kKeyTile / 4);
    if (!kSpread && tile_miss > (unsigned)(kKeyTile / 8)) {
      const unsigned have = __ballot_sync(FULL, last_miss < nbins);
      if (have) {
        const uint32_t cand = __shfl_sync(FULL, last_miss, __ffs(have) - 1);
        if (cand != hot1 && cand != hot2) {
          flush(hot1, tested - ndef - c2 + c1x);
          flush(hot2, c2 + c2x);
          hot2 = hot1;
          hot1 = cand;
          tested = ndef = c1x = c2x = c2 = 0;
          set_hot();
        }
      }
    }
    miss = 0;
    __syncwarp();
    if (lane == 0) {   // refill this stage
      fence_proxy_async_smem();
      const uint64_t nx = t + (uint64_t)kKeyStages * nw;
      if (nx < ntiles) issue(st, nx);
    }
  }
  // tail: the last n % kKeyTile keys, one element per lane per round
  for (uint64_t j = ntiles * kKeyTile + wg * 32 + lane; j < n; j += nw * 32) visit(ord(keys[j], j));
  flush(hot1, tested - ndef - c2 + c1x);
  flush(hot2, c2 + c2x);
  }
}

// ---- key histogram with lane-private counters (spans of <= 63 bins) ---------
// Spread ratio fields (cfg1/cfg4: sigma = one bin, 50 bins; cfg3: ~6 bins)
// defeat the hot pair above: most keys miss it and the deferral loop runs at
// the pace of the unluckiest lane.  With a span this small every lane owns a
// private copy of the whole histogram in shared memory -- u16 counters packed
// two bins per word, word (q / 2) of lane l at [(q / 2) * 32 + l], so a
// warp's 32 updates hit 32 distinct banks and need no conflict resolution.
// Per key: one f32 FMA + magic rounding (key_ordinal32) and one shared add;
// keys the f32 test cannot decide take the full ordinal (ord) in place.
// The u16 halves are drained into the CTA's u32 totals before they can
// overflow (every kPrivDrain tiles: <= 16 * kPrivDrain keys per lane).
constexpr uint32_t kPrivBins = 64;                  // nbins + 1 (tripwire) <= 64
constexpr uint32_t kPrivWords = kPrivBins / 2 * 32; // per warp (4 KB)
constexpr uint32_t kPrivDrain = 256;                // tiles between drains (< 65536 / 16; cheap, and
                                                    // exercised by the 2^29-element tests)

template <typename T>
__device__ __forceinline__ void hist_keys_priv(const float* __restrict__ keys, const T* __restrict__ base,
                                               const T* __restrict__ cur, uint64_t n, double gmin, double gmax,
                                               double width, double inv_w, uint32_t nbins, uint32_t* priv,
                                               uint32_t* cta_tot, float* stage, unsigned long long* bars) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const double et_c = key_bound(gmin, gmax, inv_w);
  const KeyGrid32 g32 = key_grid32(gmin, gmax, inv_w, nbins);
  for (uint32_t i = lane; i < kPrivWords; i += 32) priv[i] = 0;
  uint32_t* mine = priv + lane;
  auto bump = [&](uint32_t qi) {   // qi <= nbins < kPrivBins
#if NMK_PRIV_ATOM
    atomicAdd(&mine[(qi >> 1) * 32], 1u << ((qi & 1u) * 16));   // lane-private: never contended
#else
    mine[(qi >> 1) * 32] += 1u << ((qi & 1u) * 16);
#endif
  };
  auto slow = [&](float key, uint64_t j) {
    double q;
    if (key == key && key_ordinal_c(key, gmin, inv_w, et_c, q)) {
      bump(q < (double)nbins ? (uint32_t)q : nbins);
      return;
    }
    const uint32_t qi = key_ordinal_slow<T>(key, base, cur, j, gmin, width, inv_w, et_c, nbins);
    if (qi != kNoBin) bump(qi);
  };
  auto drain = [&]() {   // lane l sums word l and word l + 32 over the 32 lanes
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t w = lane + 32u * h;
      if (w < kPrivBins / 2) {
        uint32_t lo = 0, hi = 0;
        for (int i = 0; i < 32; ++i) {
          const uint32_t v = priv[w * 32 + ((lane + i) & 31)];   // rotated: no bank conflicts
          lo += v & 0xffffu;
          hi += v >> 16;
        }
        if (lo) atomicAdd(&cta_tot[2 * w], lo);
        if (hi) atomicAdd(&cta_tot[2 * w + 1], hi);
      }
    }
    __syncwarp();
    for (uint32_t i = lane; i < kPrivWords; i += 32) priv[i] = 0;
    __syncwarp();
  };
  const uint64_t ntiles = n / kKeyTile;
  const uint64_t wg = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  if (lane == 0) {
    for (int st = 0; st < kKeyStages; ++st) mbar_init(&bars[st], 1);
    mbar_fence_init();
  }
  __syncwarp();
  auto issue = [&](int st, uint64_t t) {   // lane 0 only
    mbar_arrive_tx(&bars[st], kKeyTile * 4);
    tma_load_1d(stage + st * kKeyTile, keys + TILE_AT(t) * kKeyTile, kKeyTile * 4, &bars[st]);
  };
  if (lane == 0)
    for (int st = 0; st < kKeyStages; ++st)
      if (wg + st * nw < ntiles) issue(st, wg + st * nw);
  uint32_t since = 0;
  for (uint64_t kk = 0;; ++kk) {   // warp-uniform
    const uint64_t t = wg + kk * nw;
    if (t >= ntiles) break;
    const int st = (int)(kk % kKeyStages);
    mbar_wait(&bars[st], (unsigned)((kk / kKeyStages) & 1));
    const float* sk = stage + st * kKeyTile;
    uint32_t defer = 0;
#pragma unroll
    for (int u = 0; u < kKeyPerLane / 4; ++u) {
      const float4 w = reinterpret_cast<const float4*>(sk)[u * 32 + lane];
      const float kv[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        uint32_t qi;
        if (key_ordinal32(kv[e], g32, qi)) bump(qi);
        else defer |= 1u << (4 * u + e);
      }
    }
    while (defer) {   // rare: undecided / invalid / out-of-range keys
      const int e = __ffs(defer) - 1;
      defer &= defer - 1;
      const int idx = ((e >> 2) * 32 + lane) * 4 + (e & 3);
      slow(sk[idx], TILE_AT(t) * kKeyTile + idx);
    }
    __syncwarp();
    if (lane == 0) {   // refill this stage
      fence_proxy_async_smem();
      const uint64_t nx = t + (uint64_t)kKeyStages * nw;
      if (nx < ntiles) issue(st, nx);
    }
    if (++since == kPrivDrain) {
      drain();
      since = 0;
    }
  }
  // tail: the last n % kKeyTile keys, one element per lane per round
  for (uint64_t j = ntiles * kKeyTile + wg * 32 + lane; j < n; j += nw * 32) {
    const float key = keys[j];
    uint32_t qi;
    if (key_ordinal32(key, g32, qi)) bump(qi);
    else slow(key, j);
  }
  drain();
  (void)FULL;
}

// Two launch shapes of the same kernel.  kW = 0: 256 threads, 3 CTAs/SM,
// key replicas of up to 8192 counters (spans of the concentrated fields).
// kW = 1 ("wide"): one 512-thread CTA per SM with 96 KB of replica counters,
// so spans of 8K..24K bins (cfg5 at E = 1e-4: 10^4 bins) still count into
// shared memory -- 2 replicas of 10^4 bins, 8 warps each -- instead of one
// 48 KB replica per CTA with run-length atomics.  The host picks the shape
// from a span hint (the previous step's span); the kernel decides its path
// from the actual span, so a wrong hint costs speed, never correctness.
#ifndef NMK_K2_MINB
#define NMK_K2_MINB 3
#endif
template <int kW> struct HistShape;
template <> struct HistShape<0> {   // concentrated fields: hot-pair policy
  static constexpr int kThreads = kHistThreads, kMinBlocks = NMK_K2_MINB;
  static constexpr uint32_t kRepWords = kKeySmemBins;
  static constexpr bool kSpread = false;
};
#ifndef NMK_WIDE_WORDS
#define NMK_WIDE_WORDS 20480    // 80 KB of counters + 32 warps x 4 KB of key stages
#endif
#ifndef NMK_WIDE_THREADS
#define NMK_WIDE_THREADS 1024   // A/B (cfg5 E=1e-4 K2): 512 0.39 ms, 768 0.29, 1024 0.26
#endif
template <> struct HistShape<1> {   // spread fields over 8K..24K bins
  static constexpr int kThreads = NMK_WIDE_THREADS, kMinBlocks = 1;
  static constexpr uint32_t kRepWords = NMK_WIDE_WORDS;
  static constexpr bool kSpread = true;
};
template <> struct HistShape<2> {   // spread fields over < 8K bins
  static constexpr int kThreads = kHistThreads, kMinBlocks = NMK_K2_MINB;
  static constexpr uint32_t kRepWords = kKeySmemBins;
  static constexpr bool kSpread = true;
};
template <int kW>
constexpr size_t hist_dev_smem() {
  return std::max<size_t>(kDevSmemBins * 4, HistShape<kW>::kRepWords * 4 +
                                                (HistShape<kW>::kThreads / 32) * kKeyStages * kKeyTile * 4);
}

template <typename T, int kW>
__global__ void __launch_bounds__(HistShape<kW>::kThreads, HistShape<kW>::kMinBlocks)
k_hist_dev(const T* __restrict__ base, const T* __restrict__ cur, const float* __restrict__ keys, uint64_t n,
           const nmk_stats* __restrict__ st, double width, unsigned long long* __restrict__ counts, bool vec_ok) {
  constexpr int kT = HistShape<kW>::kThreads;
  constexpr uint32_t kRW = HistShape<kW>::kRepWords;
  extern __shared__ uint32_t h[];
  pdl_enter();
  const unsigned long long nb64 = st->reserved;
  if (nb64 == 0 || nb64 == NMK_SPAN_SPARSE) return;
  const uint32_t nbins = (uint32_t)nb64;
  const double gmin = st->gmin;
  const double inv_w = 1.0 / width;
  if constexpr (HistShape<kW>::kSpread) {
    // spread shapes carry only their replica path (fewer registers); a span
    // they do not fit -- a stale hint -- takes the global-atomic path below
    if (keys && nbins + 1 <= kRW) {
      __shared__ unsigned long long s_bars_sp[kT / 32][kKeyStages];
      const uint32_t nb1 = nbins + 1;
      int reps = (int)(kRW / nb1);
      if (reps > kT / 32) reps = kT / 32;
      for (uint32_t i = threadIdx.x; i < nb1 * (uint32_t)reps; i += blockDim.x) h[i] = 0;
      __syncthreads();
      const int wid = threadIdx.x >> 5;
      float* stage = reinterpret_cast<float*>(h + kRW) + wid * kKeyStages * kKeyTile;
      hist_keys_hot<T, true>(keys, base, cur, n, gmin, st->gmax, width, inv_w, nbins,
                             h + (uint32_t)(wid % reps) * nb1, stage, s_bars_sp[wid]);
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < nb1; i += blockDim.x) {
        uint32_t s = 0;
        for (int r = 0; r < reps; ++r) s += h[r * nb1 + i];
        if (s) atomicAdd(&counts[i], (unsigned long long)s);
      }
      return;
    }
  } else if (nbins <= kDevSmemBins || (keys && nbins + 1 <= kRW)) {
    __shared__ unsigned long long s_bars[kT / 32][kKeyStages];
    static_assert(kPrivWords * (kT / 32) <= kRW, "private tables alias the replicas");
    if (NMK_HIST_PRIV && keys && nbins + 1 <= kPrivBins) {   // lane-private counters (tripwire = slot nbins)
      __shared__ uint32_t s_tot[kPrivBins];
      if (threadIdx.x < kPrivBins) s_tot[threadIdx.x] = 0;
      __syncthreads();
      const int wid = threadIdx.x >> 5;
      float* stage = reinterpret_cast<float*>(h + kRW) + wid * kKeyStages * kKeyTile;
      hist_keys_priv<T>(keys, base, cur, n, gmin, st->gmax, width, inv_w, nbins, h + wid * kPrivWords, s_tot, stage,
                        s_bars[wid]);
      __syncthreads();
      if (threadIdx.x <= nbins && s_tot[threadIdx.x])
        atomicAdd(&counts[threadIdx.x], (unsigned long long)s_tot[threadIdx.x]);
      return;
    }
    if (keys && nbins + 1 <= kRW) {   // replicas of nbins + 1 slots (tripwire last)
      const uint32_t nb1 = nbins + 1;
      int reps = (int)(kRW / nb1);
      if (reps > kT / 32) reps = kT / 32;
      for (uint32_t i = threadIdx.x; i < nb1 * (uint32_t)reps; i += blockDim.x) h[i] = 0;
      __syncthreads();
      const int wid = threadIdx.x >> 5;
      float* stage = reinterpret_cast<float*>(h + kRW) + wid * kKeyStages * kKeyTile;
      hist_keys_hot<T, false>(keys, base, cur, n, gmin, st->gmax, width, inv_w, nbins,
                              h + (uint32_t)(wid % reps) * nb1, stage, s_bars[wid]);
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < nb1; i += blockDim.x) {
        uint32_t s = 0;
        for (int r = 0; r < reps; ++r) s += h[r * nb1 + i];
        if (s) atomicAdd(&counts[i], (unsigned long long)s);
      }
      return;
    }
    int reps = (int)(kDevSmemBins / nbins);
    if (reps > kT / 32) reps = kT / 32;
    for (uint32_t i = threadIdx.x; i < nbins * (uint32_t)reps; i += blockDim.x) h[i] = 0;
    __syncthreads();
    uint32_t* my = h + (uint32_t)((threadIdx.x >> 5) % reps) * nbins;
    uint32_t last = 0xffffffffu, run = 0;
    auto add_q = [&](auto q) {   // float (f32 key path) or double ordinal
      const uint32_t qi = (q < (decltype(q))nbins) ? (uint32_t)q : nbins;   // nbins = tripwire
      if (qi == last) {
        ++run;
      } else {
        if (run) {
          if (last < nbins) atomicAdd(&my[last], run);
          else atomicAdd(&counts[nbins], (unsigned long long)run);
        }
        last = qi;
        run = 1;
      }
    };
    if (keys) {
      for_each_key_ordinal<T, 4>(keys, base, cur, n, gmin, st->gmax, width, inv_w, nbins, add_q);
    } else {
      for_each_pair<T, 4>(base, cur, n, vec_ok, [&](double b, double x, uint64_t) {
        double q;
        if (element_ordinal(b, x, gmin, width, inv_w, q)) add_q(q);
      });
    }
    if (run) {
      if (last < nbins) atomicAdd(&my[last], run);
      else atomicAdd(&counts[nbins], (unsigned long long)run);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nbins; i += blockDim.x) {
      uint32_t s = 0;
      for (int r = 0; r < reps; ++r) s += h[r * nbins + i];
      if (s) atomicAdd(&counts[i], (unsigned long long)s);
    }
    return;
  }
  {
    uint64_t last = ~0ULL;
    unsigned long long run = 0;
    auto add_q = [&](auto q) {
      const uint64_t qi = (q < (decltype(q))nbins) ? (uint64_t)q : nbins;
      if (qi == last) {
        ++run;
      } else {
        if (run) atomicAdd(&counts[last], run);
        last = qi;
        run = 1;
      }
    };
    if (keys) {
      for_each_key_ordinal<T, 2>(keys, base, cur, n, gmin, st->gmax, width, inv_w, nbins, add_q);
    } else {
      for_each_pair<T, 2>(base, cur, n, vec_ok, [&](double b, double x, uint64_t) {
        double q;
        if (element_ordinal(b, x, gmin, width, inv_w, q)) add_q(q);
      });
    }
    if (run) atomicAdd(&counts[last], run);
  }
}

}  // namespace nmk

extern "C" int nmk_hist_prep(nmk_stats* stats, double width, uint64_t cap_bins, unsigned long long* counts,
                             void* stream) {
  if (!stats || !counts || cap_bins == 0) return set_error(NMK_ERR_ARG, "nmk_hist_prep: bad argument");
  launch_chain(kPdlPrep, k_hist_prep, sm_count_h() * 2, 256, 0, (cudaStream_t)stream, stats, width, cap_bins, counts);
  return check_launch("k_hist_prep");
}

template <int kW>
static void launch_hist_dev(const void* base, const void* cur, const float* keys, uint64_t n, int dtype,
                            const nmk_stats* stats, double width, unsigned long long* counts, bool aligned,
                            cudaStream_t s) {
  constexpr size_t smem = hist_dev_smem<kW>();
  constexpr int kT = HistShape<kW>::kThreads;
  ensure_dyn_smem(k_hist_dev<double, kW>, smem);
  ensure_dyn_smem(k_hist_dev<float, kW>, smem);
  // one resident wave: the grid-stride loops split the work evenly over it
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_hist_dev<double, kW>, kT, smem);
  if (per_sm < 1) per_sm = 1;
  uint64_t want = (n + 8191) / 8192;
  uint64_t grid = (uint64_t)sm_count_h() * per_sm;
  if (want < grid) grid = want ? want : 1;
  if (dtype == NMK_F64)
    launch_chain(kPdlK2, k_hist_dev<double, kW>, (unsigned)grid, kT, smem, s, (const double*)base, (const double*)cur, keys, n,
                 stats, width, counts, aligned);
  else
    launch_chain(kPdlK2, k_hist_dev<float, kW>, (unsigned)grid, kT, smem, s, (const float*)base, (const float*)cur, keys, n,
                 stats, width, counts, aligned);
}

extern "C" int nmk_hist_dense_dev2(const void* base, const void* cur, const float* keys, uint64_t n, int dtype,
                                   const nmk_stats* stats, double width, unsigned long long* counts,
                                   uint64_t span_hint, int spread_hint, void* stream) {
  if (keys && ((uintptr_t)keys & 15)) return set_error(NMK_ERR_ARG, "nmk_hist_dense_dev: keys must be 16-byte aligned");
  if (!base || !cur || !stats || !counts || n == 0) return set_error(NMK_ERR_ARG, "nmk_hist_dense_dev: bad argument");
  if (dtype != NMK_F32 && dtype != NMK_F64) return set_error(NMK_ERR_ARG, "nmk_hist_dense_dev: bad dtype");
  cudaStream_t s = (cudaStream_t)stream;
  const bool aligned = (((uintptr_t)base | (uintptr_t)cur) & 15) == 0;
  // wide shape only where its replicas are the ones that fit
  const bool wide = keys && span_hint + 1 > kKeySmemBins && span_hint + 1 <= HistShape<1>::kRepWords;
  if (wide) launch_hist_dev<1>(base, cur, keys, n, dtype, stats, width, counts, aligned, s);
  else if (keys && spread_hint && span_hint + 1 > kPrivBins) launch_hist_dev<2>(base, cur, keys, n, dtype, stats, width, counts, aligned, s);
  else launch_hist_dev<0>(base, cur, keys, n, dtype, stats, width, counts, aligned, s);
  return check_launch("k_hist_dev");
}

extern "C" int nmk_hist_dense_dev(const void* base, const void* cur, const float* keys, uint64_t n, int dtype,
                                  const nmk_stats* stats, double width, unsigned long long* counts, void* stream) {
  return nmk_hist_dense_dev2(base, cur, keys, n, dtype, stats, width, counts, 0, 0, stream);
}
