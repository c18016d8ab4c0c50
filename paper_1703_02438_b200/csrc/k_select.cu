// k_select.cu — K3: single-CTA bin selection.
//
// Restates, in one 1024-thread CTA and without leaving the device:
//  * _selectable           (binning.py:135-139): bins with a finite center;
//  * select_index_length   (binning.py:155-206): auto B over [2, 16] with the
//    Eq. 6 size model, ties to the smaller B;
//  * top_k_bins            (binning.py:142-152): the k = min(2^B-1, m) bins
//    ordered by (count desc, ordinal asc), centers sorted and deduplicated;
//  * _quantize_centers     (pipeline.py:112-124): round to the storage dtype,
//    deduplicate, drop non-finite, fall back to [0.0];
//  * _degenerate_model     (pipeline.py:163-167) when no ratio is valid;
//  * the midpoint cuts used by nearest_center (binning.py:299).
//
// The k-th largest count is found with an MSB-first radix select (8-bit
// digits) over the bin counts instead of a full lexsort: the selected set is
// {count > t} plus the lowest-ordinal bins with count == t, which is exactly
// the first k rows of lexsort((ordinal, -count)).  Bins arrive in ordinal
// order and centers are monotone in the ordinal, so compacting the selected
// bins in ordinal order yields np.unique's sorted order directly.

#include "nmk_common.cuh"
#include "nmk_block.cuh"

namespace nmk {

#ifndef NMK_SEL_THREADS
#define NMK_SEL_THREADS 512   // A/B: 512 beats 1024 (cfg2 23 -> 18 us; fewer warps per barrier) and 256 (10^4 bins)
#endif
constexpr int kSelThreads = NMK_SEL_THREADS;
constexpr int kAutoLo = 2, kAutoHi = 16;           // binning.py:22
constexpr int kNSel = kAutoHi - kAutoLo + 1;       // 15 simultaneous selects (auto B)
constexpr int kNSelMax = 29;                       // B = 2..30: select_index_length's widest range

constexpr uint64_t kSelCache = 20480;  // bins whose selectable counts live in smem (160 KB)

struct BinView {
  const unsigned long long* keys;    // null -> dense (ordinal = index)
  const unsigned long long* counts;
  uint64_t m;
  double origin, width;
  const unsigned long long* cache;   // shared-memory copy of sel_count, or null
  __device__ __forceinline__ double ord(uint64_t i) const {
    return keys ? __longlong_as_double((long long)keys[i]) : (double)i;
  }
  __device__ __forceinline__ double center(uint64_t i) const { return bin_center(ord(i), origin, width); }
  // count if the bin is nonempty and selectable, else 0
  __device__ __forceinline__ unsigned long long sel_count(uint64_t i) const {
    if (cache) return cache[i];
    unsigned long long c = counts[i];
    if (c == 0) return 0;
    return finite64(center(i)) ? c : 0ULL;
  }
};

template <typename T>
__device__ __forceinline__ double quantize(double c) { return to_f64(narrow<T>(c)); }

// pass A's per-thread record: selectable bins, their total, the two largest counts
struct PassA {
  unsigned long long m, tot, a, b;
};
struct PassAOp {
  __device__ __forceinline__ PassA operator()(const PassA& x, const PassA& y) const {
    PassA r;
    r.m = x.m + y.m;
    r.tot = x.tot + y.tot;
    r.a = x.a > y.a ? x.a : y.a;
    const unsigned long long lo = x.a > y.a ? y.a : x.a;   // the smaller top
    const unsigned long long sb = x.b > y.b ? x.b : y.b;
    r.b = lo > sb ? lo : sb;
    return r;
  }
};

// NS = radix-select slots compiled in; auto B (bits_cfg < 0) runs auto_n of
// them for B = auto_lo .. auto_lo + auto_n - 1.  cov_out != null: coverage
// only (binning._coverage_by_bits) -- write the covered counts and stop.
template <typename T, int NS>
__global__ void __launch_bounds__(kSelThreads)
k_select(const unsigned long long* __restrict__ keys, const unsigned long long* __restrict__ counts,
         uint64_t m_max, const unsigned long long* __restrict__ nruns,
         const nmk_stats* __restrict__ st, double width, double tolerance, int bits_cfg,
         uint64_t n_total, double* __restrict__ centers, double* __restrict__ cuts,
         T* __restrict__ centers_t, uint64_t cap_k, nmk_model* __restrict__ model,
         int auto_lo, int auto_n, unsigned long long* __restrict__ cov_out) {
  __shared__ union {   // scratch of the CTA-wide reduce / exclusive sum (nmk_block.cuh)
    unsigned long long red[kSelThreads / 32];
    PassA reda[kSelThreads / 32];
    unsigned scan[kSelThreads / 32 + 1];
  } tmp;
  __shared__ unsigned hist[NS][256];
  __shared__ unsigned long long s_prefix[NS], s_mask[NS], s_left[NS], s_kk[NS];
  __shared__ unsigned long long s_cov[NS];
  __shared__ unsigned long long s_bcast[4];
  __shared__ int s_bits;
  __shared__ double s_prev;
  extern __shared__ unsigned long long s_cache[];

  const int tid = threadIdx.x;
  pdl_enter();
  const uint64_t nvalid = st->nvalid;
  if (nvalid == 0 && cov_out) {   // coverage of an empty histogram
    if (tid < auto_n) cov_out[tid] = 0;
    if (tid == 0) { model->status = NMK_ERR_EMPTY_HIST; model->k = 0; model->m_selectable = 0; }
    return;
  }
  if (nvalid == 0) {  // degenerate model (pipeline.py:163-167)
    if (tid == 0) {
      model->bits = bits_cfg >= 0 ? bits_cfg : 2;
      model->k = 1;
      model->status = 0;
      model->m_selectable = 0;
      model->tol_bin = tolerance;
      for (int b = 0; b < 17; ++b) model->coverage[b] = 0;
      centers[0] = 0.0;
      centers_t[0] = narrow<T>(0.0);
    }
    return;
  }
  uint64_t Mv = nruns ? (uint64_t)*nruns : m_max;
  if (!keys && m_max == 0) {   // sync-free path: span decided on the device
    Mv = st->reserved;
    if (Mv == NMK_SPAN_SPARSE) {
      if (tid == 0) { model->status = NMK_ERR_NEEDS_SPARSE; model->k = 0; model->m_selectable = 0; }
      return;
    }
  }
  if (!keys && counts[Mv] != 0) {   // dense form: K2's out-of-span tripwire slot must be empty
    if (tid == 0) { model->status = NMK_ERR_ARG; model->k = 0; model->m_selectable = 0; }
    return;
  }
  BinView bv{keys, counts, Mv, st->gmin, width, nullptr};
  const uint64_t M = bv.m;
  if ((m_max == 0 && !keys) ? M <= kSelCache : m_max <= kSelCache) {   // passes then read shared memory
    for (uint64_t i = tid; i < M; i += kSelThreads) s_cache[i] = bv.sel_count(i);
    __syncthreads();
    bv.cache = s_cache;
  }

  // ---- pass A: m (selectable bins), total selectable count, and the two
  // largest counts (the second tells the next step's K2 how much of the
  // field a hot pair of bins can hold) -- one block reduction
  PassA pa{0, 0, 0, 0};
  for (uint64_t i = tid; i < M; i += kSelThreads) {
    unsigned long long c = bv.sel_count(i);
    if (c) {
      ++pa.m;
      pa.tot += c;
      if (c > pa.a) { pa.b = pa.a; pa.a = c; }
      else if (c > pa.b) pa.b = c;
    }
  }
  pa = block_reduce<kSelThreads>(pa, PassAOp(), tmp.reda);
  if (tid == 0) { s_bcast[0] = pa.m; s_bcast[1] = pa.a; s_bcast[2] = pa.tot; s_bcast[3] = pa.b; }
  __syncthreads();
  unsigned long long m = s_bcast[0], maxc = s_bcast[1], tot = s_bcast[2];
  const unsigned long long second = s_bcast[3];
  if (m == 0) {
    if (tid == 0) { model->status = NMK_ERR_EMPTY_HIST; model->k = 0; model->m_selectable = 0; }
    if (cov_out && tid < auto_n) cov_out[tid] = 0;
    return;
  }

  // ---- multi radix select: one lane per requested k --------------------
  // slot s requests kk[s]; slot inactive when kk >= m (everything selected)
  const bool autob = bits_cfg < 0;
  if (tid < NS) {
    int b = autob ? auto_lo + tid : bits_cfg;
    unsigned long long kk = (b >= 63) ? ~0ULL : ((1ULL << b) - 1);
    if (kk > m) kk = m;
    s_kk[tid] = ((autob && tid < auto_n) || tid == 0) ? kk : m;  // fixed B uses slot 0 only
    s_prefix[tid] = 0; s_mask[tid] = 0; s_left[tid] = s_kk[tid];
  }
  __syncthreads();
  const int nslots = autob ? auto_n : 1;   // fixed B: slot 0 only
  bool any_sel = false;                   // some slot must select (k < m); else every bin is taken
  for (int s = 0; s < nslots; ++s) any_sel |= s_kk[s] < m;
  int top = 63 - __clzll(maxc | 1ULL);
  for (int shift = any_sel ? (top / 8) * 8 : -1; shift >= 0; shift -= 8) {
    for (int i = tid; i < nslots * 256; i += kSelThreads) (&hist[0][0])[i] = 0;
    __syncthreads();
    for (uint64_t i0 = 0; i0 < M; i0 += kSelThreads) {   // warp-uniform trip count
      const uint64_t i = i0 + tid;
      const unsigned long long c = i < M ? bv.sel_count(i) : 0ULL;
      const unsigned d = (unsigned)(c >> shift) & 255u;
      for (int s = 0; s < nslots; ++s) {
        if (!(s_kk[s] < m)) continue;                      // uniform
        const bool want = c && (c & s_mask[s]) == s_prefix[s];
        const unsigned act = __ballot_sync(0xffffffffu, want);
        if (want) {
          // skewed digits (the top digit is nearly constant): one atomic per
          // distinct digit per warp
          const unsigned peers = __match_any_sync(act, d);
          if ((tid & 31) == __ffs(peers) - 1) atomicAdd(&hist[s][d], (unsigned)__popc(peers));
        }
      }
    }
    __syncthreads();
    {
      // one warp per active slot: lane l owns digits 255-8l .. 248-8l; a warp
      // scan from the top digit finds where the running count reaches `left`
      const int lane = tid & 31;
      for (int w = tid >> 5; w < nslots; w += kSelThreads / 32) {
        if (!(s_kk[w] < m)) continue;
        unsigned long long h[8], sum = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          h[i] = hist[w][255 - 8 * lane - i];
          sum += h[i];
        }
        unsigned long long inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          unsigned long long v = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += v;
        }
        const unsigned long long left = s_left[w];
        const unsigned ball = __ballot_sync(0xffffffffu, inc - sum < left && left <= inc);
        const int src = ball ? __ffs(ball) - 1 : 31;
        if (lane == src) {
          unsigned long long cum = inc - sum;
          int d = 255 - 8 * lane;
          for (int i = 0; i < 7; ++i, --d) {
            if (cum + h[i] >= left) break;
            cum += h[i];
          }
          s_left[w] = left - cum;  // still needed among bins equal on this digit
          s_prefix[w] |= (unsigned long long)d << shift;
          s_mask[w] |= 255ULL << shift;
        }
      }
    }
    __syncthreads();
  }
  // now for active slot s: threshold t = s_prefix[s]; need s_left[s] bins with
  // count == t (lowest ordinals) on top of every bin with count > t.

  // ---- auto B: coverage per B, then the Eq. 6 argmin ---------------------
  if (autob) {
    unsigned long long acc[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) acc[s] = 0;
    for (uint64_t i = tid; i < M; i += kSelThreads) {
      unsigned long long c = bv.sel_count(i);
      if (!c) continue;
#pragma unroll
      for (int s = 0; s < NS; ++s)
        if (s_kk[s] < m && c > s_prefix[s]) acc[s] += c;
    }
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      unsigned long long v = block_reduce<kSelThreads>(acc[s], SumOp(), tmp.red);
      if (tid == 0) s_cov[s] = (s_kk[s] < m) ? v + s_left[s] * s_prefix[s] : tot;
      __syncthreads();
    }
    if (cov_out) {   // select_index_length's coverage table only
      if (tid < auto_n) cov_out[tid] = s_cov[tid];
      if (tid == 0) { model->status = 0; model->k = 0; model->m_selectable = (int)(m > 0x7fffffffULL ? 0x7fffffff : m); }
      return;
    }
    if (tid == 0) {
      // size(B) = 2^B*L + n*B/8 + (n - cov)*L, evaluated exactly as 8*size in
      // integers (every term is an exact integer or a multiple of 1/8 far below
      // 2^50, so the reference's float arithmetic is exact too).
      const unsigned long long L = sizeof(T);
      int best = auto_lo;
      unsigned long long best8 = 0;
      for (int s = 0; s < auto_n; ++s) {
        int b = auto_lo + s;
        unsigned long long s8 = 8ULL * (1ULL << b) * L + (unsigned long long)n_total * b +
                                8ULL * (n_total - s_cov[s]) * L;
        if (s == 0 || s8 < best8) { best8 = s8; best = b; }
      }
      s_bits = best;
    }
    __syncthreads();
  } else if (tid == 0) {
    s_bits = bits_cfg;
  }
  __syncthreads();
  const int bits = s_bits;
  const int slot = autob ? bits - auto_lo : 0;
  const unsigned long long K = s_kk[slot];
  const bool take_all = (K >= m);
  const unsigned long long t = s_prefix[slot];
  const unsigned long long need_eq = s_left[slot];
  if (K > cap_k) {
    if (tid == 0) { model->status = NMK_ERR_ARG; model->k = (int)K; }
    return;
  }

  // ---- compaction of selected bins in ordinal order -> raw centers (cuts buf)
  unsigned long long run_eq = 0, run_pos = 0;
  for (uint64_t c0 = 0; c0 < M; c0 += kSelThreads) {
    uint64_t i = c0 + tid;
    unsigned long long c = (i < M) ? bv.sel_count(i) : 0ULL;
    unsigned eq = (!take_all && c && c == t) ? 1u : 0u;
    unsigned eq_ex, eq_tot;
    eq_ex = block_exclusive_sum<kSelThreads>(eq, eq_tot, tmp.scan);
    __syncthreads();
    bool chosen = c && (take_all || c > t || (eq && run_eq + eq_ex < need_eq));
    unsigned ch = chosen ? 1u : 0u, ch_ex, ch_tot;
    ch_ex = block_exclusive_sum<kSelThreads>(ch, ch_tot, tmp.scan);
    __syncthreads();
    if (chosen) cuts[run_pos + ch_ex] = bv.center(i);
    run_eq += eq_tot;
    run_pos += ch_tot;
  }
  __syncthreads();
  const uint64_t kraw = run_pos;  // == K

  // ---- quantise + dedupe + drop non-finite (np.unique semantics) -----------
  unsigned long long kq = 0;
  if (tid == 0) s_prev = 0.0;
  __syncthreads();
  for (uint64_t c0 = 0; c0 < kraw; c0 += kSelThreads) {
    uint64_t i = c0 + tid;
    double q = 0.0;
    bool keep = false;
    if (i < kraw) {
      q = quantize<T>(cuts[i]);
      double prevq = (i == 0) ? 0.0 : quantize<T>(cuts[i - 1]);
      keep = finite64(q) && (i == 0 || !(q == prevq) || !finite64(prevq));
    }
    unsigned kp = keep ? 1u : 0u, ex, tot2;
    ex = block_exclusive_sum<kSelThreads>(kp, tot2, tmp.scan);
    __syncthreads();
    if (keep) centers[kq + ex] = q;
    kq += tot2;
  }
  __syncthreads();
  if (kq == 0) {
    if (tid == 0) centers[0] = 0.0;
    kq = 1;
  }
  __syncthreads();
  for (uint64_t i = tid; i < kq; i += kSelThreads) {
    centers_t[i] = narrow<T>(centers[i]);
    if (i + 1 < kq) cuts[i] = __dmul_rn(0.5, __dadd_rn(centers[i], centers[i + 1]));
  }
  if (tid == 0) {
    model->bits = bits;
    model->k = (int)kq;
    model->status = 0;
    model->m_selectable = (int)(m > 0x7fffffffULL ? 0x7fffffff : m);
    model->tol_bin = width / 2.0;
    for (int b = 0; b < 17; ++b) model->coverage[b] = 0;
    model->coverage[0] = maxc;   // K2's spread hint for the next step (nmk_hist_dense_dev2)
    model->coverage[1] = second;
    if (autob)
      for (int s = 0; s < auto_n && auto_lo + s <= kAutoHi; ++s) model->coverage[auto_lo + s] = s_cov[s];
  }
}

}  // namespace nmk

using namespace nmk;

extern "C" int nmk_select(const unsigned long long* keys, const unsigned long long* counts, uint64_t m_max,
                          const unsigned long long* nruns, const nmk_stats* stats, double width,
                          double tolerance, int bits, uint64_t n_total, int dtype, double* centers,
                          double* cuts, void* centers_t, uint64_t cap_k, nmk_model* model, void* stream) {
  if (!counts || !stats || !centers || !cuts || !centers_t || !model || cap_k < 1)
    return set_error(NMK_ERR_ARG, "nmk_select: bad argument");
  if (bits >= 0 && (bits < 2 || bits > 30)) return set_error(NMK_ERR_ARG, "nmk_select: bits %d outside [2, 30]", bits);
  if (keys && !nruns) return set_error(NMK_ERR_ARG, "nmk_select: sparse form needs nruns");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t smem = (m_max == 0 && !keys) ? kSelCache * 8 : (m_max <= kSelCache ? (size_t)m_max * 8 : 0);
  ensure_dyn_smem(k_select<double, kNSel>, kSelCache * 8);
  ensure_dyn_smem(k_select<float, kNSel>, kSelCache * 8);
  if (dtype == NMK_F64)
    launch_chain(kPdlK3, k_select<double, kNSel>, 1, kSelThreads, smem, s, keys, counts, m_max, nruns, stats, width, tolerance,
                 bits, n_total, centers, cuts, (double*)centers_t, cap_k, model, kAutoLo, kNSel, nullptr);
  else if (dtype == NMK_F32)
    launch_chain(kPdlK3, k_select<float, kNSel>, 1, kSelThreads, smem, s, keys, counts, m_max, nruns, stats, width, tolerance,
                 bits, n_total, centers, cuts, (float*)centers_t, cap_k, model, kAutoLo, kNSel, nullptr);
  else
    return set_error(NMK_ERR_ARG, "nmk_select: bad dtype");
  return check_launch("k_select");
}

extern "C" int nmk_coverage(const unsigned long long* keys, const unsigned long long* counts, uint64_t m_max,
                            const unsigned long long* nruns, const nmk_stats* stats, double width, int bits_lo,
                            int bits_hi, unsigned long long* coverage, nmk_model* model, void* stream) {
  if (!counts || !stats || !coverage || !model) return set_error(NMK_ERR_ARG, "nmk_coverage: bad argument");
  if (bits_lo < 2 || bits_hi > 30 || bits_lo > bits_hi)
    return set_error(NMK_ERR_ARG, "nmk_coverage: bits range [%d, %d] outside [2, 30]", bits_lo, bits_hi);
  if (keys && !nruns) return set_error(NMK_ERR_ARG, "nmk_coverage: sparse form needs nruns");
  if (!keys && m_max == 0) return set_error(NMK_ERR_ARG, "nmk_coverage: dense form needs m_max");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t smem = m_max <= kSelCache ? (size_t)m_max * 8 : 0;
  ensure_dyn_smem(k_select<double, kNSelMax>, kSelCache * 8);
  k_select<double, kNSelMax><<<1, kSelThreads, smem, s>>>(keys, counts, m_max, nruns, stats, width, width / 2.0, -1,
                                                          0, nullptr, nullptr, nullptr, 1, model, bits_lo,
                                                          bits_hi - bits_lo + 1, coverage);
  return check_launch("k_select(coverage)");
}
