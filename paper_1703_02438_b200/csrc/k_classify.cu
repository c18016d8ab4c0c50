// k_classify.cu — nearest-center assignment and the compressibility mask on
// ratio arrays: the binning-level API behind binning.nearest_center and
// binning.compressible_mask (pkg/src/nmk/binning.py:287-301,350-359).
//
// The fused encoder (K4) classifies straight from the snapshots; these
// kernels serve callers that already hold a ratio array (the reference's
// binning functions and its tests).  Semantics, element by element:
//   cuts[i] = RN(0.5 * RN(c[i] + c[i+1]))                  (binning.py:299)
//   idx     = #{i : cuts[i] < v}, NaN -> len(cuts)          (searchsorted 'left',
//             numpy orders NaN after every number)         (binning.py:300)
//   k == 1  -> idx = 0                                      (binning.py:296-297)
//   dist    = |RN(v - c[idx])|                               (binning.py:301)
//   flag    = valid && dist <= tol                           (binning.py:358)
#include "nmk_common.cuh"

namespace nmk {

__device__ __forceinline__ double cut_at(const double* __restrict__ c, int i) {
  return __dmul_rn(0.5, __dadd_rn(__ldg(c + i), __ldg(c + i + 1)));
}

__device__ __forceinline__ int nearest_idx(double v, const double* __restrict__ c, int k) {
  if (k <= 1) return 0;
  if (v != v) return k - 1;
  int lo = 0, hi = k - 1;   // lower bound over the k-1 cuts
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (cut_at(c, mid) < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(256)
k_nearest(const double* __restrict__ v, uint64_t n, const double* __restrict__ c, int k,
          long long* __restrict__ idx, double* __restrict__ dist, const uint8_t* __restrict__ valid, double tol,
          uint8_t* __restrict__ flags) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
    const double x = v[j];
    const int i = nearest_idx(x, c, k);
    const double d = fabs(__dsub_rn(x, __ldg(c + i)));
    idx[j] = i;
    if (dist) dist[j] = d;
    if (flags) flags[j] = (valid ? valid[j] != 0 : true) && d <= tol;
  }
}

}  // namespace nmk

using namespace nmk;

static unsigned classify_grid(uint64_t n) {
  uint64_t g = (n + 255) / 256;
  const uint64_t cap = (uint64_t)sm_count() * 8;
  return (unsigned)(g < cap ? (g ? g : 1) : cap);
}

extern "C" int nmk_nearest_center(const double* values, uint64_t n, const double* centers, int k, long long* idx,
                                  double* dist, void* stream) {
  if (n == 0) return NMK_OK;
  if (!values || !centers || !idx || k < 1) return set_error(NMK_ERR_ARG, "nmk_nearest_center: bad argument");
  k_nearest<<<classify_grid(n), 256, 0, (cudaStream_t)stream>>>(values, n, centers, k, idx, dist, nullptr, 0.0,
                                                                 nullptr);
  return check_launch("k_nearest");
}

extern "C" int nmk_compressible_mask(const double* ratios, const uint8_t* valid, uint64_t n, const double* centers,
                                     int k, double tolerance, uint8_t* flags, long long* idx, void* stream) {
  if (n == 0) return NMK_OK;
  if (!ratios || !valid || !centers || !flags || !idx || k < 1)
    return set_error(NMK_ERR_ARG, "nmk_compressible_mask: bad argument");
  k_nearest<<<classify_grid(n), 256, 0, (cudaStream_t)stream>>>(ratios, n, centers, k, idx, nullptr, valid,
                                                                 tolerance, flags);
  return check_launch("k_nearest");
}
