// k_sort.cu — 64-bit LSD radix sort (keys or key/value pairs) and 64-bit
// prefix sums for the sparse histogram path (k_hist.cu: spans too wide for a
// dense table -- the reference's planted-outlier case, binning.py:110-132 --
// sort the ordinals' bit patterns and run-length encode them).
//
// Eight stable passes of 8-bit digits.  Per pass:
//   k_sort_hist     a CTA counts the digits of its tile of kSortTile keys into
//                   hist[digit][tile] (digit-major, so one exclusive scan over
//                   the whole table gives every (digit, tile) its first slot);
//   chunk_scan      the look-back scan of k_scan.cu over the table;
//   k_sort_scatter  the CTA re-reads its tile in index order: every warp owns
//                   a contiguous run of it, counts its digits (one shared-memory
//                   add per distinct digit of a 32-key group, found with
//                   __match_any_sync), the 256 digit columns are scanned over
//                   the warps, and each warp then places its groups in order --
//                   a key's slot is its digit's running offset plus the number
//                   of equal digits in lower lanes of its group.
// Stability per pass makes the whole sort correct; equal keys keep their input
// order (the merge path relies on nothing more than grouping).
#include "nmk_common.cuh"
#include "nmk_scan.cuh"
#include "nmk_sort.cuh"

namespace nmk {

constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kSortPerLane = 16;                              // keys per lane: 16 groups of 32 per warp
constexpr int kSortWarpKeys = 32 * kSortPerLane;              // 512 contiguous keys per warp
constexpr int kSortTile = kSortWarps * kSortWarpKeys;         // 4096 keys per CTA
typedef unsigned long long u64;

__global__ void __launch_bounds__(kSortThreads)
k_sort_hist(const u64* __restrict__ keys, uint64_t n, int shift, uint32_t* __restrict__ hist, uint32_t ntiles) {
  __shared__ uint32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t t0 = (uint64_t)blockIdx.x * kSortTile;
  for (int j = 0; j < kSortTile / kSortThreads; ++j) {
    const uint64_t i = t0 + (uint64_t)j * kSortThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(unsigned)(keys[i] >> shift) & 255u], 1u);
  }
  __syncthreads();
  hist[(uint64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

template <bool kVals>
__global__ void __launch_bounds__(kSortThreads)
k_sort_scatter(const u64* __restrict__ keys, const u64* __restrict__ vals, uint64_t n, int shift,
               const u64* __restrict__ offsets, uint32_t ntiles, u64* __restrict__ out_keys,
               u64* __restrict__ out_vals) {
  __shared__ u64 wh[kSortWarps][256];   // per warp and digit: count, then the next output slot
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int d = lane; d < 256; d += 32) wh[w][d] = 0;
  __syncwarp();
  const uint64_t w0 = (uint64_t)blockIdx.x * kSortTile + (uint64_t)w * kSortWarpKeys;
  u64 k[kSortPerLane];
  u64 v[kVals ? kSortPerLane : 1];
#pragma unroll
  for (int g = 0; g < kSortPerLane; ++g) {
    const uint64_t i = w0 + (uint64_t)g * 32 + lane;
    k[g] = i < n ? keys[i] : 0ULL;
    if (kVals) v[g] = i < n ? vals[i] : 0ULL;
  }
  // the warp's digit counts (lanes past the end carry a digit no key has)
#pragma unroll
  for (int g = 0; g < kSortPerLane; ++g) {
    const bool in = w0 + (uint64_t)g * 32 + lane < n;
    const unsigned d = in ? (unsigned)(k[g] >> shift) & 255u : 256u + (unsigned)lane;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    if (in && lane == __ffs((int)peers) - 1) wh[w][d] += (u64)__popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {   // digit column d = threadIdx.x: first slot of every warp's keys of that digit
    const int d = threadIdx.x;
    u64 run = offsets[(uint64_t)d * ntiles + blockIdx.x];
#pragma unroll
    for (int ww = 0; ww < kSortWarps; ++ww) {
      const u64 c = wh[ww][d];
      wh[ww][d] = run;
      run += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (int g = 0; g < kSortPerLane; ++g) {   // groups in index order: stable
    const bool in = w0 + (uint64_t)g * 32 + lane < n;
    const unsigned d = in ? (unsigned)(k[g] >> shift) & 255u : 256u + (unsigned)lane;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    if (in) {
      const u64 pos = wh[w][d] + (u64)__popc(peers & ((1u << lane) - 1u));
      out_keys[pos] = k[g];
      if (kVals) out_vals[pos] = v[g];
    }
    __syncwarp();
    if (in && lane == __ffs((int)peers) - 1) wh[w][d] += (u64)__popc(peers);
    __syncwarp();
  }
}

struct SortWs {
  u64* tmp_keys;
  u64* tmp_vals;
  uint32_t* hist;
  u64* offsets;
  void* scan_ws;
  size_t total;
};

static size_t al256s(size_t x) { return (x + 255) & ~(size_t)255; }

static SortWs sort_layout(uint64_t n, bool with_vals, void* base) {
  SortWs w{};
  const uint64_t ntiles = (n + kSortTile - 1) / kSortTile;
  const uint64_t cells = 256 * (ntiles ? ntiles : 1);
  char* p = (char*)base;
  size_t off = 0;
  auto take = [&](size_t bytes) { char* q = p ? p + off : nullptr; off += al256s(bytes); return q; };
  w.tmp_keys = (u64*)take(n * 8);
  w.tmp_vals = with_vals ? (u64*)take(n * 8) : nullptr;
  w.hist = (uint32_t*)take(cells * 4);
  w.offsets = (u64*)take((cells + 1) * 8);
  w.scan_ws = take(chunk_scan_ws_bytes(cells));
  w.total = off;
  return w;
}

size_t sort64_ws_bytes(uint64_t n, bool with_vals) { return sort_layout(n, with_vals, nullptr).total; }

void sort64(const u64* keys_in, u64* keys_out, const u64* vals_in, u64* vals_out, uint64_t n, void* ws,
            cudaStream_t s) {
  if (n == 0) return;
  const bool with_vals = vals_in != nullptr;
  SortWs w = sort_layout(n, with_vals, ws);
  const uint32_t ntiles = (uint32_t)((n + kSortTile - 1) / kSortTile);
  const uint64_t cells = 256ULL * ntiles;
  const u64* src_k = keys_in;
  const u64* src_v = vals_in;
  for (int pass = 0; pass < 8; ++pass) {   // odd passes land in the outputs: the last one does
    u64* dst_k = (pass & 1) ? keys_out : w.tmp_keys;
    u64* dst_v = (pass & 1) ? vals_out : w.tmp_vals;
    const int shift = 8 * pass;
    k_sort_hist<<<ntiles, kSortThreads, 0, s>>>(src_k, n, shift, w.hist, ntiles);
    chunk_scan(w.hist, cells, w.offsets, w.scan_ws, s);
    if (with_vals)
      k_sort_scatter<true><<<ntiles, kSortThreads, 0, s>>>(src_k, src_v, n, shift, w.offsets, ntiles, dst_k, dst_v);
    else
      k_sort_scatter<false><<<ntiles, kSortThreads, 0, s>>>(src_k, nullptr, n, shift, w.offsets, ntiles, dst_k, nullptr);
    src_k = dst_k;
    src_v = dst_v;
  }
}

// ---- 64-bit prefix sums (single pass, decoupled look-back) ------------------
constexpr int kScan64Threads = 256;
constexpr int kScan64Per = 4;
constexpr int kScan64Tile = kScan64Threads * kScan64Per;

template <bool kInclusive>
__global__ void __launch_bounds__(kScan64Threads)
k_scan64(const u64* __restrict__ in, u64* __restrict__ out, uint64_t n, u64* __restrict__ status) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t i0 = (uint64_t)blockIdx.x * kScan64Tile + (uint64_t)threadIdx.x * kScan64Per;
  u64 x[kScan64Per];
  u64 sum = 0;
#pragma unroll
  for (int q = 0; q < kScan64Per; ++q) {
    x[q] = i0 + q < n ? in[i0 + q] : 0ULL;
    sum += x[q];
  }
  u64 incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u64 y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  __shared__ u64 s_w[kScan64Threads / 32];
  __shared__ u64 s_p;
  if (lane == 31) s_w[wid] = incl;
  __syncthreads();
  u64 wbase = 0, agg = 0;
#pragma unroll
  for (int ww = 0; ww < kScan64Threads / 32; ++ww) {
    const u64 t = s_w[ww];
    wbase += ww < wid ? t : 0ULL;
    agg += t;
  }
  if (wid == 0) {
    const u64 p = scan_lookback(status, blockIdx.x, agg, lane);   // sums stay below 2^62 (element counts)
    if (lane == 0) s_p = p;
  }
  __syncthreads();
  u64 run = s_p + wbase + (incl - sum);
#pragma unroll
  for (int q = 0; q < kScan64Per; ++q) {
    if (i0 + q < n) out[i0 + q] = kInclusive ? run + x[q] : run;
    run += x[q];
  }
}

size_t scan64_ws_bytes(uint64_t n) { return ((n + kScan64Tile - 1) / kScan64Tile + 1) * 8 + 256; }

void scan64(const u64* in, u64* out, uint64_t n, bool inclusive, void* ws, cudaStream_t s) {
  if (n == 0) return;
  const uint64_t ntiles = (n + kScan64Tile - 1) / kScan64Tile;
  u64* status = reinterpret_cast<u64*>(ws);
  cudaMemsetAsync(status, 0, ntiles * 8, s);
  if (inclusive) k_scan64<true><<<(unsigned)ntiles, kScan64Threads, 0, s>>>(in, out, n, status);
  else k_scan64<false><<<(unsigned)ntiles, kScan64Threads, 0, s>>>(in, out, n, status);
}

}  // namespace nmk

using namespace nmk;

extern "C" size_t nmk_sort64_ws_bytes(uint64_t n, int with_vals) { return sort64_ws_bytes(n, with_vals != 0); }

extern "C" int nmk_sort64(const unsigned long long* keys_in, unsigned long long* keys_out,
                          const unsigned long long* vals_in, unsigned long long* vals_out, uint64_t n, void* ws,
                          size_t ws_bytes, void* stream) {
  if (n == 0) return NMK_OK;
  if (!keys_in || !keys_out || !ws || (vals_in && !vals_out)) return set_error(NMK_ERR_ARG, "nmk_sort64: bad argument");
  if (keys_in == keys_out || (vals_in && vals_in == vals_out))
    return set_error(NMK_ERR_ARG, "nmk_sort64: outputs must not alias the inputs");
  if (ws_bytes < sort64_ws_bytes(n, vals_in != nullptr)) return set_error(NMK_ERR_ARG, "nmk_sort64: workspace too small");
  sort64(keys_in, keys_out, vals_in, vals_out, n, ws, (cudaStream_t)stream);
  return check_launch("nmk_sort64");
}
