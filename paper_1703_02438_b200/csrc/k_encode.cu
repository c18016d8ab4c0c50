// k_encode.cu — K4: fused classify + round-trip filter + B-bit packing +
// stable compaction of the incompressible values.
//
// One pass over both snapshots replaces phases 3a, 3b and 4a of
// compress_pair (pkg/src/nmk/pipeline.py:232-288):
//   nearest_center + compressible_mask (binning.py:287-301, 350-359),
//   _roundtrip_filter (pipeline.py:143-160), the sentinel substitution,
//   the element-order compaction current[~flags] and the per-block
//   incompressible prefix (pipeline.py:257-276), and pack_block MSB-first
//   (codec.py:83-92) into the block layout of codec.BlockLayout (codec.py:28-59).
//
// Work unit: a tile of 2048 elements = 256 threads x 8 consecutive elements,
// laid on the grid of index blocks (tiles never straddle a block), so each
// thread's 8 codes occupy exactly B whole bytes of its block.  Tiles are
// claimed in order through an atomic ticket; the running incompressible count
// is carried across tiles with a decoupled look-back (single pass, no second
// read of the inputs).  The packed bytes of a tile are staged in shared
// memory and written out with 16-byte stores before the look-back wait.
#include <cub/block/block_scan.cuh>

#include "nmk_common.cuh"

namespace nmk {

constexpr int kSmemCenters = 2048;  // centers + cuts in smem up to this k

template <int B>
__device__ __forceinline__ void pack8(const uint32_t (&code)[kGroup], uint8_t* dst) {
  // MSB-first bit string of 8 codes = B bytes; B is a compile-time constant
  // so every shift below resolves statically.
  uint8_t out[B];
  unsigned long long acc = 0;
  int nacc = 0, ob = 0;
#pragma unroll
  for (int e = 0; e < kGroup; ++e) {
    acc = (acc << B) | code[e];
    nacc += B;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (nacc >= 8) {
        out[ob++] = (uint8_t)(acc >> (nacc - 8));
        nacc -= 8;
      }
    }
  }
  // widest aligned store the byte offset tid*B allows
  if constexpr (B % 16 == 0) {
#pragma unroll
    for (int w = 0; w < B / 16; ++w) {
      uint4 v;
      uint32_t* p = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        p[q] = out[w * 16 + q * 4] | (out[w * 16 + q * 4 + 1] << 8) | (out[w * 16 + q * 4 + 2] << 16) |
               ((uint32_t)out[w * 16 + q * 4 + 3] << 24);
      reinterpret_cast<uint4*>(dst)[w] = v;
    }
  } else if constexpr (B % 8 == 0) {
#pragma unroll
    for (int w = 0; w < B / 8; ++w) {
      uint2 v;
      v.x = out[w * 8] | (out[w * 8 + 1] << 8) | (out[w * 8 + 2] << 16) | ((uint32_t)out[w * 8 + 3] << 24);
      v.y = out[w * 8 + 4] | (out[w * 8 + 5] << 8) | (out[w * 8 + 6] << 16) | ((uint32_t)out[w * 8 + 7] << 24);
      reinterpret_cast<uint2*>(dst)[w] = v;
    }
  } else if constexpr (B % 4 == 0) {
#pragma unroll
    for (int w = 0; w < B / 4; ++w)
      reinterpret_cast<uint32_t*>(dst)[w] =
          out[w * 4] | (out[w * 4 + 1] << 8) | (out[w * 4 + 2] << 16) | ((uint32_t)out[w * 4 + 3] << 24);
  } else if constexpr (B % 2 == 0) {
#pragma unroll
    for (int w = 0; w < B / 2; ++w)
      reinterpret_cast<uint16_t*>(dst)[w] = (uint16_t)(out[w * 2] | (out[w * 2 + 1] << 8));
  } else {
#pragma unroll
    for (int w = 0; w < B; ++w) dst[w] = out[w];
  }
}

template <typename T> struct EVec;
template <> struct EVec<double> { using V = double2; static constexpr int N = 2; };
template <> struct EVec<float>  { using V = float4;  static constexpr int N = 4; };

template <typename T>
__device__ __forceinline__ void load_group(const T* __restrict__ p, bool vec, int ne, T (&v)[kGroup]) {
  using V = typename EVec<T>::V;
  constexpr int VN = EVec<T>::N;
  if (vec) {
#pragma unroll
    for (int q = 0; q < kGroup / VN; ++q) {
      V w = __ldg(reinterpret_cast<const V*>(p) + q);
      const T* t = reinterpret_cast<const T*>(&w);
#pragma unroll
      for (int e = 0; e < VN; ++e) v[q * VN + e] = t[e];
    }
  } else {
#pragma unroll
    for (int e = 0; e < kGroup; ++e) v[e] = (e < ne) ? __ldg(p + e) : T(0);
  }
}

struct EncodeGeom {
  uint64_t n_local, elem0, n_total, epb, tpb, g0, ntiles, b0, stride;
};

template <typename T, int B>
__global__ void __launch_bounds__(kTileThreads)
k_encode(const T* __restrict__ base, const T* __restrict__ cur, EncodeGeom geo,
         const double* __restrict__ centers_g, const double* __restrict__ cuts_g, int k,
         double tol_bin, double tol, uint8_t* __restrict__ packed, T* __restrict__ exact,
         unsigned long long* __restrict__ prefix, unsigned long long* __restrict__ n_inc,
         unsigned long long* __restrict__ status, unsigned int* __restrict__ ticket) {
  typedef cub::BlockScan<unsigned, kTileThreads> BScan;
  __shared__ typename BScan::TempStorage scan_tmp;
  __shared__ __align__(16) uint8_t tile_bytes[kTileThreads * B + 16];
  __shared__ unsigned long long s_tile, s_excl;
  extern __shared__ double smc[];

  const int tid = threadIdx.x;
  const bool in_smem = k <= kSmemCenters;
  const double* C = centers_g;
  const double* X = cuts_g;
  if (in_smem) {
    for (int i = tid; i < k; i += kTileThreads) smc[i] = centers_g[i];
    for (int i = tid; i < k - 1; i += kTileThreads) smc[kSmemCenters + i] = cuts_g[i];
    C = smc;
    X = smc + kSmemCenters;
  }
  const uint32_t sentinel = (1u << B) - 1u;
  const uint64_t local_end = geo.elem0 + geo.n_local;

  for (;;) {
    if (tid == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint64_t t = s_tile;
    if (t >= geo.ntiles) break;
    const uint64_t g = geo.g0 + t;
    const uint64_t b = g / geo.tpb, ti = g % geo.tpb;
    const uint64_t blk_start = b * geo.epb;
    uint64_t blk_end = blk_start + geo.epb;
    if (blk_end > geo.n_total) blk_end = geo.n_total;
    const uint64_t tile_lo = blk_start + ti * kTile;
    const uint64_t grp_lo = tile_lo + (uint64_t)tid * kGroup;
    // elements of this group inside [elem0, local_end) and inside the block
    uint64_t hi = blk_end < local_end ? blk_end : local_end;
    uint64_t lo = geo.elem0;
    uint32_t code[kGroup];
    unsigned inc_mask = 0;
    T xv[kGroup];
    {
      T bv[kGroup];
      bool full = grp_lo >= lo && grp_lo + kGroup <= hi;
      int ne = 0;
      uint64_t first = grp_lo;
      if (full) {
        ne = kGroup;
      } else if (grp_lo + kGroup > lo && grp_lo < hi) {
        // partial group: clamp to [lo, hi); out-of-range lanes get code 0
        ne = -1;
      }
      if (ne == kGroup) {
        const uint64_t li = first - geo.elem0;
        constexpr int VN = EVec<T>::N;
        bool vec = (li % VN == 0) && ((((uintptr_t)base | (uintptr_t)cur) & 15) == 0);
        load_group<T>(base + li, vec, kGroup, bv);
        load_group<T>(cur + li, vec, kGroup, xv);
      } else {
#pragma unroll
        for (int e = 0; e < kGroup; ++e) {
          uint64_t j = grp_lo + e;
          bool in = (ne != 0) && j >= lo && j < hi;
          bv[e] = in ? __ldg(base + (j - geo.elem0)) : T(0);
          xv[e] = in ? __ldg(cur + (j - geo.elem0)) : T(0);
        }
      }
#pragma unroll
      for (int e = 0; e < kGroup; ++e) {
        uint64_t j = grp_lo + e;
        bool in = (ne == kGroup) || (ne != 0 && j >= lo && j < hi);
        code[e] = 0;
        if (!in) continue;
        double bd = to_f64(bv[e]), xd = to_f64(xv[e]);
        bool valid;
        double r = change_ratio(bd, xd, valid);
        uint32_t idx = lower_bound_cuts(X, k - 1, r);
        double c = C[idx];
        bool flag = valid && (fabs(__dsub_rn(r, c)) <= tol_bin);
        if (flag) flag = roundtrip_ok<T>(c, bd, xd, tol);
        code[e] = flag ? idx : sentinel;
        if (!flag) inc_mask |= 1u << e;
      }
    }
    unsigned cnt = __popc(inc_mask), ex, agg;
    BScan(scan_tmp).ExclusiveSum(cnt, ex, agg);
    if (tid == 0) st_relaxed(status + t, (t == 0 ? kFlagInc : kFlagAgg) | agg);
    pack8<B>(code, tile_bytes + tid * B);
    __syncthreads();
    // copy-out, clipped to this block's packed length
    {
      const uint64_t blk_bytes = ((blk_end - blk_start) * B + 7) / 8;
      const uint64_t off = ti * (uint64_t)(kTileThreads * B);
      uint64_t nbytes = blk_bytes > off ? blk_bytes - off : 0;
      if (nbytes > (uint64_t)kTileThreads * B) nbytes = (uint64_t)kTileThreads * B;
      uint8_t* dst = packed + (b - geo.b0) * geo.stride + off;
      const uint32_t nvec = (uint32_t)(nbytes / 16);
      for (uint32_t i = tid; i < nvec; i += kTileThreads)
        reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(tile_bytes)[i];
      for (uint32_t i = nvec * 16 + tid; i < nbytes; i += kTileThreads) dst[i] = tile_bytes[i];
    }
    // look-back for the running incompressible count
    if (tid < 32) {
      unsigned long long excl = (t == 0) ? 0ULL : lookback(status, (long long)t, 0);
      if (tid == 0) {
        if (t != 0) st_relaxed(status + t, kFlagInc | (excl + agg));
        s_excl = excl;
      }
    }
    __syncthreads();
    const unsigned long long excl = s_excl;
    if (inc_mask) {
      unsigned long long pos = excl + ex;
#pragma unroll
      for (int e = 0; e < kGroup; ++e)
        if (inc_mask >> e & 1u) exact[pos++] = xv[e];   // raw bits (NaN payloads kept)
    }
    if (tid == 0) {
      if (ti == 0 && blk_start >= geo.elem0) prefix[b - geo.b0] = excl;
      if (t == geo.ntiles - 1) *n_inc = excl + agg;
    }
    // next iteration's ticket write to s_tile is ordered by its __syncthreads
  }
}

// ---- standalone pack/unpack (codec.pack_block / unpack_block) -------------
template <int B>
__device__ __forceinline__ void unpack8(const uint8_t* src, uint32_t (&code)[kGroup]) {
  unsigned long long acc = 0;
  int nacc = 0, bi = 0;
#pragma unroll
  for (int e = 0; e < kGroup; ++e) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (nacc < B) {
        acc = (acc << 8) | src[bi++];
        nacc += 8;
      }
    }
    code[e] = (uint32_t)(acc >> (nacc - B)) & ((1u << B) - 1u);
    nacc -= B;
  }
}

template <int B>
__global__ void k_pack(const uint32_t* __restrict__ codes, uint64_t n, uint8_t* __restrict__ out) {
  const uint64_t ngrp = (n + kGroup - 1) / kGroup;
  const uint64_t nbytes = (n * B + 7) / 8;
  for (uint64_t gi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < ngrp;
       gi += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t c[kGroup];
#pragma unroll
    for (int e = 0; e < kGroup; ++e) {
      uint64_t j = gi * kGroup + e;
      c[e] = j < n ? codes[j] : 0u;
    }
    uint8_t tmp[B + 16];
    uint8_t* al = reinterpret_cast<uint8_t*>(((uintptr_t)tmp + 15) & ~(uintptr_t)15);
    pack8<B>(c, al);
#pragma unroll
    for (int w = 0; w < B; ++w) {
      uint64_t o = gi * B + w;
      if (o < nbytes) out[o] = al[w];
    }
  }
}

template <int B>
__global__ void k_unpack(const uint8_t* __restrict__ in, uint64_t n, uint32_t* __restrict__ codes) {
  const uint64_t ngrp = (n + kGroup - 1) / kGroup;
  const uint64_t nbytes = (n * B + 7) / 8;
  for (uint64_t gi = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; gi < ngrp;
       gi += (uint64_t)gridDim.x * blockDim.x) {
    uint8_t tmp[B];
#pragma unroll
    for (int w = 0; w < B; ++w) {
      uint64_t o = gi * B + w;
      tmp[w] = o < nbytes ? in[o] : 0;
    }
    uint32_t c[kGroup];
    unpack8<B>(tmp, c);
#pragma unroll
    for (int e = 0; e < kGroup; ++e) {
      uint64_t j = gi * kGroup + e;
      if (j < n) codes[j] = c[e];
    }
  }
}

static int sm_count_e() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

struct EncodeTiles {
  uint64_t b0, tpb, g0, ntiles;
};

static EncodeTiles encode_tiles(uint64_t n_local, uint64_t elem0, uint64_t epb) {
  EncodeTiles et{};
  if (n_local == 0 || epb == 0) return et;
  et.tpb = (epb + kTile - 1) / kTile;
  uint64_t last = elem0 + n_local - 1;
  uint64_t b0 = elem0 / epb, b1 = last / epb;
  uint64_t t0 = (elem0 - b0 * epb) / kTile, t1 = (last - b1 * epb) / kTile;
  et.b0 = b0;
  et.g0 = b0 * et.tpb + t0;
  et.ntiles = (b1 * et.tpb + t1) - et.g0 + 1;
  return et;
}

template <typename T, int B>
static void launch_encode(const void* base, const void* cur, const EncodeGeom& geo, const double* centers,
                          const double* cuts, int k, double tol_bin, double tol, uint8_t* packed, void* exact,
                          unsigned long long* prefix, unsigned long long* n_inc, unsigned long long* status,
                          unsigned* ticket, cudaStream_t s) {
  size_t smem = (k <= kSmemCenters) ? 2 * kSmemCenters * sizeof(double) : 0;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_encode<T, B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(2 * kSmemCenters * sizeof(double)));
    attr_set = true;
  }
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_encode<T, B>, kTileThreads, smem);
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = (uint64_t)sm_count_e() * per_sm;
  if (grid > geo.ntiles) grid = geo.ntiles;
  k_encode<T, B><<<(unsigned)grid, kTileThreads, smem, s>>>((const T*)base, (const T*)cur, geo, centers, cuts, k,
                                                            tol_bin, tol, packed, (T*)exact, prefix, n_inc,
                                                            status, ticket);
}

template <typename T>
static int dispatch_encode(int bits, const void* base, const void* cur, const EncodeGeom& geo, const double* centers,
                           const double* cuts, int k, double tol_bin, double tol, uint8_t* packed, void* exact,
                           unsigned long long* prefix, unsigned long long* n_inc, unsigned long long* status,
                           unsigned* ticket, cudaStream_t s) {
  switch (bits) {
#define NMK_ENC_CASE(BB) \
  case BB: launch_encode<T, BB>(base, cur, geo, centers, cuts, k, tol_bin, tol, packed, exact, prefix, n_inc, status, ticket, s); break;
    NMK_ENC_CASE(2) NMK_ENC_CASE(3) NMK_ENC_CASE(4) NMK_ENC_CASE(5) NMK_ENC_CASE(6) NMK_ENC_CASE(7)
    NMK_ENC_CASE(8) NMK_ENC_CASE(9) NMK_ENC_CASE(10) NMK_ENC_CASE(11) NMK_ENC_CASE(12) NMK_ENC_CASE(13)
    NMK_ENC_CASE(14) NMK_ENC_CASE(15) NMK_ENC_CASE(16) NMK_ENC_CASE(17) NMK_ENC_CASE(18) NMK_ENC_CASE(19)
    NMK_ENC_CASE(20) NMK_ENC_CASE(21) NMK_ENC_CASE(22) NMK_ENC_CASE(23) NMK_ENC_CASE(24) NMK_ENC_CASE(25)
    NMK_ENC_CASE(26) NMK_ENC_CASE(27) NMK_ENC_CASE(28) NMK_ENC_CASE(29) NMK_ENC_CASE(30)
#undef NMK_ENC_CASE
    default: return set_error(NMK_ERR_ARG, "nmk_encode: bits %d outside [2, 30]", bits);
  }
  return check_launch("k_encode");
}

}  // namespace nmk

using namespace nmk;

extern "C" size_t nmk_encode_ws_bytes(uint64_t n_local, uint64_t elem0, uint64_t epb) {
  EncodeTiles et = encode_tiles(n_local, elem0, epb);
  return 256 + (size_t)(et.ntiles + 1) * sizeof(unsigned long long);
}

extern "C" int nmk_encode(const void* base, const void* cur, uint64_t n_local, uint64_t elem0, uint64_t n_total,
                          int dtype, const double* centers, const double* cuts, int k, int bits, double tol_bin,
                          double tolerance, uint64_t epb, uint8_t* packed, uint64_t block_stride, void* exact,
                          unsigned long long* prefix, unsigned long long* n_inc, void* ws, size_t ws_bytes,
                          void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n_local == 0) {
    cudaMemsetAsync(n_inc, 0, sizeof(unsigned long long), s);
    return check_launch("nmk_encode(empty)");
  }
  if (!base || !cur || !centers || !packed || !exact || !prefix || !n_inc || !ws || k < 1)
    return set_error(NMK_ERR_ARG, "nmk_encode: bad argument");
  if (k > 1 && !cuts) return set_error(NMK_ERR_ARG, "nmk_encode: cuts required for k > 1");
  if (bits < 2 || bits > 30) return set_error(NMK_ERR_ARG, "nmk_encode: bits %d outside [2, 30]", bits);
  if ((uint64_t)k > (1ULL << bits) - 1) return set_error(NMK_ERR_ARG, "nmk_encode: k %d exceeds 2^B-1", k);
  if (epb == 0 || elem0 + n_local > n_total) return set_error(NMK_ERR_ARG, "nmk_encode: bad geometry");
  if (block_stride % 16 || block_stride < (epb * bits + 7) / 8)
    return set_error(NMK_ERR_ARG, "nmk_encode: block_stride must be >= ceil(epb*B/8) and a multiple of 16");
  if ((uintptr_t)packed & 15) return set_error(NMK_ERR_ARG, "nmk_encode: packed must be 16-byte aligned");
  if (ws_bytes < nmk_encode_ws_bytes(n_local, elem0, epb)) return set_error(NMK_ERR_ARG, "nmk_encode: workspace too small");
  EncodeTiles et = encode_tiles(n_local, elem0, epb);
  EncodeGeom geo{n_local, elem0, n_total, epb, et.tpb, et.g0, et.ntiles, et.b0, block_stride};
  unsigned* ticket = (unsigned*)ws;
  unsigned long long* status = (unsigned long long*)((char*)ws + 256);
  cudaMemsetAsync(ws, 0, nmk_encode_ws_bytes(n_local, elem0, epb), s);
  // A range starting inside a block: zero the packed bytes of the tiles in
  // front of it so they decode as non-sentinel codes and OR-merge neutrally.
  const uint64_t t0_in_blk = (elem0 - et.b0 * epb) / kTile;
  if (t0_in_blk) cudaMemsetAsync(packed, 0, t0_in_blk * (uint64_t)kTileThreads * bits, s);
  if (dtype == NMK_F64)
    return dispatch_encode<double>(bits, base, cur, geo, centers, cuts, k, tol_bin, tolerance, packed, exact, prefix,
                                   n_inc, status, ticket, s);
  if (dtype == NMK_F32)
    return dispatch_encode<float>(bits, base, cur, geo, centers, cuts, k, tol_bin, tolerance, packed, exact, prefix,
                                  n_inc, status, ticket, s);
  return set_error(NMK_ERR_ARG, "nmk_encode: bad dtype");
}

template <int B>
static void launch_pack(const uint32_t* codes, uint64_t n, uint8_t* out, uint8_t* unused, cudaStream_t s, bool unpack,
                        const uint8_t* in, uint32_t* codes_out) {
  uint64_t ngrp = (n + kGroup - 1) / kGroup;
  unsigned grid = (unsigned)((ngrp + 255) / 256);
  if (grid > 4096) grid = 4096;
  if (grid == 0) grid = 1;
  if (unpack) k_unpack<B><<<grid, 256, 0, s>>>(in, n, codes_out);
  else k_pack<B><<<grid, 256, 0, s>>>(codes, n, out);
}

static int dispatch_pack(int bits, bool unpack, const uint32_t* codes, uint64_t n, uint8_t* out, const uint8_t* in,
                         uint32_t* codes_out, cudaStream_t s) {
  switch (bits) {
#define NMK_PK_CASE(BB) case BB: launch_pack<BB>(codes, n, out, nullptr, s, unpack, in, codes_out); break;
    NMK_PK_CASE(2) NMK_PK_CASE(3) NMK_PK_CASE(4) NMK_PK_CASE(5) NMK_PK_CASE(6) NMK_PK_CASE(7) NMK_PK_CASE(8)
    NMK_PK_CASE(9) NMK_PK_CASE(10) NMK_PK_CASE(11) NMK_PK_CASE(12) NMK_PK_CASE(13) NMK_PK_CASE(14)
    NMK_PK_CASE(15) NMK_PK_CASE(16) NMK_PK_CASE(17) NMK_PK_CASE(18) NMK_PK_CASE(19) NMK_PK_CASE(20)
    NMK_PK_CASE(21) NMK_PK_CASE(22) NMK_PK_CASE(23) NMK_PK_CASE(24) NMK_PK_CASE(25) NMK_PK_CASE(26)
    NMK_PK_CASE(27) NMK_PK_CASE(28) NMK_PK_CASE(29) NMK_PK_CASE(30)
#undef NMK_PK_CASE
    default: return set_error(NMK_ERR_ARG, "bits %d outside [2, 30]", bits);
  }
  return check_launch(unpack ? "k_unpack" : "k_pack");
}

extern "C" int nmk_pack(const uint32_t* codes, uint64_t n, int bits, uint8_t* out, void* stream) {
  if (n == 0) return NMK_OK;
  if (!codes || !out) return set_error(NMK_ERR_ARG, "nmk_pack: null pointer");
  return dispatch_pack(bits, false, codes, n, out, nullptr, nullptr, (cudaStream_t)stream);
}

extern "C" int nmk_unpack(const uint8_t* packed, uint64_t n, int bits, uint32_t* codes, void* stream) {
  if (n == 0) return NMK_OK;
  if (!packed || !codes) return set_error(NMK_ERR_ARG, "nmk_unpack: null pointer");
  return dispatch_pack(bits, true, nullptr, n, nullptr, packed, codes, (cudaStream_t)stream);
}
