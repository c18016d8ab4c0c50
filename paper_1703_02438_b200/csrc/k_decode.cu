// k_decode.cu — K5: fused unpack + sentinel rank + reconstruct, batched over
// element ranges ("segments").
//
// Replaces, for full and partial decompression, the per-block loop of
// codec._decode_range (pkg/src/nmk/codec.py:204-239): unpack_block
// (codec.py:95-105), the seek into the incompressible table
// (inc_before = prefix[first] + #sentinels ahead, codec.py:231-236) and
// core.reconstruct (core.py:158-208): sentinel -> next exact value (raw
// bits), otherwise T((1 + c[idx]) * f64(base)); ids in [k, sentinel) are an
// error, as is running out of exact values.
//
// Chunks are the encoder's 256-element warp chunks on the block grid.
//   1. k_dec_count: sentinels per chunk of the covering span (reads the
//      packed stream only, B/8 bytes per element);
//   2. chunk_scan (k_scan.cu): chunk offsets;
//   3. k_dec_chunks: one warp per (segment, chunk): unpack, rank the
//      sentinels (block prefix + in-block chunk offset + warp scan), gather
//      exact values, reconstruct, store.  No inter-warp dependency.
#include "nmk_common.cuh"
#include "nmk_scan.cuh"

namespace nmk {

constexpr int kDChunk = 32 * kGroup;   // 256 elements per warp chunk
constexpr int kDecThreads = 256;

struct Seg {
  uint64_t start, count, out;   // global element range, output offset
  uint64_t item0;               // first work item (linear across segments)
  uint64_t gfirst;              // global chunk id of the segment's first chunk
};

struct DecodeGeom {
  uint64_t epb, cpb, n_total, first_block, stride, n_exact, nchunks, nitems;
  int nseg, k;
};

struct DChunk {
  uint64_t b, ci, blk_start, blk_end, chunk_lo, chunk_hi, crel;
};

__device__ __forceinline__ DChunk dchunk(const DecodeGeom& geo, uint64_t g) {
  DChunk d;
  d.b = g / geo.cpb;
  d.ci = g - d.b * geo.cpb;
  d.blk_start = d.b * geo.epb;
  d.blk_end = d.blk_start + geo.epb;
  if (d.blk_end > geo.n_total) d.blk_end = geo.n_total;
  d.chunk_lo = d.blk_start + d.ci * kDChunk;
  d.chunk_hi = d.chunk_lo + kDChunk;
  if (d.chunk_hi > d.blk_end) d.chunk_hi = d.blk_end;
  d.crel = g - geo.first_block * geo.cpb;
  return d;
}

// Packed-byte span of a chunk: base pointer and valid byte count (bytes at
// or beyond it are padding and decode as zero bits).
struct ChunkBytes {
  const uint8_t* src;
  uint32_t nbytes;
};

template <int B>
__device__ __forceinline__ ChunkBytes chunk_bytes(const uint8_t* __restrict__ packed, const DecodeGeom& geo,
                                                  const DChunk& d) {
  const uint64_t blk_bytes = ((d.blk_end - d.blk_start) * B + 7) / 8;
  const uint64_t off = d.ci * (uint64_t)(32 * B);
  uint64_t nbytes = blk_bytes > off ? blk_bytes - off : 0;
  if (nbytes > (uint64_t)(32 * B)) nbytes = 32 * B;
  return ChunkBytes{packed + (d.b - geo.first_block) * geo.stride + off, (uint32_t)nbytes};
}

// This lane's B bytes (offset lane*B of a 16-byte aligned chunk) with the
// widest aligned loads B allows; the chunk's last lanes may be clipped.
template <int B>
__device__ __forceinline__ void lane_bytes(const ChunkBytes& cb, int lane, uint8_t (&o)[B]) {
  const uint32_t s0 = (uint32_t)lane * B;
  constexpr int W = (B % 8 == 0) ? 8 : (B % 4 == 0) ? 4 : (B % 2 == 0) ? 2 : 1;
  if (s0 + B <= cb.nbytes) {
#pragma unroll
    for (int w = 0; w < B / W; ++w) {
      const uint8_t* p = cb.src + s0 + w * W;
      unsigned long long v;
      if constexpr (W == 8) v = __ldg(reinterpret_cast<const unsigned long long*>(p));
      else if constexpr (W == 4) v = __ldg(reinterpret_cast<const unsigned int*>(p));
      else if constexpr (W == 2) v = __ldg(reinterpret_cast<const unsigned short*>(p));
      else v = __ldg(p);
#pragma unroll
      for (int i = 0; i < W; ++i) o[w * W + i] = (uint8_t)(v >> (8 * i));
    }
  } else {
#pragma unroll
    for (int i = 0; i < B; ++i) o[i] = (s0 + i < cb.nbytes) ? __ldg(cb.src + s0 + i) : (uint8_t)0;
  }
}

template <int B>
__device__ __forceinline__ void codes_of(const uint8_t (&src)[B], uint32_t (&code)[kGroup]) {
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
__global__ void __launch_bounds__(kDecThreads)
k_dec_count(const uint8_t* __restrict__ packed, DecodeGeom geo, uint32_t* __restrict__ counts) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t sentinel = (1u << B) - 1u;
  const uint64_t nwarps = (uint64_t)gridDim.x * (kDecThreads / 32);
  const uint64_t g0 = geo.first_block * geo.cpb;
  for (uint64_t c = (uint64_t)blockIdx.x * (kDecThreads / 32) + wid; c < geo.nchunks; c += nwarps) {
    const DChunk d = dchunk(geo, g0 + c);
    uint8_t raw[B];
    lane_bytes<B>(chunk_bytes<B>(packed, geo, d), lane, raw);
    uint32_t code[kGroup];
    codes_of<B>(raw, code);
    const uint64_t grp_lo = d.chunk_lo + (uint64_t)lane * kGroup;
    unsigned n = 0;
#pragma unroll
    for (int e = 0; e < kGroup; ++e) n += (grp_lo + e < d.chunk_hi && code[e] == sentinel);
    n = __reduce_add_sync(0xffffffffu, n);
    if (lane == 0) counts[c] = n;
  }
}

template <typename T> struct DVec;
template <> struct DVec<double> { using V = double2; static constexpr int N = 2; };
template <> struct DVec<float>  { using V = float4;  static constexpr int N = 4; };

template <typename T, int B>
__global__ void __launch_bounds__(kDecThreads, 3)
k_dec_chunks(const uint8_t* __restrict__ packed, DecodeGeom geo, const Seg* __restrict__ segs,
             const unsigned long long* __restrict__ offsets, const unsigned long long* __restrict__ prefix_rel,
             const double* __restrict__ centers_g, const T* __restrict__ exact, const T* __restrict__ base,
             T* __restrict__ out, nmk_segment_info* __restrict__ info, nmk_decode_err* __restrict__ err) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int k = geo.k;
  const uint32_t sentinel = (1u << B) - 1u;
  constexpr int VN = DVec<T>::N;
  using V = typename DVec<T>::V;
  const bool out_al = (((uintptr_t)out | (uintptr_t)base) & 15) == 0;
  const uint64_t nwarps = (uint64_t)gridDim.x * (kDecThreads / 32);

  for (uint64_t it = (uint64_t)blockIdx.x * (kDecThreads / 32) + wid; it < geo.nitems; it += nwarps) {
    int lo_s = 0, hi_s = geo.nseg - 1;
    while (lo_s < hi_s) {
      int mid = (lo_s + hi_s + 1) >> 1;
      if (segs[mid].item0 <= it) lo_s = mid; else hi_s = mid - 1;
    }
    const Seg sg = segs[lo_s];
    const uint64_t g = sg.gfirst + (it - sg.item0);
    const DChunk d = dchunk(geo, g);
    const uint64_t seg_lo = sg.start, seg_hi = sg.start + sg.count;
    const uint64_t grp_lo = d.chunk_lo + (uint64_t)lane * kGroup;
    // base values first (independent of the codes), then the packed bytes
    unsigned inmask = 0;
#pragma unroll
    for (int e = 0; e < kGroup; ++e) {
      const uint64_t j = grp_lo + e;
      if (j < d.chunk_hi && j >= seg_lo && j < seg_hi) inmask |= 1u << e;
    }
    T bv[kGroup], ov[kGroup];
    const int64_t oi = (int64_t)sg.out + ((int64_t)grp_lo - (int64_t)seg_lo);
    const bool vec = inmask == 0xffu && out_al && (oi % VN) == 0;
    if (vec) {
#pragma unroll
      for (int q = 0; q < kGroup / VN; ++q) {
        V w = __ldg(reinterpret_cast<const V*>(base + oi) + q);
        const T* tw = reinterpret_cast<const T*>(&w);
#pragma unroll
        for (int e = 0; e < VN; ++e) bv[q * VN + e] = tw[e];
      }
    } else {
#pragma unroll
      for (int e = 0; e < kGroup; ++e) bv[e] = (inmask >> e & 1u) ? __ldg(base + (oi + e)) : T(0);
    }
    uint8_t raw[B];
    lane_bytes<B>(chunk_bytes<B>(packed, geo, d), lane, raw);
    uint32_t code[kGroup];
    codes_of<B>(raw, code);
    unsigned smask = 0, ahead = 0;
#pragma unroll
    for (int e = 0; e < kGroup; ++e) {
      const uint64_t j = grp_lo + e;
      if (j < d.chunk_hi && code[e] == sentinel) {
        smask |= 1u << e;
        if (j < seg_lo) ++ahead;
      }
    }
    // rank of this lane's first sentinel, anchored like the reference on the
    // prefix entry of the segment's FIRST block and counted from there
    // (codec.py:231-236): prefix + chunk offset + warp exclusive scan
    const uint64_t ab = sg.gfirst / geo.cpb - geo.first_block;
    const unsigned long long chunk_off = prefix_rel[ab] + (offsets[d.crel] - offsets[ab * geo.cpb]);
    const unsigned cnt = __popc(smask);
    unsigned incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    unsigned long long pos = chunk_off + (incl - cnt);
    unsigned bad = 0, maxbad = 0, exhausted = 0;
#pragma unroll
    for (int e = 0; e < kGroup; ++e) {
      ov[e] = T(0);
      if (smask >> e & 1u) {
        if (inmask >> e & 1u) {
          if (pos < geo.n_exact) ov[e] = exact[pos];
          else exhausted = 1;
        }
        ++pos;
      } else if (inmask >> e & 1u) {
        if (code[e] >= (uint32_t)k) {
          bad = 1;
          maxbad = code[e] > maxbad ? code[e] : maxbad;
        } else {
          ov[e] = apply_center<T>(__ldg(centers_g + code[e]), to_f64(bv[e]));   // L1-resident table
        }
      }
    }
    if (vec) {
#pragma unroll
      for (int q = 0; q < kGroup / VN; ++q)
        reinterpret_cast<V*>(out + oi)[q] = *reinterpret_cast<const V*>(&ov[q * VN]);
    } else {
#pragma unroll
      for (int e = 0; e < kGroup; ++e)
        if (inmask >> e & 1u) out[oi + e] = ov[e];
    }
    if (bad) {
      atomicOr(&err->bad_index, 1u);
      atomicMax(&err->max_bad_index, maxbad);
    }
    if (exhausted) atomicOr(&err->exhausted, 1u);
    // segment bookkeeping
    const unsigned in_s = __reduce_add_sync(0xffffffffu, __popc(smask & inmask));
    if (lane == 0 && in_s) atomicAdd(&info[lo_s].n_sentinel, (unsigned long long)in_s);
    if (g == sg.gfirst) {
      const unsigned ah = __reduce_add_sync(0xffffffffu, ahead);
      if (lane == 0) info[lo_s].inc_before = chunk_off + ah;
    }
    __syncwarp();
  }
}

static int sm_count_d() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

struct DecodePlan {
  uint64_t cpb, nchunks, nitems;
  size_t off_counts, off_offsets, off_scan, off_segs, total;
};

static DecodePlan decode_plan(const uint64_t* st, const uint64_t* ct, int nseg, uint64_t epb, uint64_t first_block) {
  DecodePlan p{};
  p.cpb = (epb + kDChunk - 1) / kDChunk;
  uint64_t items = 0, last = 0;
  const uint64_t g0 = first_block * p.cpb;
  for (int s = 0; s < nseg; ++s) {
    if (ct[s] == 0) continue;
    uint64_t e = st[s] + ct[s] - 1;
    uint64_t ga = (st[s] / epb) * p.cpb + (st[s] % epb) / kDChunk;
    uint64_t gz = (e / epb) * p.cpb + (e % epb) / kDChunk;
    items += gz - ga + 1;
    if (gz + 1 - g0 > last) last = gz + 1 - g0;
  }
  p.nchunks = last;
  p.nitems = items;
  p.off_counts = 0;
  p.off_offsets = al256(p.nchunks * 4);
  p.off_scan = p.off_offsets + al256(p.nchunks * 8 + 8);
  p.off_segs = p.off_scan + al256(chunk_scan_ws_bytes(p.nchunks));
  p.total = p.off_segs + al256((size_t)(nseg + 1) * sizeof(Seg));
  return p;
}

template <typename T, int B>
static void launch_decode(const uint8_t* packed, const DecodeGeom& geo, const Seg* segs, uint32_t* counts,
                          unsigned long long* offsets, void* scan_ws, const unsigned long long* prefix_rel,
                          const double* centers, const void* exact, const void* base, void* out,
                          nmk_segment_info* info, nmk_decode_err* err, cudaStream_t s) {
  const int sms = sm_count_d();
  uint64_t g1 = (geo.nchunks + 7) / 8;
  unsigned grid1 = (unsigned)(g1 < (uint64_t)sms * 8 ? g1 : (uint64_t)sms * 8);
  k_dec_count<B><<<grid1, kDecThreads, 0, s>>>(packed, geo, counts);
  chunk_scan(counts, geo.nchunks, offsets, nullptr, scan_ws, s);
  const size_t smem = 0;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dec_chunks<T, B>, kDecThreads, smem);
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = (uint64_t)sms * per_sm;
  uint64_t need = (geo.nitems + 7) / 8;
  if (grid > need) grid = need;
  k_dec_chunks<T, B><<<(unsigned)grid, kDecThreads, smem, s>>>(packed, geo, segs, offsets, prefix_rel, centers,
                                                                (const T*)exact, (const T*)base, (T*)out, info,
                                                                err);
}

template <typename T>
static int dispatch_decode(int bits, const uint8_t* packed, const DecodeGeom& geo, const Seg* segs, uint32_t* counts,
                           unsigned long long* offsets, void* scan_ws, const unsigned long long* prefix_rel,
                           const double* centers, const void* exact, const void* base, void* out,
                           nmk_segment_info* info, nmk_decode_err* err, cudaStream_t s) {
  switch (bits) {
#define NMK_DEC_CASE(BB)                                                                                    \
  case BB: launch_decode<T, BB>(packed, geo, segs, counts, offsets, scan_ws, prefix_rel, centers, exact, base, \
                                out, info, err, s); break;
    NMK_DEC_CASE(2) NMK_DEC_CASE(3) NMK_DEC_CASE(4) NMK_DEC_CASE(5) NMK_DEC_CASE(6) NMK_DEC_CASE(7)
    NMK_DEC_CASE(8) NMK_DEC_CASE(9) NMK_DEC_CASE(10) NMK_DEC_CASE(11) NMK_DEC_CASE(12) NMK_DEC_CASE(13)
    NMK_DEC_CASE(14) NMK_DEC_CASE(15) NMK_DEC_CASE(16) NMK_DEC_CASE(17) NMK_DEC_CASE(18) NMK_DEC_CASE(19)
    NMK_DEC_CASE(20) NMK_DEC_CASE(21) NMK_DEC_CASE(22) NMK_DEC_CASE(23) NMK_DEC_CASE(24) NMK_DEC_CASE(25)
    NMK_DEC_CASE(26) NMK_DEC_CASE(27) NMK_DEC_CASE(28) NMK_DEC_CASE(29) NMK_DEC_CASE(30)
#undef NMK_DEC_CASE
    default: return set_error(NMK_ERR_ARG, "nmk_decode: bits %d outside [2, 30]", bits);
  }
  return check_launch("k_dec_chunks");
}

}  // namespace nmk

using namespace nmk;

extern "C" size_t nmk_decode_ws_bytes(const uint64_t* h_seg_start, const uint64_t* h_seg_count, int nseg,
                                      uint64_t epb, uint64_t first_block) {
  if (nseg < 0 || epb == 0) return 0;
  return decode_plan(h_seg_start, h_seg_count, nseg, epb, first_block).total;
}

extern "C" int nmk_decode(const uint8_t* packed, uint64_t block_stride, uint64_t first_block, int bits,
                          uint64_t epb, uint64_t n_total, const unsigned long long* prefix_rel,
                          const double* centers, int k, const void* exact, uint64_t n_exact, const void* base,
                          void* out, int dtype, const uint64_t* h_seg_start, const uint64_t* h_seg_count,
                          const uint64_t* h_seg_out, int nseg, nmk_segment_info* seg_info,
                          nmk_decode_err* err, void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (nseg < 1 || !h_seg_start || !h_seg_count || !h_seg_out || !seg_info || !err || !ws)
    return set_error(NMK_ERR_ARG, "nmk_decode: bad argument");
  if (bits < 2 || bits > 30 || epb == 0 || k < 1) return set_error(NMK_ERR_ARG, "nmk_decode: bad geometry");
  if (block_stride % 16 || ((uintptr_t)packed & 15)) return set_error(NMK_ERR_ARG, "nmk_decode: packed alignment");
  if (dtype != NMK_F32 && dtype != NMK_F64) return set_error(NMK_ERR_ARG, "nmk_decode: bad dtype");
  for (int i = 0; i < nseg; ++i) {
    uint64_t st = h_seg_start[i], ct = h_seg_count[i];
    if (ct == 0 || st + ct > n_total || st / epb < first_block)
      return set_error(NMK_ERR_ARG, "nmk_decode: segment %d empty or outside the covered blocks", i);
  }
  if (!packed || !centers || !base || !out || !prefix_rel) return set_error(NMK_ERR_ARG, "nmk_decode: null pointer");
  DecodePlan p = decode_plan(h_seg_start, h_seg_count, nseg, epb, first_block);
  if (ws_bytes < p.total) return set_error(NMK_ERR_ARG, "nmk_decode: workspace too small");
  Seg* hs = (Seg*)malloc(sizeof(Seg) * (size_t)nseg);
  uint64_t item0 = 0;
  for (int i = 0; i < nseg; ++i) {
    const uint64_t st = h_seg_start[i], ct = h_seg_count[i], e = st + ct - 1;
    Seg sg;
    sg.start = st;
    sg.count = ct;
    sg.out = h_seg_out[i];
    sg.gfirst = (st / epb) * p.cpb + (st % epb) / kDChunk;
    sg.item0 = item0;
    item0 += (e / epb) * p.cpb + (e % epb) / kDChunk - sg.gfirst + 1;
    hs[i] = sg;
  }
  char* w = (char*)ws;
  uint32_t* counts = (uint32_t*)(w + p.off_counts);
  unsigned long long* offsets = (unsigned long long*)(w + p.off_offsets);
  Seg* dsegs = (Seg*)(w + p.off_segs);
  cudaMemsetAsync(seg_info, 0, sizeof(nmk_segment_info) * (size_t)nseg, s);
  cudaMemsetAsync(err, 0, sizeof(nmk_decode_err), s);
  // a pageable H2D cudaMemcpyAsync returns after staging the source, so the
  // host table can be released immediately (no stream synchronisation)
  cudaMemcpyAsync(dsegs, hs, sizeof(Seg) * (size_t)nseg, cudaMemcpyHostToDevice, s);
  free(hs);
  DecodeGeom geo{epb, p.cpb, n_total, first_block, block_stride, n_exact, p.nchunks, p.nitems, nseg, k};
  if (dtype == NMK_F64)
    return dispatch_decode<double>(bits, packed, geo, dsegs, counts, offsets, w + p.off_scan, prefix_rel, centers,
                                   exact, base, out, seg_info, err, s);
  return dispatch_decode<float>(bits, packed, geo, dsegs, counts, offsets, w + p.off_scan, prefix_rel, centers,
                                exact, base, out, seg_info, err, s);
}
