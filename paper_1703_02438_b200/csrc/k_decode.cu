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
//   3. k_dec_chunks: per-warp TMA pipeline over (segment, chunk) items:
//      rank the sentinels (segment anchor + chunk offset + warp scan),
//      gather exact values, reconstruct, store.  No inter-warp dependency.
// Geometry is computed once per chunk in 32-bit form (magic-number division
// for chunk -> block); elements only do 32-bit compares.
#include "nmk_common.cuh"
#include "nmk_scan.cuh"

namespace nmk {

constexpr int kDChunk = 32 * kGroup;   // 256 elements per warp chunk
constexpr int kDecThreads = 256;       // k_dec_count CTA
constexpr int kSmemSegs = 64;          // segment records cached in shared memory
constexpr int kTmaWarps = 4;           // k_dec_chunks CTA = 4 independent warps
constexpr int kTmaThreads = 32 * kTmaWarps;
#ifndef NMK_STAGES
#define NMK_STAGES 6   // measured: 6 stages x 4 CTAs/SM beats 4x6 by 30% (latency-bound)
#endif
#ifndef NMK_TMA_MINB
#define NMK_TMA_MINB 4
#endif
constexpr int kStages = NMK_STAGES;    // chunks in flight per warp
#ifndef NMK_STAGES_DENSE
#define NMK_STAGES_DENSE 5   // A/B: 5 beats 6 by 8-15 % of K5 when sentinels fill most chunks (profiles/README)
#endif
constexpr int kStagesDense = NMK_STAGES_DENSE;
// f32 chunks carry half the bytes of f64 ones: more of them in flight
#ifndef NMK_STAGES_F32
#define NMK_STAGES_F32 4   // A/B on cfg3 (512-element f32 items): 3 and 4 beat 5 and 6 (occupancy)
#endif
#ifndef NMK_STAGES_DENSE_F32
#define NMK_STAGES_DENSE_F32 3
#endif
template <typename T> struct Rings { static constexpr int kS = kStages, kD = kStagesDense; };
template <> struct Rings<float> { static constexpr int kS = NMK_STAGES_F32, kD = NMK_STAGES_DENSE_F32; };
#ifndef NMK_DENSE_DIV
#define NMK_DENSE_DIV 400    // "dense": more than 1 exact value per 400 elements (cfg2 0.16 % sparse, cfg4 0.5 % dense)
#endif
// Which ring depth decodes the stream.  A shallower ring leaves more of the
// unified shared/L1 array to L1, which serves the exact-value loads.  The
// density is the exact values available over the elements of the decoded
// chunk span (not the variable's n: a rank or a partial range decodes less).
__host__ __device__ inline bool dec_dense(uint64_t n_exact, uint64_t span_chunks) {
  return n_exact * (uint64_t)NMK_DENSE_DIV > span_chunks * 256ULL;
}

struct Seg {
  uint64_t start, count, out;   // global element range, output offset
  uint64_t item0;               // first work item (linear across segments)
  uint64_t gfirst;              // global chunk id of the segment's first chunk
};

struct SegParams {
  Seg s[NMK_DEV_MAX_SEG];
};

struct DecodeGeom {
  uint64_t epb, n_total, first_block, stride, n_exact, nchunks, nitems;
  uint32_t cpb;        // encoder chunks (256 elements) per block: the count pass and its offsets
  FastDiv fd_cpb;
  uint32_t cpb_d;      // decode chunks (DC elements) per block: k_dec_chunks' work items
  FastDiv fd_cpb_d;
  int nseg, k;
  ZeroList zl;   // scan tile status, segment info and error words: zeroed by the count pass
};

// One chunk: block b, in-block chunk ci, element/byte extents (32-bit).
struct DChunk {
  uint32_t b, ci;
  uint64_t chunk_lo;   // global index of the chunk's first element
  uint32_t valid;      // elements of the chunk inside its block (<= 256)
  uint32_t nbytes;     // packed bytes of the chunk inside its block
  uint32_t crel;       // chunk id relative to first_block's first chunk
};

template <int B>
__device__ __forceinline__ DChunk dchunk(const DecodeGeom& geo, uint32_t g) {
  DChunk d;
  d.b = geo.fd_cpb.div(g);
  d.ci = g - d.b * geo.cpb;
  const uint64_t blk_start = (uint64_t)d.b * geo.epb;
  const uint64_t rem = geo.n_total - blk_start;
  const uint32_t blk_len = (uint32_t)(rem < geo.epb ? rem : geo.epb);
  const uint32_t off = d.ci * kDChunk;
  d.chunk_lo = blk_start + off;
  d.valid = min((uint32_t)kDChunk, blk_len - off);
  const uint32_t blk_bytes = (uint32_t)(((uint64_t)blk_len * B + 7) / 8);
  d.nbytes = min((uint32_t)(32 * B), blk_bytes - d.ci * (32 * B));
  d.crel = g - (uint32_t)(geo.first_block * geo.cpb);
  return d;
}

template <int B>
__device__ __forceinline__ const uint8_t* chunk_src(const uint8_t* packed, const DecodeGeom& geo, const DChunk& d) {
  return packed + (uint64_t)(d.b - (uint32_t)geo.first_block) * geo.stride + (uint64_t)d.ci * (32 * B);
}

// Decode chunk g (DC = 256 or 512 elements: f32 decodes two encoder chunks
// per work item, so each item moves as many bytes as an f64 one and the
// per-item overhead is paid half as often).  crel is the encoder-chunk
// index (relative to first_block) of its first half; crel_end one past its
// last encoder chunk -- the count pass's offsets stay per 256 elements.
template <int B, int DC>
__device__ __forceinline__ DChunk dchunk_d(const DecodeGeom& geo, uint32_t g, uint32_t& crel_end) {
  constexpr uint32_t R = DC / kDChunk;
  DChunk d;
  d.b = geo.fd_cpb_d.div(g);
  d.ci = g - d.b * geo.cpb_d;
  const uint64_t blk_start = (uint64_t)d.b * geo.epb;
  const uint64_t rem = geo.n_total - blk_start;
  const uint32_t blk_len = (uint32_t)(rem < geo.epb ? rem : geo.epb);
  const uint32_t off = d.ci * DC;
  d.chunk_lo = blk_start + off;
  d.valid = min((uint32_t)DC, blk_len - off);
  const uint32_t blk_bytes = (uint32_t)(((uint64_t)blk_len * B + 7) / 8);
  d.nbytes = min((uint32_t)(DC / 8 * B), blk_bytes - d.ci * (DC / 8 * B));
  const uint32_t rb = (d.b - (uint32_t)geo.first_block) * geo.cpb;
  d.crel = rb + d.ci * R;
  crel_end = rb + min(d.ci * R + R, geo.cpb);
  return d;
}

template <int B, int DC>
__device__ __forceinline__ const uint8_t* chunk_src_d(const uint8_t* packed, const DecodeGeom& geo, const DChunk& d) {
  return packed + (uint64_t)(d.b - (uint32_t)geo.first_block) * geo.stride + (uint64_t)d.ci * (DC / 8 * B);
}

// This lane's B bytes (offset lane*B of a 16-byte aligned chunk) with the
// widest aligned loads B allows; bytes at or past nbytes read as zero.
template <int B>
__device__ __forceinline__ void lane_bytes(const uint8_t* src, uint32_t nbytes, int lane, uint8_t (&o)[B]) {
  const uint32_t s0 = (uint32_t)lane * B;
  constexpr int W = (B % 8 == 0) ? 8 : (B % 4 == 0) ? 4 : (B % 2 == 0) ? 2 : 1;
  if (s0 + B <= nbytes) {
#pragma unroll
    for (int w = 0; w < B / W; ++w) {
      const uint8_t* p = src + s0 + w * W;
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
    for (int i = 0; i < B; ++i) o[i] = (s0 + i < nbytes) ? __ldg(src + s0 + i) : (uint8_t)0;
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

// ---- 1. sentinels per chunk -------------------------------------------------
template <int B>
__device__ __forceinline__ unsigned lane_sentinels(const uint8_t (&raw)[B], uint32_t valid, int lane) {
  const uint32_t sentinel = (1u << B) - 1u;
  if constexpr (B == 8) {
    // one code per byte: count 0xff bytes four at a time (bytes past the
    // block end read as zero, never 0xff)
    const uint32_t lo = raw[0] | (raw[1] << 8) | (raw[2] << 16) | ((uint32_t)raw[3] << 24);
    const uint32_t hi = raw[4] | (raw[5] << 8) | (raw[6] << 16) | ((uint32_t)raw[7] << 24);
    return (__popc(__vcmpeq4(lo, 0xffffffffu)) + __popc(__vcmpeq4(hi, 0xffffffffu))) >> 3;
  } else {
    uint32_t code[kGroup];
    codes_of<B>(raw, code);
    const int s0 = lane * kGroup;
    unsigned n = 0;
#pragma unroll
    for (int e = 0; e < kGroup; ++e) n += (s0 + e < (int)valid && code[e] == sentinel);
    return n;
  }
}

// SWAR sentinel count for B in {10, 12, 14} (cfg3's and cfg5's widths):
// the lane's B bytes as a big-endian 128-bit string (hi:lo), its 8 codes as
// fields from the top.  A code is the sentinel iff its field in ~X is zero;
// per 64-bit word of whole fields, ((Z & LO) + LO) | Z) & MSB sets a field's
// top bit iff the field is nonzero (the add never carries out of a field).
// Padding never forms a sentinel: bits past the block's last code are zero
// and fewer than 8 (B > 8), bytes past nbytes read as zero.
template <int B>
struct SwarCount {
  static constexpr bool kOn = B == 10 || B == 12 || B == 14;
  static constexpr int kFa = 64 / B;        // whole fields in the top word
  static constexpr int kFb = 8 - kFa;       // the rest, top-aligned in the second word
  static constexpr unsigned long long fields(int nf, bool msb) {
    unsigned long long m = 0;
    for (int e = 0; e < nf; ++e) {
      const int lo = 64 - (e + 1) * B;
      m |= msb ? (1ULL << (lo + B - 1)) : (((1ULL << (B - 1)) - 1ULL) << lo);
    }
    return m;
  }
};

template <int B>
__device__ __forceinline__ unsigned lane_sentinels_swar(const uint8_t* src, uint32_t nbytes, int lane) {
  using S = SwarCount<B>;
  const uint32_t s0 = (uint32_t)lane * B;
  uint32_t w[4] = {0u, 0u, 0u, 0u};   // little-endian words of bytes s0 .. s0 + 15
  if (s0 + B <= nbytes) {
    if constexpr (B == 12) {
#pragma unroll
      for (int j = 0; j < 3; ++j) w[j] = __ldg(reinterpret_cast<const unsigned int*>(src + s0) + j);
    } else {
      const unsigned short* h = reinterpret_cast<const unsigned short*>(src + s0);
#pragma unroll
      for (int j = 0; j < B / 2; ++j) w[j >> 1] |= (uint32_t)__ldg(h + j) << (16 * (j & 1));
    }
  } else {
    for (int i = 0; i < B; ++i)
      if (s0 + i < nbytes) w[i >> 2] |= (uint32_t)__ldg(src + s0 + i) << (8 * (i & 3));
  }
  const unsigned long long hi = ((unsigned long long)__byte_perm(w[0], 0, 0x0123) << 32) | __byte_perm(w[1], 0, 0x0123);
  const unsigned long long lo = ((unsigned long long)__byte_perm(w[2], 0, 0x0123) << 32) | __byte_perm(w[3], 0, 0x0123);
  constexpr int sh = S::kFa * B;   // < 64
  const unsigned long long wb = (hi << sh) | (lo >> (64 - sh));
  auto zero_fields = [](unsigned long long x, unsigned long long lom, unsigned long long msb, int nf) {
    const unsigned long long z = ~x;
    const unsigned long long t = (((z & lom) + lom) | z) & msb;
    return (unsigned)(nf - __popcll(t));
  };
  return zero_fields(hi, S::fields(S::kFa, false), S::fields(S::kFa, true), S::kFa) +
         zero_fields(wb, S::fields(S::kFb, false), S::fields(S::kFb, true), S::kFb);
}

template <int B>
__global__ void __launch_bounds__(kDecThreads)
k_dec_count(const uint8_t* __restrict__ packed, DecodeGeom geo, uint32_t* __restrict__ counts) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  pdl_enter();
  zero_list_run(geo.zl);
  const uint32_t nwarps = gridDim.x * (kDecThreads / 32);
  const uint32_t g0 = (uint32_t)(geo.first_block * geo.cpb);
  // (A/B on cfg3 / cfg5 B12: 2, 4 or 8 chunks per warp iteration no faster)
  for (uint32_t c = blockIdx.x * (kDecThreads / 32) + wid; c < (uint32_t)geo.nchunks; c += nwarps) {
    const DChunk d = dchunk<B>(geo, g0 + c);
    unsigned mine;
    if constexpr (SwarCount<B>::kOn) {
      mine = lane_sentinels_swar<B>(chunk_src<B>(packed, geo, d), d.nbytes, lane);
    } else {
      uint8_t raw[B];
      lane_bytes<B>(chunk_src<B>(packed, geo, d), d.nbytes, lane, raw);
      mine = lane_sentinels<B>(raw, d.valid, lane);
    }
    const unsigned n = __reduce_add_sync(0xffffffffu, mine);
    if (lane == 0) counts[c] = n;
  }
}

// Byte-aligned code widths (B = 8, 16): a half-warp per chunk, 16-byte
// coalesced loads (a warp reads two chunks' 2 x 32B bytes per instruction,
// kDecPairs pairs in flight) and SIMD compares (a sentinel is an all-ones
// byte / halfword), reduced over the half-warp.
template <int B>
__device__ __forceinline__ unsigned sentinels_in_word(uint32_t w) {
  if constexpr (B == 8) return __popc(__vcmpeq4(w, 0xffffffffu)) >> 3;
  else return __popc(__vcmpeq2(w, 0xffffffffu)) >> 4;
}

template <int B>
__device__ __forceinline__ unsigned sentinels_in_vec(const uint4& v) {
  return sentinels_in_word<B>(v.x) + sentinels_in_word<B>(v.y) + sentinels_in_word<B>(v.z) +
         sentinels_in_word<B>(v.w);
}

#ifndef NMK_DEC_WIN96
#define NMK_DEC_WIN96 1   // codes_at: one 96-bit window for VN * B <= 64
#endif
#ifndef NMK_DEC_PAIRS
#define NMK_DEC_PAIRS 4   // A/B: 2 and 8 pairs, 4 or 8 CTAs/SM all within 1 %
#endif
#ifndef NMK_CNT_CTAS
#define NMK_CNT_CTAS 4
#endif
constexpr int kDecPairs = NMK_DEC_PAIRS;   // chunk pairs per warp iteration

// Each warp counts a contiguous run of chunks; half-warp h takes chunks
// cA + h, cA + h + 2, ... through a cursor advanced without division.
template <int B>
__global__ void __launch_bounds__(kDecThreads)
k_dec_count_wide(const uint8_t* __restrict__ packed, DecodeGeom geo, uint32_t* __restrict__ counts) {
  static_assert(B == 8 || B == 16, "byte-aligned codes only");
  constexpr int kPer = (32 * B / 16) / 16;   // 16-byte vectors per lane per chunk (1 or 2)
  const int lane = threadIdx.x & 31, half = lane >> 4, sub = lane & 15;
  pdl_enter();
  zero_list_run(geo.zl);
  const uint32_t g0 = (uint32_t)(geo.first_block * geo.cpb);
  const uint32_t nch = (uint32_t)geo.nchunks;
  const uint32_t nwarps = gridDim.x * (kDecThreads / 32);
  const uint32_t wg = blockIdx.x * (kDecThreads / 32) + (threadIdx.x >> 5);
  const uint32_t per = nch / nwarps, rem = nch % nwarps;
  const uint32_t cA = wg * per + min(wg, rem), cB = cA + per + (wg < rem ? 1u : 0u);
  if (cA >= cB) return;
  const uint32_t cpb = geo.cpb;
  // cursor of this half's next chunk
  uint32_t c = cA + half;
  const DChunk d0 = dchunk<B>(geo, g0 + min(c, nch - 1));
  uint32_t b = d0.b, ci = d0.ci;
  auto adv2 = [&]() {
    c += 2;
    ci += 2;
    if (ci >= cpb) { ci -= cpb; ++b; }
  };
  while (__any_sync(0xffffffffu, c < cB)) {
    uint4 w[kDecPairs][kPer];
    uint32_t cc[kDecPairs], nb[kDecPairs];
    const uint8_t* src[kDecPairs];
#pragma unroll
    for (int u = 0; u < kDecPairs; ++u) {
      cc[u] = c;
      nb[u] = 0;
      src[u] = packed + (uint64_t)(b - (uint32_t)geo.first_block) * geo.stride + (uint64_t)ci * (32 * B);
      if (c < cB) {
        // bytes of this chunk inside its block (all 32 B unless it is the block's clipped tail)
        const uint64_t blk_start = (uint64_t)b * geo.epb;
        const uint64_t rem_el = geo.n_total - blk_start;
        const uint32_t blk_len = (uint32_t)(rem_el < geo.epb ? rem_el : geo.epb);
        const uint32_t blk_bytes = (uint32_t)(((uint64_t)blk_len * B + 7) / 8);
        nb[u] = min((uint32_t)(32 * B), blk_bytes - ci * (32 * B));
        const uint4* v4 = reinterpret_cast<const uint4*>(src[u]);   // 16-byte aligned
#pragma unroll
        for (int p = 0; p < kPer; ++p) {
          const uint32_t o = (uint32_t)(sub + 16 * p) * 16;
          w[u][p] = o + 16 <= nb[u] ? __ldg(v4 + sub + 16 * p) : make_uint4(0, 0, 0, 0);
        }
      }
      adv2();
    }
#pragma unroll
    for (int u = 0; u < kDecPairs; ++u) {
      unsigned n = 0;
#pragma unroll
      for (int p = 0; p < kPer; ++p) {
        const uint32_t o = (uint32_t)(sub + 16 * p) * 16;
        if (o + 16 <= nb[u]) {
          n += sentinels_in_vec<B>(w[u][p]);
        } else if (o < nb[u]) {   // the block's last, clipped vector
          for (uint32_t i = o; i < nb[u]; i += B / 8) {
            if constexpr (B == 8) n += src[u][i] == 0xff;
            else n += (src[u][i] & src[u][i + 1]) == 0xff;
          }
        }
      }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);   // within the half-warp
      if (sub == 0 && cc[u] < cB) counts[cc[u]] = n;
    }
  }
}

// ---- 3. reconstruct: per-warp TMA pipeline ---------------------------------
// Each warp owns kStages shared-memory stages.  Lane 0 keeps kStages chunks in
// flight with 1-D bulk copies (the chunk's base values + its packed bytes),
// completion tracked by one mbarrier per stage (transaction bytes), so the
// bytes in flight cost no registers.  Lanes read a stage conflict-free (lane
// l takes 16-byte vector l of each 512-byte row) and store fully coalesced.
// Chunks that cannot be bulk-copied (segment edges, misaligned base, packed
// bytes running past the block's stride) fall back to direct loads.
template <typename T> struct DVec;
template <> struct DVec<double> { using V = double2; static constexpr int N = 2; };
template <> struct DVec<float>  { using V = float4;  static constexpr int N = 4; };

// decode-chunk size: 512 elements for f32 (two encoder chunks), 256 for f64
template <typename T> struct DecChunk { static constexpr int kDC = sizeof(T) == 4 ? 512 : 256; };

template <typename T, int B, int S = kStages>
struct DecStage {
  static constexpr int kDC = DecChunk<T>::kDC;
  static constexpr int kBase = kDC * (int)sizeof(T);        // 2048 bytes for both dtypes
  static constexpr int kPk = kDC / 8 * B;                   // a multiple of 16
  static constexpr int kAux = kBase + kPk + 16;             // +16: 8-byte code windows
  static constexpr int kBytes = kAux + 32;                  // rank anchors (4 x u64)
  static constexpr size_t kSmem = (size_t)kTmaWarps * S * kBytes;
};

// B-bit code of chunk element e from the staged packed bytes (MSB-first).
template <int B>
__device__ __forceinline__ uint32_t code_at(const uint8_t* pk, int e) {
  if constexpr (B == 8) {
    return pk[e];
  } else {
    const int bit = e * B;
    const int w = (bit >> 5) << 2;                          // aligned 4-byte word
    const uint32_t a = __byte_perm(*reinterpret_cast<const uint32_t*>(pk + w), 0, 0x0123);
    const uint32_t z = __byte_perm(*reinterpret_cast<const uint32_t*>(pk + w + 4), 0, 0x0123);
    const unsigned long long x = ((unsigned long long)a << 32) | z;
    const int off = bit & 31;                               // off + B <= 61
    return (uint32_t)(x >> (64 - off - B)) & ((1u << B) - 1u);
  }
}

// The VN consecutive codes of elements e0 .. e0+VN-1 (MSB-first) from one
// 64-bit window when they fit (VN*B <= 33), else one code at a time.
template <int B, int VN>
__device__ __forceinline__ void codes_at(const uint8_t* pk, int e0, uint32_t (&cd)[VN]) {
  if constexpr (B == 8 && VN == 2) {
    const uint32_t two = *reinterpret_cast<const uint16_t*>(pk + e0);   // e0 even
    cd[0] = two & 255u;
    cd[1] = two >> 8;
  } else if constexpr (B == 8 && VN == 4) {
    const uint32_t four = *reinterpret_cast<const uint32_t*>(pk + e0);  // e0 % 4 == 0
#pragma unroll
    for (int v = 0; v < 4; ++v) cd[v] = (four >> (8 * v)) & 255u;
  } else if constexpr (VN * B <= 33) {
    const int bit = e0 * B;
    const int w = (bit >> 5) << 2;
    const uint32_t a = __byte_perm(*reinterpret_cast<const uint32_t*>(pk + w), 0, 0x0123);
    const uint32_t z = __byte_perm(*reinterpret_cast<const uint32_t*>(pk + w + 4), 0, 0x0123);
    const unsigned long long x = ((unsigned long long)a << 32) | z;
    const int off = bit & 31;
#pragma unroll
    for (int v = 0; v < VN; ++v) cd[v] = (uint32_t)(x >> (64 - off - (v + 1) * B)) & ((1u << B) - 1u);
  } else if constexpr (VN * B <= 64 && NMK_DEC_WIN96) {
    // a 96-bit window (three aligned words) holds the VN codes at any offset
    // (off + VN*B <= 31 + 64); the stage's +16 pad keeps the third word in bounds
    const int bit = e0 * B;
    const int w = (bit >> 5) << 2;
    const uint32_t a = __byte_perm(*reinterpret_cast<const uint32_t*>(pk + w), 0, 0x0123);
    const uint32_t m = __byte_perm(*reinterpret_cast<const uint32_t*>(pk + w + 4), 0, 0x0123);
    const uint32_t z = __byte_perm(*reinterpret_cast<const uint32_t*>(pk + w + 8), 0, 0x0123);
    const int off = bit & 31;
    const unsigned long long top = ((((unsigned long long)a << 32) | m) << off) |
                                   ((((unsigned long long)z) << off) >> 32);
#pragma unroll
    for (int v = 0; v < VN; ++v) cd[v] = (uint32_t)(top >> (64 - (v + 1) * B)) & ((1u << B) - 1u);
  } else {
#pragma unroll
    for (int v = 0; v < VN; ++v) cd[v] = code_at<B>(pk, e0 + v);
  }
}

// (1 + c) per code, in shared memory for small code books
constexpr int kOpcMax = 2048;

struct DItem {
  int seg;
  DChunk d;
  uint32_t crel_end;         // one past the item's last encoder chunk (offsets index)
  uint32_t lo_rel, hi_rel;   // in-segment elements of the chunk: [lo_rel, hi_rel)
  int64_t oi0;               // base/out index of the chunk's first element
  uint32_t anchor;           // block (relative) of the segment's first chunk
  bool first, last;          // the segment's first / last chunk
  bool base_tma, pk_tma;
};

template <typename T, int B>
__device__ __forceinline__ DItem decode_item(uint64_t it, const DecodeGeom& geo, const Seg* SG,
                                             const T* __restrict__ base) {
  constexpr int DC = DecChunk<T>::kDC;
  int s = 0;
  if (geo.nseg > 1) {
    int hi_s = geo.nseg - 1;
    while (s < hi_s) {
      int mid = (s + hi_s + 1) >> 1;
      if (SG[mid].item0 <= it) s = mid; else hi_s = mid - 1;
    }
  }
  const Seg sg = SG[s];
  DItem t;
  t.seg = s;
  const uint32_t rel = (uint32_t)(it - sg.item0);
  t.d = dchunk_d<B, DC>(geo, (uint32_t)sg.gfirst + rel, t.crel_end);
  t.first = rel == 0;
  const int64_t lo = (int64_t)sg.start - (int64_t)t.d.chunk_lo;
  const int64_t hi = lo + (int64_t)sg.count;
  t.lo_rel = (uint32_t)(lo < 0 ? 0 : lo);
  t.hi_rel = (uint32_t)(hi > (int64_t)t.d.valid ? (int64_t)t.d.valid : hi);
  t.last = hi <= (int64_t)t.d.valid;
  t.oi0 = (int64_t)sg.out - lo;
  t.anchor = geo.fd_cpb_d.div((uint32_t)sg.gfirst) - (uint32_t)geo.first_block;
  t.base_tma = t.lo_rel == 0 && t.hi_rel == (uint32_t)DC && ((uintptr_t)(base + t.oi0) & 15) == 0;
  t.pk_tma = (uint64_t)(t.d.ci + 1) * (DC / 8 * B) <= geo.stride;
  return t;
}

// 8-byte asynchronous copy into shared memory, and an mbarrier arrival once
// this thread's prior cp.async copies have landed
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Per stage: lane 0 issues the chunk's base values and packed bytes as TMA
// bulk copies plus four 8-byte cp.async copies of its rank anchors
// (offsets[c], offsets[c+1], the anchor block's first offset and prefix);
// the stage's mbarrier (2 arrivals: expect_tx + the cp.async group) completes
// when all of them landed, so no global load sits on a warp's critical path
// except the exact values, which are fetched right after the wait (one per
// lane, coalesced) and handed to the sentinels by shuffle.
template <typename T, int B, int S>
__global__ void __launch_bounds__(kTmaThreads, NMK_TMA_MINB)
k_dec_chunks(const uint8_t* __restrict__ packed, DecodeGeom geo, const Seg* __restrict__ segs, SegParams sp,
             const unsigned long long* __restrict__ offsets, const unsigned long long* __restrict__ prefix_rel,
             const double* __restrict__ centers_g, const T* __restrict__ exact, const T* __restrict__ base,
             T* __restrict__ out, nmk_segment_info* __restrict__ info, nmk_decode_err* __restrict__ err,
             const nmk_model* __restrict__ model, const unsigned long long* __restrict__ n_exact_dev,
             int regime) {
  using ST = DecStage<T, B, S>;
  constexpr int VN = DVec<T>::N;          // elements per 16-byte vector
  constexpr int DC = DecChunk<T>::kDC;    // elements per work item
  constexpr int Q = DC / 32 / VN;         // vectors per lane per item (4 for both dtypes)
  using V = typename DVec<T>::V;
  const unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(128) uint8_t dsm[];
  __shared__ __align__(8) unsigned long long bars[kTmaWarps][S];
  __shared__ Seg s_segs[kSmemSegs];
  __shared__ DItem s_items[kTmaWarps][S];   // geometry of each staged chunk (written at issue)
  constexpr bool kOpcSmem = ((1 << B) - 1) <= kOpcMax;
  double* s_opc = reinterpret_cast<double*>(dsm + DecStage<T, B, S>::kSmem);   // [2^B - 1] when kOpcSmem
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  pdl_enter();
  if (model) {                       // sync-free path: scalars from the device
    if (model->status != 0) return;
    geo.k = model->k;
  }
  if (n_exact_dev) geo.n_exact = *n_exact_dev;
  if (regime != 0 && (regime == 2) != dec_dense(geo.n_exact, geo.nchunks)) return;   // the other ring runs
  const bool seg_smem = geo.nseg <= kSmemSegs;
  if (!segs)
    for (int i = threadIdx.x; i < geo.nseg; i += kTmaThreads) s_segs[i] = sp.s[i];
  else if (seg_smem)
    for (int i = threadIdx.x; i < geo.nseg; i += kTmaThreads) s_segs[i] = segs[i];
  if (lane == 0) {
    for (int st = 0; st < S; ++st) mbar_init(&bars[wid][st], 2);
    mbar_fence_init();
  }
  if constexpr (kOpcSmem) {   // decoder arithmetic (1 + c) (core.py:202-205); codes >= k are errors
    for (int i = threadIdx.x; i < (1 << B) - 1; i += kTmaThreads)
      s_opc[i] = __dadd_rn(1.0, __ldg(centers_g + min(i, geo.k - 1)));
  }
  __syncthreads();
  const Seg* SG = (seg_smem || !segs) ? s_segs : segs;
  uint8_t* wst = dsm + (size_t)wid * S * ST::kBytes;
  const uint32_t sentinel = (1u << B) - 1u;
  const uint32_t k = (uint32_t)geo.k;
  const bool out_al = ((uintptr_t)out & 15) == 0;
  const uint64_t gw = (uint64_t)blockIdx.x * kTmaWarps + wid, nw = (uint64_t)gridDim.x * kTmaWarps;

  auto issue = [&](int st, uint64_t it) {       // lane 0 only
    const DItem t = decode_item<T, B>(it, geo, SG, base);
    s_items[wid][st] = t;
    uint8_t* sb = wst + st * ST::kBytes;
    mbar_arrive_tx(&bars[wid][st], (t.base_tma ? ST::kBase : 0) + (t.pk_tma ? ST::kPk : 0));
    if (t.base_tma) tma_load_1d(sb, base + t.oi0, ST::kBase, &bars[wid][st]);
    if (t.pk_tma) tma_load_1d(sb + ST::kBase, chunk_src_d<B, DC>(packed, geo, t.d), ST::kPk, &bars[wid][st]);
    const uint32_t aux = smem_u32(sb + ST::kAux);
    cp_async8(aux, offsets + t.d.crel);
    cp_async8(aux + 8, offsets + t.crel_end);
    cp_async8(aux + 16, offsets + (uint64_t)t.anchor * geo.cpb);
    cp_async8(aux + 24, prefix_rel + t.anchor);
    cp_async_arrive(&bars[wid][st]);
  };
  if (lane == 0)
    for (int st = 0; st < S; ++st)
      if (gw + st * nw < geo.nitems) issue(st, gw + st * nw);
  __syncwarp();

  for (uint64_t kk = 0;; ++kk) {
    const uint64_t it = gw + kk * nw;
    if (it >= geo.nitems) break;
    const int st = (int)(kk % S);
    uint8_t* sb = wst + st * ST::kBytes;
    const DItem t = s_items[wid][st];
    T bv[Q][VN];
    if (!t.base_tma) {
#pragma unroll
      for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int v = 0; v < VN; ++v) {
          const uint32_t e = VN * lane + 32 * VN * q + v;
          bv[q][v] = (e >= t.lo_rel && e < t.hi_rel) ? __ldg(base + (t.oi0 + e)) : T(0);
        }
    }
    mbar_wait(&bars[wid][st], (unsigned)((kk / S) & 1));
    // the chunk's rank anchor (codec.py:231-236: prefix of the segment's first
    // block + sentinels counted since) and its sentinel count
    const unsigned long long* ax = reinterpret_cast<const unsigned long long*>(sb + ST::kAux);
    const unsigned long long chunk_off = ax[3] + (ax[0] - ax[2]);
    const uint32_t nsent = (uint32_t)(ax[1] - ax[0]);
    if (!t.pk_tma) {
      const uint8_t* src = chunk_src_d<B, DC>(packed, geo, t.d);
      for (int i = lane; i < ST::kPk; i += 32) sb[ST::kBase + i] = (uint32_t)i < t.d.nbytes ? __ldg(src + i) : 0;
      __syncwarp();
    }
    if (t.base_tma && out_al) {
      // fast path: the whole chunk lies inside the segment and its block, so
      // no element needs a bounds test.  Exact values first (latency hides
      // behind the arithmetic): lane j holds the chunk's j-th one.
      const bool few = nsent <= 32;
      T exv = T(0);
      if (nsent && few && lane < (int)nsent && chunk_off + lane < geo.n_exact) exv = exact[chunk_off + lane];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const V w = *reinterpret_cast<const V*>(sb + 16 * lane + 512 * q);
        const T* tw = reinterpret_cast<const T*>(&w);
#pragma unroll
        for (int v = 0; v < VN; ++v) bv[q][v] = tw[v];
      }
      uint32_t code[Q][VN];
      T ov[Q][VN];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        codes_at<B, VN>(sb + ST::kBase, VN * lane + 32 * VN * q, code[q]);
#pragma unroll
        for (int v = 0; v < VN; ++v) {
          const uint32_t cd = code[q][v];
          if constexpr (kOpcSmem)
            ov[q][v] = narrow<T>(__dmul_rn(s_opc[min(cd, (uint32_t)(1 << B) - 2u)], to_f64(bv[q][v])));
          else
            ov[q][v] = apply_center<T>(__ldg(centers_g + min(cd, k - 1)), to_f64(bv[q][v]));
        }
      }
      // ids in [k, sentinel) are errors; impossible with a full code book
      // ((code + 1) mod 2^B) maps the sentinel to 0 and id c to c + 1, so one
      // max per element finds the largest non-sentinel id
      if (k < sentinel) {
        uint32_t mx = 0;
#pragma unroll
        for (int q = 0; q < Q; ++q)
#pragma unroll
          for (int v = 0; v < VN; ++v) mx = max(mx, (code[q][v] + 1u) & sentinel);
        if (mx > k) {
          atomicOr(&err->bad_index, 1u);
          atomicMax(&err->max_bad_index, mx - 1u);
        }
      }
      if (nsent) {   // warp-uniform (from the count pass)
        unsigned smask = 0, cnt_pk = 0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          unsigned c = 0;
#pragma unroll
          for (int v = 0; v < VN; ++v) {
            const bool snt = code[q][v] == sentinel;
            smask |= (snt ? 1u : 0u) << (q * VN + v);
            c += snt;
          }
          cnt_pk |= c << (8 * q);
        }
        unsigned incl = cnt_pk;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(FULL, incl, o);
          if (lane >= o) incl += y;
        }
        const unsigned tot = __shfl_sync(FULL, incl, 31);
        const unsigned excl = incl - cnt_pk;
        unsigned before_q = 0, exhausted = 0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          unsigned r = before_q + ((excl >> (8 * q)) & 255u);   // rank within the chunk
          before_q += (tot >> (8 * q)) & 255u;
#pragma unroll
          for (int v = 0; v < VN; ++v) {
            const bool snt = smask >> (q * VN + v) & 1u;
            if (few) {
              const T got = __shfl_sync(FULL, exv, (int)(r & 31u));
              if (snt) {
                if (chunk_off + r < geo.n_exact) ov[q][v] = got;
                else exhausted = 1;
              }
            } else if (snt) {
              if (chunk_off + r < geo.n_exact) ov[q][v] = exact[chunk_off + r];
              else exhausted = 1;
            }
            r += snt ? 1u : 0u;
          }
        }
        if (exhausted) atomicOr(&err->exhausted, 1u);
      }
#pragma unroll
      for (int q = 0; q < Q; ++q)
        *reinterpret_cast<V*>(out + t.oi0 + VN * lane + 32 * VN * q) = *reinterpret_cast<const V*>(&ov[q][0]);
      // segment bookkeeping: inc_before = rank at the segment start, and
      // n_sentinel = rank(end) - rank(start), added by the last / first chunk
      if (lane == 0) {
        if (t.first) {
          info[t.seg].inc_before = chunk_off;
          atomicAdd(&info[t.seg].n_sentinel, 0ULL - chunk_off);
        }
        if (t.last) atomicAdd(&info[t.seg].n_sentinel, chunk_off + nsent);
      }
      __syncwarp();
      if (lane == 0) {
        fence_proxy_async_smem();
        const uint64_t nx = it + (uint64_t)S * nw;
        if (nx < geo.nitems) issue(st, nx);
      }
      continue;
    }
    if (t.base_tma) {
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const V w = *reinterpret_cast<const V*>(sb + 16 * lane + 512 * q);
        const T* tw = reinterpret_cast<const T*>(&w);
#pragma unroll
        for (int v = 0; v < VN; ++v) bv[q][v] = tw[v];
      }
    }
    // codes and masks; element order is (q, lane, v)
    uint32_t code[Q][VN];
    unsigned smask = 0, inmask = 0, cnt_pk = 0, ahead = 0, upto = 0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      unsigned c = 0;
#pragma unroll
      for (int v = 0; v < VN; ++v) {
        const uint32_t e = VN * lane + 32 * VN * q + v;
        code[q][v] = code_at<B>(sb + ST::kBase, e);
        const int bitp = q * VN + v;
        if (e < t.d.valid && code[q][v] == sentinel) {
          smask |= 1u << bitp;
          ++c;
          ahead += e < t.lo_rel;
          upto += e < t.hi_rel;
        }
        if (e >= t.lo_rel && e < t.hi_rel) inmask |= 1u << bitp;
      }
      cnt_pk |= c << (8 * q);
    }
    // per-q sentinel ranks with one packed warp scan (byte lanes, <= 128 each)
    unsigned incl = cnt_pk;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const unsigned tot = __shfl_sync(FULL, incl, 31);
    const unsigned excl = incl - cnt_pk;
    T ov[Q][VN];
    unsigned bad = 0, maxbad = 0, exhausted = 0;
    unsigned long long before_q = 0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      unsigned long long pos = chunk_off + before_q + ((excl >> (8 * q)) & 255u);
      before_q += (tot >> (8 * q)) & 255u;
#pragma unroll
      for (int v = 0; v < VN; ++v) {
        const int bitp = q * VN + v;
        ov[q][v] = T(0);
        if (smask >> bitp & 1u) {
          if (inmask >> bitp & 1u) {
            if (pos < geo.n_exact) ov[q][v] = exact[pos];
            else exhausted = 1;
          }
          ++pos;
        } else if (inmask >> bitp & 1u) {
          const uint32_t cd = code[q][v];
          if (cd >= k) {
            bad = 1;
            maxbad = cd > maxbad ? cd : maxbad;
          } else {
            ov[q][v] = apply_center<T>(__ldg(centers_g + cd), to_f64(bv[q][v]));
          }
        }
      }
    }
    if (t.base_tma && out_al) {
#pragma unroll
      for (int q = 0; q < Q; ++q)
        *reinterpret_cast<V*>(out + t.oi0 + VN * lane + 32 * VN * q) = *reinterpret_cast<const V*>(&ov[q][0]);
    } else {
#pragma unroll
      for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int v = 0; v < VN; ++v)
          if (inmask >> (q * VN + v) & 1u) out[t.oi0 + VN * lane + 32 * VN * q + v] = ov[q][v];
    }
    if (bad) {
      atomicOr(&err->bad_index, 1u);
      atomicMax(&err->max_bad_index, maxbad);
    }
    if (exhausted) atomicOr(&err->exhausted, 1u);
    if (t.first || t.last) {
      const unsigned ah = __reduce_add_sync(FULL, ahead), up = __reduce_add_sync(FULL, upto);
      if (lane == 0) {
        if (t.first) {
          info[t.seg].inc_before = chunk_off + ah;
          atomicAdd(&info[t.seg].n_sentinel, 0ULL - (chunk_off + ah));
        }
        if (t.last) atomicAdd(&info[t.seg].n_sentinel, chunk_off + up);
      }
    }
    // stage consumed: refill it S chunks ahead
    __syncwarp();
    if (lane == 0) {
      fence_proxy_async_smem();
      const uint64_t nx = it + (uint64_t)S * nw;
      if (nx < geo.nitems) issue(st, nx);
    }
  }
}

static int sm_count_d() { return sm_count(); }

static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

struct DecodePlan {
  uint64_t cpb, cpb_d, nchunks, nitems;
  size_t off_counts, off_offsets, off_scan, off_segs, total;
};

// dc = decode-chunk size (k_dec_chunks' items); the count pass covers every
// encoder chunk of the decode chunks touched, so the workspace is sized with
// the largest dc (nmk_decode_ws_bytes has no dtype)
static DecodePlan decode_plan(const uint64_t* st, const uint64_t* ct, int nseg, uint64_t epb, uint64_t first_block,
                              uint64_t dc = 512) {
  DecodePlan p{};
  p.cpb = (epb + kDChunk - 1) / kDChunk;
  p.cpb_d = (epb + dc - 1) / dc;
  const uint64_t R = dc / kDChunk;
  uint64_t items = 0, last = 0;
  const uint64_t g0 = first_block * p.cpb;
  for (int s = 0; s < nseg; ++s) {
    if (ct[s] == 0) continue;
    uint64_t e = st[s] + ct[s] - 1;
    uint64_t ga = (st[s] / epb) * p.cpb_d + (st[s] % epb) / dc;
    uint64_t gz = (e / epb) * p.cpb_d + (e % epb) / dc;
    items += gz - ga + 1;
    const uint64_t ci_end = (e % epb) / dc * R + R;
    const uint64_t end = (e / epb) * p.cpb + (ci_end < p.cpb ? ci_end : p.cpb);
    if (end - g0 > last) last = end - g0;
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

template <typename T, int B, int S>
static void launch_dec_chunks(const uint8_t* packed, const DecodeGeom& geo, const Seg* segs, const SegParams& sp,
                              const unsigned long long* offsets, const unsigned long long* prefix_rel,
                              const double* centers, const void* exact, const void* base, void* out,
                              nmk_segment_info* info, nmk_decode_err* err, const nmk_model* model,
                              const unsigned long long* n_exact_dev, int regime, cudaStream_t s) {
  const int sms = sm_count_d();
  const size_t smem = DecStage<T, B, S>::kSmem + (((1 << B) - 1) <= kOpcMax ? (size_t)((1 << B) - 1) * 8 : 0);
  ensure_dyn_smem(k_dec_chunks<T, B, S>, smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dec_chunks<T, B, S>, kTmaThreads, smem);
  if (per_sm < 1) per_sm = 1;
  uint64_t grid = (uint64_t)sms * per_sm;
  const uint64_t need = (geo.nitems + kTmaWarps - 1) / kTmaWarps;   // nitems: decode chunks
  if (grid > need) grid = need;
  launch_chain(kPdlDecode, k_dec_chunks<T, B, S>, (unsigned)grid, kTmaThreads, smem, s, packed, geo, segs, sp, offsets, prefix_rel,
               centers, (const T*)exact, (const T*)base, (T*)out, info, err, model, n_exact_dev, regime);
}

template <typename T, int B>
static void launch_decode(const uint8_t* packed, const DecodeGeom& geo, const Seg* segs, const SegParams& sp,
                          uint32_t* counts, unsigned long long* offsets, void* scan_ws,
                          const unsigned long long* prefix_rel, const double* centers, const void* exact,
                          const void* base, void* out, nmk_segment_info* info, nmk_decode_err* err,
                          const nmk_model* model, const unsigned long long* n_exact_dev, int ring_hint,
                          cudaStream_t s) {
  const int sms = sm_count_d();
  if constexpr (B == 8 || B == 16) {
    const uint64_t per_cta = (uint64_t)(kDecThreads / 32) * 2 * kDecPairs;
    const uint64_t g1 = (geo.nchunks + per_cta - 1) / per_cta;
    const unsigned grid1 = (unsigned)(g1 < (uint64_t)sms * NMK_CNT_CTAS ? g1 : (uint64_t)sms * NMK_CNT_CTAS);
    launch_chain(kPdlCount, k_dec_count_wide<B>, grid1, kDecThreads, 0, s, packed, geo, counts);
  } else {
    const uint64_t g1 = (geo.nchunks + 7) / 8;
    const unsigned grid1 = (unsigned)(g1 < (uint64_t)sms * 8 ? g1 : (uint64_t)sms * 8);
    launch_chain(kPdlCount, k_dec_count<B>, grid1, kDecThreads, 0, s, packed, geo, counts);
  }
  chunk_scan(counts, geo.nchunks, offsets, scan_ws, s, true);
  // The host knows the exact count on the host-scalar path and picks one ring.
  // The sync-free path only knows it on the device: both rings launch and
  // the one whose regime does not match exits at entry.  (CUDA graph IF
  // nodes set by the count pass were measured slower than the empty launch:
  // cfg2 +25 us, cfg3 +19 us per step.)
  // ring_hint (1 sparse, 2 dense: the regime the caller observed on the
  // previous step) launches that ring alone; either ring decodes any stream,
  // so the hint only affects speed.
  if (!n_exact_dev || ring_hint == 1 || ring_hint == 2) {
    if (n_exact_dev ? ring_hint == 2 : dec_dense(geo.n_exact, geo.nchunks))
      launch_dec_chunks<T, B, Rings<T>::kD>(packed, geo, segs, sp, offsets, prefix_rel, centers, exact, base, out,
                                            info, err, model, n_exact_dev, 0, s);
    else
      launch_dec_chunks<T, B, Rings<T>::kS>(packed, geo, segs, sp, offsets, prefix_rel, centers, exact, base, out, info,
                                       err, model, n_exact_dev, 0, s);
  } else {
    launch_dec_chunks<T, B, Rings<T>::kS>(packed, geo, segs, sp, offsets, prefix_rel, centers, exact, base, out, info,
                                     err, model, n_exact_dev, 1, s);
    launch_dec_chunks<T, B, Rings<T>::kD>(packed, geo, segs, sp, offsets, prefix_rel, centers, exact, base, out,
                                          info, err, model, n_exact_dev, 2, s);
  }
}

template <typename T>
static int dispatch_decode(int bits, const uint8_t* packed, const DecodeGeom& geo, const Seg* segs,
                           const SegParams& sp, uint32_t* counts, unsigned long long* offsets, void* scan_ws,
                           const unsigned long long* prefix_rel, const double* centers, const void* exact,
                           const void* base, void* out, nmk_segment_info* info, nmk_decode_err* err,
                           const nmk_model* model, const unsigned long long* n_exact_dev, int ring_hint,
                           cudaStream_t s) {
  switch (bits) {
#define NMK_DEC_CASE(BB)                                                                                    \
  case BB: launch_decode<T, BB>(packed, geo, segs, sp, counts, offsets, scan_ws, prefix_rel, centers, exact, \
                                base, out, info, err, model, n_exact_dev, ring_hint, s); break;
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

static int decode_impl(const uint8_t* packed, uint64_t block_stride, uint64_t first_block, int bits, uint64_t epb,
                       uint64_t n_total, const unsigned long long* prefix_rel, const double* centers, int k,
                       const nmk_model* model, const void* exact, uint64_t n_exact,
                       const unsigned long long* n_exact_dev, const void* base, void* out, int dtype,
                       const uint64_t* h_seg_start, const uint64_t* h_seg_count, const uint64_t* h_seg_out, int nseg,
                       nmk_segment_info* seg_info, nmk_decode_err* err, void* ws, size_t ws_bytes, cudaStream_t s,
                       int ring_hint = 0) {
  if (nseg < 1 || !h_seg_start || !h_seg_count || !h_seg_out || !seg_info || !err || !ws)
    return set_error(NMK_ERR_ARG, "nmk_decode: bad argument");
  if (bits < 2 || bits > 30 || epb == 0 || k < 1) return set_error(NMK_ERR_ARG, "nmk_decode: bad geometry");
  if (epb >= (1ULL << 31) || (n_total + kDChunk - 1) / kDChunk >= (1ULL << 32))
    return set_error(NMK_ERR_ARG, "nmk_decode: block or stream too large for 32-bit chunk indexing");
  if (block_stride % 16 || ((uintptr_t)packed & 15)) return set_error(NMK_ERR_ARG, "nmk_decode: packed alignment");
  if (dtype != NMK_F32 && dtype != NMK_F64) return set_error(NMK_ERR_ARG, "nmk_decode: bad dtype");
  for (int i = 0; i < nseg; ++i) {
    uint64_t st = h_seg_start[i], ct = h_seg_count[i];
    if (ct == 0 || st + ct > n_total || st / epb < first_block)
      return set_error(NMK_ERR_ARG, "nmk_decode: segment %d empty or outside the covered blocks", i);
  }
  if (!packed || !centers || !base || !out || !prefix_rel) return set_error(NMK_ERR_ARG, "nmk_decode: null pointer");
  const uint64_t dc = dtype == NMK_F32 ? 512 : 256;   // DecChunk<T>::kDC
  DecodePlan p = decode_plan(h_seg_start, h_seg_count, nseg, epb, first_block, dc);
  if (ws_bytes < p.total) return set_error(NMK_ERR_ARG, "nmk_decode: workspace too small");
  Seg* hs = (Seg*)malloc(sizeof(Seg) * (size_t)nseg);
  uint64_t item0 = 0;
  for (int i = 0; i < nseg; ++i) {
    const uint64_t st = h_seg_start[i], ct = h_seg_count[i], e = st + ct - 1;
    Seg sg;
    sg.start = st;
    sg.count = ct;
    sg.out = h_seg_out[i];
    sg.gfirst = (st / epb) * p.cpb_d + (st % epb) / dc;
    sg.item0 = item0;
    item0 += (e / epb) * p.cpb_d + (e % epb) / dc - sg.gfirst + 1;
    hs[i] = sg;
  }
  char* w = (char*)ws;
  uint32_t* counts = (uint32_t*)(w + p.off_counts);
  unsigned long long* offsets = (unsigned long long*)(w + p.off_offsets);
  Seg* dsegs = (Seg*)(w + p.off_segs);
  // a pageable H2D cudaMemcpyAsync returns after staging the source, so the
  // host table can be released immediately (no stream synchronisation)
  SegParams sp{};
  const bool by_value = model != nullptr && nseg <= NMK_DEV_MAX_SEG;
  if (by_value) {
    for (int i = 0; i < nseg; ++i) sp.s[i] = hs[i];
    dsegs = nullptr;   // no host->device copy: graph-capturable
  } else {
    cudaMemcpyAsync(dsegs, hs, sizeof(Seg) * (size_t)nseg, cudaMemcpyHostToDevice, s);
  }
  free(hs);
  DecodeGeom geo{};
  geo.epb = epb;
  geo.n_total = n_total;
  geo.first_block = first_block;
  geo.stride = block_stride;
  geo.n_exact = n_exact;
  geo.nchunks = p.nchunks;
  geo.nitems = p.nitems;
  geo.cpb = (uint32_t)p.cpb;
  geo.fd_cpb.init((uint32_t)p.cpb);
  geo.cpb_d = (uint32_t)p.cpb_d;
  geo.fd_cpb_d.init((uint32_t)p.cpb_d);
  geo.nseg = nseg;
  geo.k = k;
  // zeroed by the count pass (block 0) for the kernels behind it on the stream
  geo.zl.p[0] = (unsigned long long*)(w + p.off_scan);
  geo.zl.n[0] = chunk_scan_tiles(p.nchunks);
  geo.zl.p[1] = (unsigned long long*)seg_info;
  geo.zl.n[1] = (uint32_t)nseg * (uint32_t)(sizeof(nmk_segment_info) / 8);
  geo.zl.p[2] = (unsigned long long*)err;
  geo.zl.n[2] = (uint32_t)(sizeof(nmk_decode_err) / 8);
  if (dtype == NMK_F64)
    return dispatch_decode<double>(bits, packed, geo, dsegs, sp, counts, offsets, w + p.off_scan, prefix_rel,
                                   centers, exact, base, out, seg_info, err, model, n_exact_dev, ring_hint, s);
  return dispatch_decode<float>(bits, packed, geo, dsegs, sp, counts, offsets, w + p.off_scan, prefix_rel, centers,
                                exact, base, out, seg_info, err, model, n_exact_dev, ring_hint, s);
}

extern "C" int nmk_decode(const uint8_t* packed, uint64_t block_stride, uint64_t first_block, int bits,
                          uint64_t epb, uint64_t n_total, const unsigned long long* prefix_rel,
                          const double* centers, int k, const void* exact, uint64_t n_exact, const void* base,
                          void* out, int dtype, const uint64_t* h_seg_start, const uint64_t* h_seg_count,
                          const uint64_t* h_seg_out, int nseg, nmk_segment_info* seg_info,
                          nmk_decode_err* err, void* ws, size_t ws_bytes, void* stream) {
  return decode_impl(packed, block_stride, first_block, bits, epb, n_total, prefix_rel, centers, k, nullptr, exact,
                     n_exact, nullptr, base, out, dtype, h_seg_start, h_seg_count, h_seg_out, nseg, seg_info, err, ws,
                     ws_bytes, (cudaStream_t)stream);
}

extern "C" int nmk_decode_dev2(const uint8_t* packed, uint64_t block_stride, uint64_t first_block, int bits,
                               uint64_t epb, uint64_t n_total, const unsigned long long* prefix_rel,
                               const double* centers, const nmk_model* model, const void* exact,
                               const unsigned long long* n_exact, const void* base, void* out, int dtype,
                               const uint64_t* h_seg_start, const uint64_t* h_seg_count, const uint64_t* h_seg_out,
                               int nseg, nmk_segment_info* seg_info, nmk_decode_err* err, int ring_hint, void* ws,
                               size_t ws_bytes, void* stream) {
  if (!model || !n_exact) return set_error(NMK_ERR_ARG, "nmk_decode_dev: model and n_exact required");
  return decode_impl(packed, block_stride, first_block, bits, epb, n_total, prefix_rel, centers, 1, model, exact, 0,
                     n_exact, base, out, dtype, h_seg_start, h_seg_count, h_seg_out, nseg, seg_info, err, ws, ws_bytes,
                     (cudaStream_t)stream, ring_hint);
}

extern "C" int nmk_decode_dev(const uint8_t* packed, uint64_t block_stride, uint64_t first_block, int bits,
                              uint64_t epb, uint64_t n_total, const unsigned long long* prefix_rel,
                              const double* centers, const nmk_model* model, const void* exact,
                              const unsigned long long* n_exact, const void* base, void* out, int dtype,
                              const uint64_t* h_seg_start, const uint64_t* h_seg_count, const uint64_t* h_seg_out,
                              int nseg, nmk_segment_info* seg_info, nmk_decode_err* err, void* ws, size_t ws_bytes,
                              void* stream) {
  return nmk_decode_dev2(packed, block_stride, first_block, bits, epb, n_total, prefix_rel, centers, model, exact,
                         n_exact, base, out, dtype, h_seg_start, h_seg_count, h_seg_out, nseg, seg_info, err, 0, ws,
                         ws_bytes, stream);
}

// the ring depth nmk_decode_dev2's hint should name for a span of n_elems
// elements holding n_exact exact values (1 sparse, 2 dense)
extern "C" int nmk_decode_ring_for(uint64_t n_exact, uint64_t n_elems) {
  return dec_dense(n_exact, (n_elems + kDChunk - 1) / kDChunk) ? 2 : 1;
}
