// k_deflate.cu — optional GPU replacement of the lossless index-table stage
// (codec.compress_block, pkg/src/nmk/codec.py:108-116).
//
// Each index block (pipeline.py:290-304: one raw RFC 1951 stream per block)
// is cut into segments of seg_bytes.  One WARP compresses one segment:
//  * LZ77, 32 positions per step: every lane hashes the 3 bytes at its
//    position, reads the candidate the table held before this step, and the
//    lanes insert their positions (highest lane per hash value wins, so both
//    passes see the same table).  A lane extends three candidates -- the
//    previous byte (runs), the last distance used (periodic B-bit codes) and
//    the hash candidate -- 4 bytes per compare.  The greedy parse over the
//    step's 32 results is done with ballots: literals up to the next lane
//    holding a match leave together, the match jumps the cursor.
//  * pass 1 counts symbols (shared-memory atomics); the segment's own
//    length-limited Huffman codes are built by a warp-parallel rank sort and
//    a two-queue merge; pass 2 repeats the parse and emits: every lane turns
//    its token into <= 48 bits, a warp scan gives the bit offsets, the bits
//    are OR-ed into a shared-memory ring whose complete words are flushed
//    coalesced.  The fixed code (BTYPE = 01) is used when not larger.
// The segment's block is closed with the end-of-block symbol followed by an
// empty stored block (BTYPE = 00, LEN = 0), which byte-aligns the bit stream
// -- so the segments of a block concatenate into one valid raw DEFLATE stream
// by a plain byte copy (the last segment's stored block carries BFINAL).  Any
// inflater (zlib included) reproduces the packed bytes exactly; the
// compressed bytes differ from zlib's, which the reference does not pin
// (SURVEY 8c), so this stage is opt-in.
//
// Pipeline: k_deflate_segments (warp per segment) -> chunk_scan over segment
// lengths -> k_deflate_gather (warp per segment into the compact output).
#include <type_traits>

#include "nmk_common.cuh"
#include "nmk_scan.cuh"

namespace nmk {

#ifndef NMK_DEF_WARPS
#define NMK_DEF_WARPS 4
#endif
constexpr int kDefWarps = NMK_DEF_WARPS;
constexpr int kDefThreads = 32 * kDefWarps;
#ifndef NMK_DEF_LONGHASH
// The two u16 slots of a bucket word are two tables: slot 0 keyed by the next
// NMK_DEF_SHORTLEN bytes, slot 1 by the next NMK_DEF_LONGLEN.  Index streams
// reward long contexts (their short repeats cost more than literals): against
// a two-way 3-byte table, (6, 10) takes cfg3 (B = 10) from ratio 6.23 to 7.40
// and cfg2 from 6.21 to 6.28, and is faster (fewer useless candidates).
// A/B: (3,8) 7.13 / 6.23, (4,8) 7.20 / 6.25, (6,8) 7.29 / 6.28, (6,12) 7.39 / 6.26.
#define NMK_DEF_LONGHASH 1
#endif
#ifndef NMK_DEF_LONGLEN
#define NMK_DEF_LONGLEN 10   // bytes under the second table's hash (5..12)
#endif
constexpr uint32_t kLongMask = NMK_DEF_LONGLEN >= 8 ? 0xffffffffu : ((1u << (8 * (NMK_DEF_LONGLEN - 4))) - 1u);
constexpr uint32_t kLongMask2 = NMK_DEF_LONGLEN >= 12 || NMK_DEF_LONGLEN <= 8 ? 0xffffffffu : ((1u << (8 * (NMK_DEF_LONGLEN - 8))) - 1u);
#ifndef NMK_DEF_SHORTLEN
#define NMK_DEF_SHORTLEN 6   // bytes under the first table's hash (3..6)
#endif
#ifndef NMK_DEF_WAYS
#define NMK_DEF_WAYS 2   // u16 positions per bucket word: 2 (one per table, 2048 u32 buckets) or 4 (two per table,
                         // 1024 u64 buckets; A/B: cfg3 ratio 7.40 -> 7.56, cfg2 unchanged, 28-40 % slower)
#endif
constexpr int kDefWays = NMK_DEF_WAYS;
constexpr int kDefHashBits = kDefWays == 4 ? 10 : 11;
constexpr int kDefHash = 1 << kDefHashBits;      // buckets of kDefWays u16 positions (newest low): 8 KB per warp
typedef typename std::conditional<kDefWays == 4, unsigned long long, uint32_t>::type bucket_t;
constexpr uint32_t kNoPos = 0xffffu;
constexpr bucket_t kEmptyBucket = (bucket_t)~(bucket_t)0;
constexpr int kMinMatch = 3, kMaxMatch = 258;
// estimated bits of a match's length symbol / a near (1 or repeated) / any other distance symbol,
// and the length from which a match is always taken (tuned on cfg2's index stream: ratio 4.9 -> 6.4 in a CPU model)
constexpr int kProbe = 32;   // bytes a lane compares per candidate
#ifndef NMK_DEF_COSTLONG
#define NMK_DEF_COSTLONG 24   // matches shorter than this pass the literal-cost filter (0: off -- cfg2 ratio 6.21 -> 5.21)
#endif
constexpr uint32_t kCostLen = 4, kCostNear = 1, kCostDist = 6, kCostLong = NMK_DEF_COSTLONG;
constexpr int kStageWords = 128;                 // output bit ring per warp (a step emits <= 17 words)
constexpr unsigned FULLW = 0xffffffffu;

// worst case of one segment: the fixed code (chosen whenever the dynamic one
// is not smaller) spends <= 9 bits per byte, plus the block headers,
// end-of-block and the empty stored block, rounded up to 16 bytes
__host__ __device__ inline uint32_t seg_bound(uint32_t seg_bytes) { return ((seg_bytes * 9 + 7) / 8 + 32 + 15) & ~15u; }

__device__ __forceinline__ uint32_t rev_bits(uint32_t v, int len) { return __brev(v) >> (32 - len); }

// fixed literal/length code (RFC 1951 3.2.6), returned bit-reversed for LSB-first output
__device__ __forceinline__ void fixed_litlen(uint32_t sym, uint32_t& code, int& len) {
  if (sym < 144) { code = 0x30 + sym; len = 8; }
  else if (sym < 256) { code = 0x190 + (sym - 144); len = 9; }
  else if (sym < 280) { code = sym - 256; len = 7; }
  else { code = 0xC0 + (sym - 280); len = 8; }
  code = rev_bits(code, len);
}

__device__ __forceinline__ uint32_t hash3(uint32_t v) {
  return ((NMK_DEF_SHORTLEN >= 4 ? v : v & 0xffffffu) * 2654435761u) >> (32 - kDefHashBits);
}

// length 3..258 -> litlen symbol, extra bits, extra value (RFC 1951 3.2.5)
__device__ __forceinline__ void len_symbol(uint32_t len, uint32_t& sym, uint32_t& ebits, uint32_t& eval) {
  ebits = eval = 0;
  if (len == 258) {
    sym = 285;
  } else if (len <= 10) {
    sym = 257 + (len - 3);
  } else {
    const uint32_t l = len - 3;
    const int e = 31 - __clz(l) - 2;
    sym = 261 + 4 * e + ((l >> e) & 3);
    ebits = (uint32_t)e;
    eval = l & ((1u << e) - 1);
  }
}
// distance 1..32768 -> code, extra bits, extra value
__device__ __forceinline__ void dist_symbol(uint32_t dist, uint32_t& code, uint32_t& ebits, uint32_t& eval) {
  const uint32_t d = dist - 1;
  ebits = eval = 0;
  if (d < 4) {
    code = d;
  } else {
    const int e = 31 - __clz(d) - 1;
    code = 2 * (uint32_t)e + 2 + ((d >> e) & 1);
    ebits = (uint32_t)e;
    eval = d & ((1u << e) - 1);
  }
}

// ---- per-warp shared memory ----------------------------------------------------
constexpr int kHuffMax = 288;
struct HuffWork {          // scratch of the code construction (aliases the hash table between the passes)
  uint32_t f0[kHuffMax];   // used symbols' frequencies, symbol order
  uint32_t f[kHuffMax];    // sorted by (frequency, symbol)
  uint32_t nf[2 * kHuffMax];
  uint16_t leaf0[kHuffMax], leaf[kHuffMax];
  uint16_t par[2 * kHuffMax];
  uint8_t dep[2 * kHuffMax];
};
struct __align__(16) DefWarp {
  union {
    bucket_t hash[kDefHash];
    HuffWork hw;
  };
  uint32_t lf[kHuffMax];   // literal/length symbol counts
  uint32_t df[32];         // distance symbol counts
  uint32_t cf[32];         // code-length symbol counts
  uint32_t stage[kStageWords];
  uint16_t lc[kHuffMax], dc[32], cc[32];   // codes (bit-reversed)
  uint8_t ll[kHuffMax], dl[32], cl[32];    // code lengths
  uint8_t rs[320], rx[320];                // run-length coded code lengths and their extra values
  uint16_t cost[256];                      // literal cost estimate, 1/8 bit: -log2 of the byte's share of the segment
};
static_assert(kCostLong <= (uint32_t)kProbe, "the cost filter reads the probe window");
static_assert(sizeof(HuffWork) <= kDefHash * sizeof(bucket_t), "Huffman scratch must fit the hash table");

// bytes p .. p + 3 of the segment (little-endian); words beyond the segment read 0
__device__ __forceinline__ uint32_t word_at(const uint32_t* __restrict__ W, uint32_t nw, uint32_t p) {
  const uint32_t k = p >> 2;
  const uint32_t a = k < nw ? __ldg(W + k) : 0u;
  const uint32_t b = k + 1 < nw ? __ldg(W + k + 1) : 0u;
  return __funnelshift_r(a, b, (p & 3u) * 8u);
}

// common prefix of the bytes at j and i (j < i), at most maxl
__device__ __forceinline__ uint32_t extend(const uint32_t* __restrict__ W, uint32_t nw, uint32_t j, uint32_t i,
                                           uint32_t maxl) {
  uint32_t l = 0;
  while (l < maxl) {
    const uint32_t x = word_at(W, nw, j + l) ^ word_at(W, nw, i + l);
    if (x) {
      l += (uint32_t)(__ffs((int)x) - 1) >> 3;
      break;
    }
    l += 4;
  }
  return min(l, maxl);
}

// The whole warp extends one match beyond the l0 bytes already known equal:
// lane l compares bytes l0 + 4 l .. + 3 of each 128-byte stretch.
__device__ __forceinline__ uint32_t extend_coop(const uint32_t* __restrict__ W, uint32_t nw, uint32_t j, uint32_t i,
                                                uint32_t maxl, uint32_t l0, int lane) {
  uint32_t l = l0;
  while (l < maxl) {
    const uint32_t k = l + 4u * (uint32_t)lane;
    const uint32_t x = k < maxl ? word_at(W, nw, j + k) ^ word_at(W, nw, i + k) : 0u;
    const unsigned mm = __ballot_sync(FULLW, x != 0u);
    if (mm) {
      const int f = __ffs((int)mm) - 1;
      const uint32_t xf = __shfl_sync(FULLW, x, f);
      l += 4u * (uint32_t)f + ((uint32_t)(__ffs((int)xf) - 1) >> 3);
      break;
    }
    l += 128u;
  }
  return min(l, maxl);
}

// Warp-cooperative LZ77 over one segment.  `tokens(nlit_lo, nlit_hi, byte, mlane, len, dist)`
// is called warp-uniformly once per parse step: lanes in [nlit_lo, nlit_hi)
// each hold a literal (`byte` = their own), and lane `mlane` (32: none) holds
// a match (len, dist) that follows those literals.  Deterministic: both passes
// produce the same token sequence.
template <typename Tokens>
__device__ __forceinline__ void lz77_warp(const uint32_t* __restrict__ W, uint32_t n, bucket_t* hash,
                                          const uint16_t* cost, int lane, Tokens&& tokens) {
  const uint32_t nw = (n + 3) >> 2;
  for (int k = lane; k < kDefHash; k += 32) hash[k] = kEmptyBucket;
  __syncwarp();
  uint32_t pos = 0, rep = 0;
  while (pos < n) {
    const uint32_t i = pos + lane;
    const bool valid = i < n;
    // the lane's own kProbe bytes, read once for all of its candidates
    uint32_t a[kProbe / 4];
    {
      uint32_t v[kProbe / 4 + 1];
      const uint32_t k0 = i >> 2;
#pragma unroll
      for (int q = 0; q <= kProbe / 4; ++q) v[q] = (valid && k0 + q < nw) ? __ldg(W + k0 + q) : 0u;
#pragma unroll
      for (int q = 0; q < kProbe / 4; ++q) a[q] = __funnelshift_r(v[q], v[q + 1], (i & 3u) * 8u);
    }
    const uint32_t w0 = a[0];
    const bool hashed = valid && i + kMinMatch <= n;
    uint32_t h = hash3(w0);
    if (NMK_DEF_SHORTLEN > 4)
      h = ((w0 * 2654435761u) ^ ((a[1] & ((1u << (8 * (NMK_DEF_SHORTLEN - 4))) - 1u)) * 2246822519u)) >> (32 - kDefHashBits);
#if NMK_DEF_LONGHASH
    // two tables in one array: a bucket word's first half is keyed by the next
    // NMK_DEF_SHORTLEN bytes, its second half by the next NMK_DEF_LONGLEN
    // (one u16 position each with 2 ways, two -- newest low -- with 4)
    const bool hashed8 = valid && i + NMK_DEF_LONGLEN <= n;
    uint32_t hl = (a[0] * 2654435761u) ^ ((NMK_DEF_LONGLEN >= 8 ? a[1] : a[1] & kLongMask) * 2246822519u);
    if (NMK_DEF_LONGLEN > 8) hl ^= (NMK_DEF_LONGLEN >= 12 ? a[2] : a[2] & kLongMask2) * 3266489917u;
    hl >>= 32 - kDefHashBits;
    const unsigned grp = __match_any_sync(FULLW, hashed ? h : (0x80000000u | (uint32_t)lane));
    const unsigned grp8 = __match_any_sync(FULLW, hashed8 ? hl : (0x80000000u | (uint32_t)lane));
    bucket_t bucket;   // the tables as they were before this step
    if constexpr (kDefWays == 2) {
      uint16_t* h16 = reinterpret_cast<uint16_t*>(hash);
      const uint32_t c3 = hashed ? h16[2 * h] : kNoPos, c8 = hashed8 ? h16[2 * hl + 1] : kNoPos;
      bucket = (bucket_t)c3 | ((bucket_t)c8 << 16);
      __syncwarp();
      if (hashed && lane == 31 - __clz(grp)) h16[2 * h] = (uint16_t)i;        // highest lane (latest position) wins
      if (hashed8 && lane == 31 - __clz(grp8)) h16[2 * hl + 1] = (uint16_t)i;
    } else {
      uint32_t* h32 = reinterpret_cast<uint32_t*>(hash);
      const uint32_t c3 = hashed ? h32[2 * h] : 0xffffffffu, c8 = hashed8 ? h32[2 * hl + 1] : 0xffffffffu;
      bucket = (bucket_t)c3 | ((bucket_t)c8 << 32);
      __syncwarp();
      if (hashed && lane == 31 - __clz(grp)) h32[2 * h] = (c3 << 16) | i;
      if (hashed8 && lane == 31 - __clz(grp8)) h32[2 * hl + 1] = (c8 << 16) | i;
    }
    __syncwarp();
#else
    const bucket_t bucket = hashed ? hash[h] : kEmptyBucket;   // the table as it was before this step
    __syncwarp();
    const unsigned grp = __match_any_sync(FULLW, hashed ? h : (0x80000000u | (uint32_t)lane));
    if (hashed && lane == 31 - __clz(grp)) hash[h] = (bucket_t)(bucket << 16) | (bucket_t)i;   // highest lane (latest position) wins
    __syncwarp();
#endif
    uint32_t best = 0, bd = 0;
    if (hashed) {
      // lanes measure their candidates up to kProbe bytes (all loads of a
      // candidate in flight together); the match the parse takes is then
      // extended to its full length by the whole warp
      const uint32_t maxl = min((uint32_t)kProbe, n - i);
      auto consider = [&](uint32_t d) {
        if (best >= maxl || d == 0 || d > i || d > 32768u) return;
        const uint32_t j = i - d, k0 = j >> 2;
        uint32_t v[kProbe / 4 + 1];
#pragma unroll
        for (int q = 0; q <= kProbe / 4; ++q) v[q] = k0 + q < nw ? __ldg(W + k0 + q) : 0u;
        uint32_t l = kProbe;
#pragma unroll
        for (int q = kProbe / 4 - 1; q >= 0; --q) {
          const uint32_t x = a[q] ^ __funnelshift_r(v[q], v[q + 1], (j & 3u) * 8u);
          if (x) l = 4u * q + ((uint32_t)(__ffs((int)x) - 1) >> 3);
        }
        l = min(l, maxl);
        if (l > best) { best = l; bd = d; }
      };
      consider(1);                                   // runs
      if (rep > 1) consider(rep);                    // the last distance used (periodic codes)
      const unsigned lower = grp & ((1u << lane) - 1u);
      const uint32_t d_in = lower ? (uint32_t)(lane - (31 - __clz(lower))) : 0u;   // same hash earlier in this step
      if (d_in > 1 && d_in != rep) consider(d_in);
#pragma unroll
      for (int w = 0; w < kDefWays; ++w) {
        const uint32_t j = (uint32_t)(bucket >> (16 * w)) & 0xffffu;
        if (j == kNoPos) continue;
        const uint32_t d = i - j;
        if (d != 1 && d != rep && d != d_in) consider(d);
      }
      if (best == (uint32_t)kMinMatch && bd > 4096u) best = 0;   // a far 3-byte match costs more than 3 literals
      // Index streams are dominated by one or two byte values whose Huffman
      // codes take 1-2 bits, so a short match is often dearer than its bytes
      // as literals (zlib level 1-3 loses to Huffman-only on them): keep a
      // short match only if its estimated cost beats the literals' (1/8 bit).
      if (best >= (uint32_t)kMinMatch && best < (uint32_t)kCostLong) {
        uint32_t litc = 0;
#pragma unroll
        for (int w = 0; w < (int)(kCostLong + 3) / 4 && w < kProbe / 4; ++w) {   // the match's bytes are in a[]
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if ((uint32_t)(4 * w + q) < best) litc += cost[(a[w] >> (8 * q)) & 0xffu];
        }
        uint32_t sy, ebl, ebd, ev;
        len_symbol(best, sy, ebl, ev);
        dist_symbol(bd, sy, ebd, ev);
        const uint32_t mc = 8u * (kCostLen + ebl + ((bd == 1 || bd == rep) ? kCostNear : kCostDist + ebd));
        if (mc >= litc) best = 0;
      }
    }
    const unsigned m3 = __ballot_sync(FULLW, best >= (uint32_t)kMinMatch);
    const uint32_t lim = min(32u, n - pos);   // positions of this step inside the segment
    uint32_t c = 0, scan = 0;
    while (true) {
      const unsigned ahead = scan < 32 ? (m3 >> scan) << scan : 0u;
      const uint32_t nxt = ahead ? (uint32_t)__ffs((int)ahead) - 1u : 32u;
      if (nxt >= lim) {   // literals to the end of the step
        tokens(c, lim, w0 & 0xffu, 32u, 0u, 0u);
        c = lim;
        break;
      }
      uint32_t L = __shfl_sync(FULLW, best, (int)nxt);
      const uint32_t D = __shfl_sync(FULLW, bd, (int)nxt);
      if (nxt + 1 < lim && L < (uint32_t)kProbe) {   // lazy: a longer match one byte later wins
        const uint32_t L1 = __shfl_sync(FULLW, best, (int)nxt + 1);
        if (L1 > L) {
          scan = nxt + 1;
          continue;
        }
      }
      if (L == (uint32_t)kProbe) {
        const uint32_t ip = pos + nxt;
        L = extend_coop(W, nw, ip - D, ip, min((uint32_t)kMaxMatch, n - ip), L, lane);
      }
      tokens(c, nxt, w0 & 0xffu, nxt, L, D);
      rep = D;
      c = nxt + L;
      scan = c;
      if (c >= lim) break;
    }
    pos += c;
  }
}

// ---- Huffman code lengths <= maxlen for freq[0 .. nsym), whole warp -------------
// Used symbols are ranked by (frequency, symbol) with an all-pairs count (each
// lane ranks its symbols), lane 0 runs the two-queue merge over the sorted
// leaves and the depths; frequencies are halved (>= 1) until the depth fits.
// A lone used symbol gets a partner so every code is complete.
__device__ void huff_lengths_warp(const uint32_t* freq, int nsym, int maxlen, uint8_t* len, HuffWork& hw, int lane) {
  int m = 0;
  for (int s0 = 0; s0 < nsym; s0 += 32) {
    const int s = s0 + lane;
    const bool used = s < nsym && freq[s] != 0;
    if (s < nsym) len[s] = 0;
    const unsigned mk = __ballot_sync(FULLW, used);
    if (used) {
      const int idx = m + __popc(mk & ((1u << lane) - 1u));
      hw.leaf0[idx] = (uint16_t)s;
      hw.f0[idx] = freq[s];
    }
    m += __popc(mk);
  }
  __syncwarp();
  if (m == 0) return;
  if (m == 1) {   // one symbol: length 1 plus an unused partner of length 1
    if (lane == 0) {
      const int s = hw.leaf0[0];
      len[s] = 1;
      len[s == 0 ? 1 : 0] = 1;
    }
    __syncwarp();
    return;
  }
  for (;;) {
    for (int a = lane; a < m; a += 32) {   // leaves are in symbol order: ties rank by index
      const uint32_t fa = hw.f0[a];
      int r = 0;
      for (int b = 0; b < m; ++b) {
        const uint32_t fb = hw.f0[b];
        r += (fb < fa) || (fb == fa && b < a);
      }
      hw.f[r] = fa;
      hw.leaf[r] = hw.leaf0[a];
    }
    __syncwarp();
    int maxd = 0;
    if (lane == 0) {
      for (int a = 0; a < m; ++a) hw.nf[a] = hw.f[a];
      int li = 0, ii = m, nn = m;
      auto take = [&]() -> int {
        if (li < m && (ii >= nn || hw.nf[li] <= hw.nf[ii])) return li++;
        return ii++;
      };
      while (nn < 2 * m - 1) {
        const int x = take(), y = take();
        hw.nf[nn] = hw.nf[x] + hw.nf[y];
        hw.par[x] = hw.par[y] = (uint16_t)nn;
        ++nn;
      }
      hw.dep[nn - 1] = 0;
      for (int k = nn - 2; k >= 0; --k) {
        const int d = hw.dep[hw.par[k]] + 1;
        hw.dep[k] = (uint8_t)d;
        if (k < m && d > maxd) maxd = d;
      }
    }
    maxd = __shfl_sync(FULLW, maxd, 0);
    __syncwarp();
    if (maxd <= maxlen) {
      for (int a = lane; a < m; a += 32) len[hw.leaf[a]] = hw.dep[a];
      __syncwarp();
      return;
    }
    for (int a = lane; a < m; a += 32) hw.f0[a] = max(1u, hw.f0[a] >> 1);
    __syncwarp();
  }
}

// canonical codes (RFC 1951 3.2.2), bit-reversed for LSB-first output (lane 0)
__device__ void huff_codes(const uint8_t* len, int nsym, uint16_t* code) {
  uint32_t cnt[16] = {0}, next[16];
  for (int s = 0; s < nsym; ++s) ++cnt[len[s]];
  cnt[0] = 0;
  uint32_t c = 0;
  next[0] = 0;
  for (int b = 1; b < 16; ++b) {
    c = (c + cnt[b - 1]) << 1;
    next[b] = c;
  }
  for (int s = 0; s < nsym; ++s)
    code[s] = len[s] ? (uint16_t)rev_bits(next[len[s]]++, len[s]) : 0;
}

__constant__ uint8_t kClOrder[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};

// Every lane with nb > 0 appends its nb (<= 48) bits v, in lane order, at
// *bitpos of the segment's output; complete 32-bit words leave the ring.
__device__ __forceinline__ void emit_bits(unsigned long long v, uint32_t nb, uint32_t& bitpos, uint32_t* stage,
                                          uint32_t* __restrict__ out, int lane) {
  uint32_t incl = nb;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULLW, incl, o);
    if (lane >= o) incl += y;
  }
  const uint32_t total = __shfl_sync(FULLW, incl, 31);
  if (nb) {
    const uint32_t o = bitpos + incl - nb;
    const uint32_t w = o >> 5, s = o & 31u;
    atomicOr(&stage[w & (kStageWords - 1)], (uint32_t)(v << s));
    const unsigned long long rest = s ? (v >> (32u - s)) : (v >> 32);
    if (rest) {
      atomicOr(&stage[(w + 1) & (kStageWords - 1)], (uint32_t)rest);
      if (rest >> 32) atomicOr(&stage[(w + 2) & (kStageWords - 1)], (uint32_t)(rest >> 32));
    }
  }
  __syncwarp();
  const uint32_t w0 = bitpos >> 5, w1 = (bitpos + total) >> 5;
  for (uint32_t w = w0 + lane; w < w1; w += 32) {
    out[w] = stage[w & (kStageWords - 1)];
    stage[w & (kStageWords - 1)] = 0u;
  }
  __syncwarp();
  bitpos += total;
}

__global__ void __launch_bounds__(kDefThreads)
k_deflate_segments(const uint8_t* __restrict__ packed, uint64_t stride, uint64_t nblocks, uint64_t block_len,
                   uint64_t last_len, uint32_t seg_bytes, uint32_t segs_per_block, uint8_t* __restrict__ scratch,
                   uint32_t* __restrict__ seg_len) {
  extern __shared__ __align__(16) uint8_t s_def[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  DefWarp& m = reinterpret_cast<DefWarp*>(s_def)[wid];
  const uint64_t nseg = nblocks * segs_per_block;
  for (uint64_t sg = (uint64_t)blockIdx.x * kDefWarps + wid; sg < nseg; sg += (uint64_t)gridDim.x * kDefWarps) {
    const uint64_t b = sg / segs_per_block;
    const uint32_t s = (uint32_t)(sg - b * segs_per_block);
    const uint64_t blen = (b + 1 == nblocks) ? last_len : block_len;
    const uint64_t lo = (uint64_t)s * seg_bytes;
    if (lo >= blen) {   // segment past a short last block: nothing
      if (lane == 0) seg_len[sg] = 0;
      continue;
    }
    const uint32_t n = (uint32_t)min((uint64_t)seg_bytes, blen - lo);
    const bool last = lo + n == blen;
    // the segment starts 16-byte aligned (stride and seg_bytes are multiples of 16)
    const uint32_t* W = reinterpret_cast<const uint32_t*>(packed + b * stride + lo);
    uint32_t* out = reinterpret_cast<uint32_t*>(scratch + sg * (uint64_t)seg_bound(seg_bytes));

    // ---- pass 0: byte shares -> literal cost estimates ----
    for (int k = lane; k < 256; k += 32) m.lf[k] = 0;
    __syncwarp();
    for (uint32_t w = lane; w < ((n + 3) >> 2); w += 32) {
      const uint32_t x = __ldg(W + w);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (4 * w + q < n) atomicAdd(&m.lf[(x >> (8 * q)) & 0xffu], 1u);
    }
    __syncwarp();
    {
      const float lgn = __log2f((float)n);
      for (int k = lane; k < 256; k += 32) {
        const uint32_t c = m.lf[k];
        m.cost[k] = (uint16_t)(c ? __float2int_rn(8.0f * (lgn - __log2f((float)c))) : 255);
      }
    }
    __syncwarp();
    // ---- pass 1: symbol statistics ----
    for (int k = lane; k < kHuffMax; k += 32) m.lf[k] = 0;
    m.df[lane] = 0;
    m.cf[lane] = 0;
    for (int k = lane; k < kStageWords; k += 32) m.stage[k] = 0;
    __syncwarp();
    lz77_warp(W, n, m.hash, m.cost, lane, [&](uint32_t c0, uint32_t c1, uint32_t byte, uint32_t ml, uint32_t L, uint32_t D) {
      if ((uint32_t)lane >= c0 && (uint32_t)lane < c1) atomicAdd(&m.lf[byte], 1u);
      if ((uint32_t)lane == ml) {
        uint32_t sy, eb, ev;
        len_symbol(L, sy, eb, ev);
        atomicAdd(&m.lf[sy], 1u);
        dist_symbol(D, sy, eb, ev);
        atomicAdd(&m.df[sy], 1u);
      }
    });
    if (lane == 0) m.lf[256] = 1;   // end of block
    __syncwarp();

    // ---- dynamic code: lengths, run-length coded lengths, their code ----
    huff_lengths_warp(m.lf, 286, 15, m.ll, m.hw, lane);
    huff_lengths_warp(m.df, 30, 15, m.dl, m.hw, lane);
    int hlit = 0, hdist = 0, nr = 0;
    if (lane == 0) {
      hlit = 286;
      hdist = 30;
      while (hlit > 257 && m.ll[hlit - 1] == 0) --hlit;
      while (hdist > 1 && m.dl[hdist - 1] == 0) --hdist;
      auto LN = [&](int i) -> uint32_t { return i < hlit ? m.ll[i] : m.dl[i - hlit]; };
      const int tot = hlit + hdist;
      int i = 0;
      while (i < tot) {
        const uint32_t v = LN(i);
        int run = 1;
        while (i + run < tot && LN(i + run) == v) ++run;
        if (v == 0) {
          int r = run;
          while (r >= 11) { const int t = min(r, 138); m.rs[nr] = 18; m.rx[nr++] = (uint8_t)(t - 11); r -= t; }
          if (r >= 3) { m.rs[nr] = 17; m.rx[nr++] = (uint8_t)(r - 3); r = 0; }
          while (r > 0) { m.rs[nr] = 0; m.rx[nr++] = 0; --r; }
        } else {
          m.rs[nr] = (uint8_t)v; m.rx[nr++] = 0;
          int r = run - 1;
          while (r >= 3) { const int t = min(r, 6); m.rs[nr] = 16; m.rx[nr++] = (uint8_t)(t - 3); r -= t; }
          while (r > 0) { m.rs[nr] = (uint8_t)v; m.rx[nr++] = 0; --r; }
        }
        i += run;
      }
      for (int k = 0; k < nr; ++k) ++m.cf[m.rs[k]];
    }
    hlit = __shfl_sync(FULLW, hlit, 0);
    hdist = __shfl_sync(FULLW, hdist, 0);
    nr = __shfl_sync(FULLW, nr, 0);
    __syncwarp();
    huff_lengths_warp(m.cf, 19, 7, m.cl, m.hw, lane);
    int hclen = 19;
    while (hclen > 4 && m.cl[kClOrder[hclen - 1]] == 0) --hclen;
    // cost of the two encodings (extra bits are the same for both)
    unsigned long long dyn = 0, fix = 0;
    for (int k = lane; k < nr; k += 32) {
      const uint32_t r = m.rs[k];
      dyn += m.cl[r] + (r == 16 ? 2 : r == 17 ? 3 : r == 18 ? 7 : 0);
    }
    for (int k = lane; k < 286; k += 32) {
      const unsigned long long f = m.lf[k];
      dyn += f * m.ll[k];
      fix += f * (k < 144 ? 8 : k < 256 ? 9 : k < 280 ? 7 : 8);
    }
    if (lane < 30) { dyn += (unsigned long long)m.df[lane] * m.dl[lane]; fix += (unsigned long long)m.df[lane] * 5; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      dyn += __shfl_xor_sync(FULLW, dyn, o);
      fix += __shfl_xor_sync(FULLW, fix, o);
    }
    dyn += 14 + 3 * (unsigned long long)hclen;
    const bool use_dyn = dyn < fix;

    // ---- pass 2: emit ----
    uint32_t bitpos = 0;
    if (use_dyn) {
      if (lane == 0) {
        huff_codes(m.ll, 286, m.lc);
        huff_codes(m.dl, 30, m.dc);
        huff_codes(m.cl, 19, m.cc);
      }
      __syncwarp();
      // BFINAL = 0, BTYPE = 10 | HLIT | HDIST | HCLEN
      const uint32_t hdr = 0u | (2u << 1) | ((uint32_t)(hlit - 257) << 3) | ((uint32_t)(hdist - 1) << 8) |
                           ((uint32_t)(hclen - 4) << 13);
      emit_bits(hdr, lane == 0 ? 17u : 0u, bitpos, m.stage, out, lane);
      emit_bits(lane < hclen ? m.cl[kClOrder[lane < 19 ? lane : 0]] : 0u, lane < hclen ? 3u : 0u, bitpos, m.stage, out,
                lane);
      for (int k0 = 0; k0 < nr; k0 += 32) {
        const int k = k0 + lane;
        unsigned long long v = 0;
        uint32_t nb = 0;
        if (k < nr) {
          const uint32_t r = m.rs[k];
          nb = m.cl[r];
          v = m.cc[r];
          const uint32_t xb = r == 16 ? 2u : r == 17 ? 3u : r == 18 ? 7u : 0u;
          v |= (unsigned long long)m.rx[k] << nb;
          nb += xb;
        }
        emit_bits(v, nb, bitpos, m.stage, out, lane);
      }
    } else {
      for (int k = lane; k < 286; k += 32) {
        uint32_t c;
        int l;
        fixed_litlen((uint32_t)k, c, l);
        m.lc[k] = (uint16_t)c;
        m.ll[k] = (uint8_t)l;
      }
      if (lane < 30) { m.dc[lane] = (uint16_t)rev_bits((uint32_t)lane, 5); m.dl[lane] = 5; }
      __syncwarp();
      emit_bits(0u | (1u << 1), lane == 0 ? 3u : 0u, bitpos, m.stage, out, lane);   // BFINAL = 0, BTYPE = 01
    }
    lz77_warp(W, n, m.hash, m.cost, lane, [&](uint32_t c0, uint32_t c1, uint32_t byte, uint32_t ml, uint32_t L, uint32_t D) {
      unsigned long long v = 0;
      uint32_t nb = 0;
      if ((uint32_t)lane >= c0 && (uint32_t)lane < c1) {
        v = m.lc[byte];
        nb = m.ll[byte];
      } else if ((uint32_t)lane == ml) {
        uint32_t sy, eb, ev;
        len_symbol(L, sy, eb, ev);
        v = m.lc[sy];
        nb = m.ll[sy];
        v |= (unsigned long long)ev << nb;
        nb += eb;
        dist_symbol(D, sy, eb, ev);
        v |= (unsigned long long)m.dc[sy] << nb;
        nb += m.dl[sy];
        v |= (unsigned long long)ev << nb;
        nb += eb;
      }
      emit_bits(v, nb, bitpos, m.stage, out, lane);
    });
    // end of block, then an empty stored block byte-aligns the stream (BFINAL
    // on the last segment): 3 header bits, zero padding, LEN = 0, NLEN = 0xffff
    {
      unsigned long long v = m.lc[256];
      uint32_t nb = m.ll[256];
      v |= (unsigned long long)(last ? 1u : 0u) << nb;
      nb += 3;
      emit_bits(v, lane == 0 ? nb : 0u, bitpos, m.stage, out, lane);
      const uint32_t pad = (8u - (bitpos & 7u)) & 7u;
      emit_bits(0xffff0000ULL << pad, lane == 0 ? pad + 32u : 0u, bitpos, m.stage, out, lane);
    }
    if (lane == 0) {
      if (bitpos & 31u) out[bitpos >> 5] = m.stage[(bitpos >> 5) & (kStageWords - 1)];   // the partial word
      seg_len[sg] = bitpos >> 3;
    }
    __syncwarp();
  }
}

// warp per segment: copy its bytes to the compact output at offsets[sg]
__global__ void __launch_bounds__(256)
k_deflate_gather(const uint8_t* __restrict__ scratch, const uint32_t* __restrict__ seg_len,
                 const unsigned long long* __restrict__ offsets, uint64_t nseg, uint32_t seg_bytes,
                 uint32_t segs_per_block, uint8_t* __restrict__ out, unsigned long long* __restrict__ block_off,
                 uint64_t nblocks) {
  const int lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t sg = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; sg < nseg; sg += nw) {
    const uint32_t len = seg_len[sg];
    const unsigned long long o = offsets[sg];
    const uint8_t* src = scratch + sg * (uint64_t)seg_bound(seg_bytes);
    for (uint32_t k = lane; k < len; k += 32) out[o + k] = src[k];
    if (lane == 0 && sg % segs_per_block == 0) block_off[sg / segs_per_block] = o;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) block_off[nblocks] = offsets[nseg];
}

static size_t al256d(size_t x) { return (x + 255) & ~(size_t)255; }

struct DeflatePlan {
  uint64_t segs_per_block, nseg;
  size_t off_scratch, off_len, off_offsets, off_scan, total;
};

static DeflatePlan deflate_plan(uint64_t nblocks, uint64_t block_len, uint32_t seg_bytes) {
  DeflatePlan p{};
  p.segs_per_block = (block_len + seg_bytes - 1) / seg_bytes;
  p.nseg = p.segs_per_block * nblocks;
  p.off_scratch = 0;
  p.off_len = al256d(p.nseg * (size_t)seg_bound(seg_bytes));
  p.off_offsets = p.off_len + al256d(p.nseg * 4);
  p.off_scan = p.off_offsets + al256d(p.nseg * 8 + 8);
  p.total = p.off_scan + al256d(chunk_scan_ws_bytes(p.nseg));
  return p;
}

}  // namespace nmk

using namespace nmk;

extern "C" size_t nmk_deflate_ws_bytes(uint64_t nblocks, uint64_t block_len, uint32_t seg_bytes) {
  if (!nblocks || !block_len || seg_bytes < 64 || seg_bytes > 65535) return 0;
  return deflate_plan(nblocks, block_len, seg_bytes).total;
}

extern "C" uint64_t nmk_deflate_bound(uint64_t nblocks, uint64_t block_len, uint32_t seg_bytes) {
  if (!nblocks || !block_len || seg_bytes < 64 || seg_bytes > 65535) return 0;
  return deflate_plan(nblocks, block_len, seg_bytes).nseg * (uint64_t)seg_bound(seg_bytes);
}

extern "C" int nmk_deflate(const uint8_t* packed, uint64_t block_stride, uint64_t nblocks, uint64_t block_len,
                           uint64_t last_len, uint32_t seg_bytes, uint8_t* out, unsigned long long* block_off,
                           void* ws, size_t ws_bytes, void* stream) {
  if (!packed || !out || !block_off || !ws || nblocks == 0 || block_len == 0 || last_len == 0 ||
      last_len > block_len || block_stride < block_len)
    return set_error(NMK_ERR_ARG, "nmk_deflate: bad argument");
  if (seg_bytes < 64 || seg_bytes > 65535 || seg_bytes % 16)
    return set_error(NMK_ERR_ARG, "nmk_deflate: seg_bytes must be a multiple of 16 in [64, 65535]");
  const DeflatePlan p = deflate_plan(nblocks, block_len, seg_bytes);
  if (ws_bytes < p.total) return set_error(NMK_ERR_ARG, "nmk_deflate: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  char* wb = (char*)ws;
  uint8_t* scratch = (uint8_t*)(wb + p.off_scratch);
  uint32_t* seg_len = (uint32_t*)(wb + p.off_len);
  unsigned long long* offsets = (unsigned long long*)(wb + p.off_offsets);
  const size_t smem = (size_t)kDefWarps * sizeof(DefWarp);
  ensure_dyn_smem(k_deflate_segments, smem);
  uint64_t g1 = (p.nseg + kDefWarps - 1) / kDefWarps;
  if (g1 > (uint64_t)sm_count() * 16) g1 = (uint64_t)sm_count() * 16;
  k_deflate_segments<<<(unsigned)g1, kDefThreads, smem, s>>>(packed, block_stride, nblocks, block_len, last_len,
                                                             seg_bytes, (uint32_t)p.segs_per_block, scratch,
                                                             seg_len);
  chunk_scan(seg_len, p.nseg, offsets, wb + p.off_scan, s);
  uint64_t g2 = (p.nseg + 7) / 8;
  if (g2 > 148 * 16) g2 = 148 * 16;
  k_deflate_gather<<<(unsigned)g2, 256, 0, s>>>(scratch, seg_len, offsets, p.nseg, seg_bytes,
                                                 (uint32_t)p.segs_per_block, out, block_off, nblocks);
  return check_launch("k_deflate");
}
