// k_deflate.cu — optional GPU replacement of the lossless index-table stage
// (codec.compress_block, pkg/src/nmk/codec.py:108-116).
//
// Each index block (pipeline.py:290-304: one raw RFC 1951 stream per block)
// is cut into segments of seg_bytes.  One thread compresses one segment:
// LZ77 over the segment (3-byte hash, 4-way buckets, run candidate, one-step
// lazy evaluation, window = the segment), a counting pass builds the
// segment's own length-limited Huffman codes, and the emitting pass writes a
// dynamic-Huffman block (BTYPE = 10) -- or the fixed code (BTYPE = 01) when
// that is not larger.  The segment's block is then closed with the end-of-block
// symbol followed by an empty stored block (BTYPE = 00, LEN = 0), which
// byte-aligns the bit stream -- so the segments of a block concatenate into
// one valid raw DEFLATE stream by a plain byte copy (the last segment's
// stored block carries BFINAL).  Any inflater (zlib included) reproduces the
// packed bytes exactly; the compressed bytes differ from zlib's, which the
// reference does not pin, so this stage is opt-in.
//
// Pipeline: k_deflate_segments (thread per segment, per-thread hash table in
// shared memory) -> chunk_scan over segment lengths -> k_deflate_gather
// (warp per segment, 16-byte copies into the compact output).
#include "nmk_common.cuh"
#include "nmk_scan.cuh"

namespace nmk {

constexpr int kDefThreads = 32;                  // 64 KB of hash tables per CTA (3 CTAs / SM)
constexpr int kDefHashBits = 8;                  // 256 buckets x 4 ways (u16 positions in a u64) per thread
constexpr int kDefHash = 1 << kDefHashBits;
constexpr uint64_t kEmptyBucket = ~0ULL;         // four 0xffff slots
constexpr int kMinMatch = 3, kMaxMatch = 258;

// worst case of one segment: the fixed code (chosen whenever the dynamic one
// is not smaller) spends <= 9 bits per byte, plus the block headers,
// end-of-block and the empty stored block, rounded up to 16 bytes
__host__ __device__ inline uint32_t seg_bound(uint32_t seg_bytes) { return ((seg_bytes * 9 + 7) / 8 + 32 + 15) & ~15u; }

struct BitWriter {
  uint32_t* out;      // word-aligned
  unsigned long long acc;
  int nbits;
  uint32_t nwords;
  __device__ __forceinline__ void put(uint32_t bits, int len) {   // LSB-first
    acc |= (unsigned long long)bits << nbits;
    nbits += len;
    if (nbits >= 32) {
      out[nwords++] = (uint32_t)acc;
      acc >>= 32;
      nbits -= 32;
    }
  }
  // pad to a byte boundary (zeros)
  __device__ __forceinline__ void align() { nbits = (nbits + 7) & ~7; }
  __device__ __forceinline__ uint32_t finish() {   // bytes written (byte-aligned stream)
    const uint32_t bytes = nwords * 4 + (uint32_t)(nbits >> 3);
    if (nbits) out[nwords] = (uint32_t)acc;   // the partial word (bytes past `bytes` are ignored)
    return bytes;
  }
};

__device__ __forceinline__ uint32_t rev_bits(uint32_t v, int len) { return __brev(v) >> (32 - len); }

// fixed literal/length code (RFC 1951 3.2.6), returned bit-reversed for LSB-first output
__device__ __forceinline__ void fixed_litlen(uint32_t sym, uint32_t& code, int& len) {
  if (sym < 144) { code = 0x30 + sym; len = 8; }
  else if (sym < 256) { code = 0x190 + (sym - 144); len = 9; }
  else if (sym < 280) { code = sym - 256; len = 7; }
  else { code = 0xC0 + (sym - 280); len = 8; }
  code = rev_bits(code, len);
}

__device__ __forceinline__ uint32_t hash3(uint32_t v) { return ((v & 0xffffffu) * 2654435761u) >> (32 - kDefHashBits); }

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

// Greedy LZ77 over one segment: distance-1 candidate (runs) and one hash
// candidate, 32-bit compare-extend; deterministic, so the counting pass and
// the emitting pass make identical decisions.
// LZ77 over one segment: candidates are the previous byte (runs) and the
// four most recent positions of the 3-byte hash bucket (a u64 holding four
// u16 positions, newest in the low bits); one-step lazy evaluation defers a
// short match when the next position matches longer.  Deterministic, so the
// counting pass and the emitting pass make identical decisions.
template <typename Lit, typename Match>
__device__ __forceinline__ void lz77(const uint8_t* __restrict__ src, uint32_t n, uint64_t* ht, Lit&& lit,
                                     Match&& match) {
  for (int i = 0; i < kDefHash; ++i) ht[i] = kEmptyBucket;
  auto word_at = [&](uint32_t i) -> uint32_t {   // bytes past n read as 0
    uint32_t v = 0;
    if (i + 4 <= n) {
      v = (uint32_t)src[i] | ((uint32_t)src[i + 1] << 8) | ((uint32_t)src[i + 2] << 16) | ((uint32_t)src[i + 3] << 24);
    } else {
      for (uint32_t k = 0; k < 4 && i + k < n; ++k) v |= (uint32_t)src[i + k] << (8 * k);
    }
    return v;
  };
  auto extend = [&](uint32_t j, uint32_t i) -> uint32_t {
    const uint32_t maxl = min((uint32_t)kMaxMatch, n - i);
    uint32_t l = 0;
    while (l + 4 <= maxl && word_at(j + l) == word_at(i + l)) l += 4;
    while (l < maxl && src[j + l] == src[i + l]) ++l;
    return l;
  };
  // longest match at i (0 if none); inserts i into its bucket
  auto find = [&](uint32_t i, uint32_t& dist) -> uint32_t {
    uint32_t best = 0;
    if (i + kMinMatch > n) return 0;
    const uint32_t h = hash3(word_at(i));
    const uint64_t bucket = ht[h];
    ht[h] = (bucket << 16) | i;
    if (i >= 1) {
      best = extend(i - 1, i);
      dist = 1;
    }
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const uint32_t j = (uint32_t)(bucket >> (16 * w)) & 0xffffu;
      if (j == 0xffffu || j + 1 >= i || i - j > 32768u) continue;   // j = i-1 already tried; RFC 1951 window
      const uint32_t l = extend(j, i);
      if (l > best) { best = l; dist = i - j; }
    }
    return best;
  };
  auto insert = [&](uint32_t p) {
    if (p + kMinMatch <= n) {
      const uint32_t h = hash3(word_at(p));
      ht[h] = (ht[h] << 16) | p;
    }
  };
  uint32_t i = 0;
  uint32_t dist = 0;
  uint32_t best = find(0, dist);
  while (i < n) {
    if (best >= kMinMatch) {
      if (best < 32 && i + 1 < n) {   // lazy: a longer match one byte later wins
        uint32_t d2 = 0;
        const uint32_t b2 = find(i + 1, d2);
        if (b2 > best) {
          lit(src[i]);
          ++i;
          best = b2;
          dist = d2;
          continue;
        }
        // i+1 is inserted already; emit the match at i
        match(best, dist);
        const uint32_t end = i + best;
        for (uint32_t p = i + 2; p < end && p < i + 8; ++p) insert(p);
        i = end;
      } else {
        match(best, dist);
        const uint32_t end = i + best;
        for (uint32_t p = i + 1; p < end && p < i + 8; ++p) insert(p);
        i = end;
      }
    } else {
      lit(src[i]);
      ++i;
    }
    if (i < n) best = find(i, dist);
  }
}

// Huffman code lengths <= maxlen for freq[0..nsym) (0 for unused symbols):
// two-queue construction over the sorted leaves, frequencies halved (>= 1)
// until the depth fits.  A lone used symbol gets a partner so every code is
// complete.  Work arrays are per thread (local memory).
constexpr int kHuffMax = 288;
__device__ void huff_lengths(const uint32_t* freq, int nsym, int maxlen, uint8_t* len) {
  uint32_t f[kHuffMax];
  uint16_t leaf[kHuffMax];
  uint32_t nf[2 * kHuffMax];
  uint16_t par[2 * kHuffMax];
  uint8_t dep[2 * kHuffMax];
  int m = 0;
  for (int s = 0; s < nsym; ++s) {
    len[s] = 0;
    if (freq[s]) { leaf[m] = (uint16_t)s; f[m] = freq[s]; ++m; }
  }
  if (m == 0) return;
  if (m == 1) {   // one symbol: length 1 plus an unused partner of length 1
    len[leaf[0]] = 1;
    len[leaf[0] == 0 ? 1 : 0] = 1;
    return;
  }
  for (;;) {
    // insertion sort of the leaves by (freq, symbol)
    for (int a = 1; a < m; ++a) {
      const uint32_t fa = f[a];
      const uint16_t la = leaf[a];
      int b = a - 1;
      while (b >= 0 && (f[b] > fa || (f[b] == fa && leaf[b] > la))) { f[b + 1] = f[b]; leaf[b + 1] = leaf[b]; --b; }
      f[b + 1] = fa;
      leaf[b + 1] = la;
    }
    for (int a = 0; a < m; ++a) nf[a] = f[a];
    int li = 0, ii = m, nn = m;
    auto take = [&]() -> int {
      if (li < m && (ii >= nn || nf[li] <= nf[ii])) return li++;
      return ii++;
    };
    while (nn < 2 * m - 1) {
      const int x = take(), y = take();
      nf[nn] = nf[x] + nf[y];
      par[x] = par[y] = (uint16_t)nn;
      ++nn;
    }
    dep[nn - 1] = 0;
    int maxd = 0;
    for (int k = nn - 2; k >= 0; --k) {
      dep[k] = dep[par[k]] + 1;
      if (k < m && dep[k] > maxd) maxd = dep[k];
    }
    if (maxd <= maxlen) {
      for (int a = 0; a < m; ++a) len[leaf[a]] = dep[a];
      return;
    }
    for (int a = 0; a < m; ++a) f[a] = max(1u, f[a] >> 1);
  }
}

// canonical codes (RFC 1951 3.2.2), bit-reversed for LSB-first output
__device__ void huff_codes(const uint8_t* len, int nsym, uint16_t* code) {
  uint32_t cnt[16] = {0}, next[16];
  for (int s = 0; s < nsym; ++s) ++cnt[len[s]];
  cnt[0] = 0;
  uint32_t c = 0;
  for (int b = 1; b < 16; ++b) {
    c = (c + cnt[b - 1]) << 1;
    next[b] = c;
  }
  for (int s = 0; s < nsym; ++s)
    code[s] = len[s] ? (uint16_t)rev_bits(next[len[s]]++, len[s]) : 0;
}

__constant__ uint8_t kClOrder[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};

__global__ void __launch_bounds__(kDefThreads)
k_deflate_segments(const uint8_t* __restrict__ packed, uint64_t stride, uint64_t nblocks, uint64_t block_len,
                   uint64_t last_len, uint32_t seg_bytes, uint32_t segs_per_block, uint8_t* __restrict__ scratch,
                   uint32_t* __restrict__ seg_len) {
  extern __shared__ uint64_t s_hash[];   // kDefThreads x kDefHash buckets
  const uint64_t nseg = nblocks * segs_per_block;
  uint64_t* ht = s_hash + (size_t)threadIdx.x * kDefHash;
  for (uint64_t sg = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; sg < nseg;
       sg += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = sg / segs_per_block;
    const uint32_t s = (uint32_t)(sg - b * segs_per_block);
    const uint64_t blen = (b + 1 == nblocks) ? last_len : block_len;
    const uint64_t lo = (uint64_t)s * seg_bytes;
    uint8_t* dst = scratch + sg * (uint64_t)seg_bound(seg_bytes);
    if (lo >= blen) {   // segment past a short last block: nothing
      seg_len[sg] = 0;
      continue;
    }
    const uint32_t n = (uint32_t)min((uint64_t)seg_bytes, blen - lo);
    const bool last = lo + n == blen;
    const uint8_t* src = packed + b * stride + lo;

    // ---- pass 1: symbol statistics ----
    uint32_t lf[286], df[30];
    for (int k = 0; k < 286; ++k) lf[k] = 0;
    for (int k = 0; k < 30; ++k) df[k] = 0;
    uint64_t extra = 0;
    lz77(src, n, ht, [&](uint32_t byte) { ++lf[byte]; },
         [&](uint32_t len, uint32_t dist) {
           uint32_t sy, eb, ev;
           len_symbol(len, sy, eb, ev);
           ++lf[sy];
           extra += eb;
           dist_symbol(dist, sy, eb, ev);
           ++df[sy];
           extra += eb;
         });
    lf[256] = 1;   // end of block

    // ---- dynamic code: lengths, run-length coded lengths, their code ----
    uint8_t ll[286], dl[30];
    huff_lengths(lf, 286, 15, ll);
    huff_lengths(df, 30, 15, dl);
    int hlit = 286, hdist = 30;
    while (hlit > 257 && ll[hlit - 1] == 0) --hlit;
    while (hdist > 1 && dl[hdist - 1] == 0) --hdist;
    uint8_t rs[316], rx[316];   // RLE symbols and their extra values
    int nr = 0;
    {
      auto L = [&](int i) -> uint32_t { return i < hlit ? ll[i] : dl[i - hlit]; };
      const int tot = hlit + hdist;
      int i = 0;
      while (i < tot) {
        const uint32_t v = L(i);
        int run = 1;
        while (i + run < tot && L(i + run) == v) ++run;
        if (v == 0) {
          int r = run;
          while (r >= 11) { const int t = min(r, 138); rs[nr] = 18; rx[nr++] = (uint8_t)(t - 11); r -= t; }
          if (r >= 3) { rs[nr] = 17; rx[nr++] = (uint8_t)(r - 3); r = 0; }
          while (r > 0) { rs[nr] = 0; rx[nr++] = 0; --r; }
        } else {
          rs[nr] = (uint8_t)v; rx[nr++] = 0;
          int r = run - 1;
          while (r >= 3) { const int t = min(r, 6); rs[nr] = 16; rx[nr++] = (uint8_t)(t - 3); r -= t; }
          while (r > 0) { rs[nr] = (uint8_t)v; rx[nr++] = 0; --r; }
        }
        i += run;
      }
    }
    uint32_t cf[19];
    for (int k = 0; k < 19; ++k) cf[k] = 0;
    for (int k = 0; k < nr; ++k) ++cf[rs[k]];
    uint8_t cl[19];
    huff_lengths(cf, 19, 7, cl);
    int hclen = 19;
    while (hclen > 4 && cl[kClOrder[hclen - 1]] == 0) --hclen;
    // cost of the two encodings (extra bits are the same for both)
    uint64_t dyn = 14 + 3 * (uint64_t)hclen, fix = 0;
    for (int k = 0; k < nr; ++k) dyn += cl[rs[k]] + (rs[k] == 16 ? 2 : rs[k] == 17 ? 3 : rs[k] == 18 ? 7 : 0);
    for (int k = 0; k < 286; ++k) {
      if (!lf[k]) continue;
      dyn += (uint64_t)lf[k] * ll[k];
      fix += (uint64_t)lf[k] * (k < 144 ? 8 : k < 256 ? 9 : k < 280 ? 7 : 8);
    }
    for (int k = 0; k < 30; ++k) { dyn += (uint64_t)df[k] * dl[k]; fix += (uint64_t)df[k] * 5; }
    const bool use_dyn = dyn < fix;
    (void)extra;

    // ---- pass 2: emit ----
    BitWriter w{reinterpret_cast<uint32_t*>(dst), 0ULL, 0, 0};
    uint16_t lc[286], dc[30];
    if (use_dyn) {
      uint16_t cc[19];
      huff_codes(ll, 286, lc);
      huff_codes(dl, 30, dc);
      huff_codes(cl, 19, cc);
      w.put(0u | (2u << 1), 3);   // BFINAL = 0, BTYPE = 10 (dynamic Huffman)
      w.put((uint32_t)(hlit - 257), 5);
      w.put((uint32_t)(hdist - 1), 5);
      w.put((uint32_t)(hclen - 4), 4);
      for (int k = 0; k < hclen; ++k) w.put(cl[kClOrder[k]], 3);
      for (int k = 0; k < nr; ++k) {
        w.put(cc[rs[k]], cl[rs[k]]);
        if (rs[k] == 16) w.put(rx[k], 2);
        else if (rs[k] == 17) w.put(rx[k], 3);
        else if (rs[k] == 18) w.put(rx[k], 7);
      }
    } else {
      for (int k = 0; k < 286; ++k) {
        uint32_t c;
        int l;
        fixed_litlen((uint32_t)k, c, l);
        lc[k] = (uint16_t)c;
        ll[k] = (uint8_t)l;
      }
      for (int k = 0; k < 30; ++k) { dc[k] = (uint16_t)rev_bits((uint32_t)k, 5); dl[k] = 5; }
      w.put(0u | (1u << 1), 3);   // BFINAL = 0, BTYPE = 01 (fixed Huffman)
    }
    lz77(src, n, ht, [&](uint32_t byte) { w.put(lc[byte], ll[byte]); },
         [&](uint32_t len, uint32_t dist) {
           uint32_t sy, eb, ev;
           len_symbol(len, sy, eb, ev);
           w.put(lc[sy], ll[sy]);
           if (eb) w.put(ev, (int)eb);
           dist_symbol(dist, sy, eb, ev);
           w.put(dc[sy], dl[sy]);
           if (eb) w.put(ev, (int)eb);
         });
    w.put(lc[256], ll[256]);    // end of block
    // an empty stored block byte-aligns the stream (BFINAL on the last segment)
    w.put(last ? 1u : 0u, 3);
    w.align();
    w.put(0x0000u, 16);         // LEN
    w.put(0xffffu, 16);         // NLEN
    seg_len[sg] = w.finish();
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
  const size_t smem = (size_t)kDefThreads * kDefHash * sizeof(uint64_t);
  ensure_dyn_smem(k_deflate_segments, smem);
  const uint64_t g1 = (p.nseg + kDefThreads - 1) / kDefThreads;
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
