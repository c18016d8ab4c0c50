// k_inflate.cu — GPU inflate of raw DEFLATE streams (RFC 1951): the decode
// half of the lossless index-table stage (codec.decompress_block,
// pkg/src/nmk/codec.py:119-128).
//
// Every 1 MiB index block of a variable is one raw DEFLATE stream, written
// either by the host's zlib (the reference's bytes) or by k_deflate.cu, so
// the blocks inflate independently: one warp per stream, into the strided
// packed-block layout K5 reads, so a decode never ships inflated bytes over
// PCIe.  Inside a stream DEFLATE is sequential; all 32 lanes run the same
// bit-reader and Huffman decode (their state is identical, loads broadcast)
// and split the bytes of every match (and stored block) between them --
// out[pos + j] = out[pos - dist + (j mod dist)] holds for overlapping
// matches too, since the source bytes precede pos.
//
// Huffman decode: a 2^10-entry table per code (canonical codes, bit-reversed
// as they arrive LSB first) resolves every code of <= 10 bits in one lookup;
// longer codes take the canonical count walk (zlib's puff).  Validation
// follows zlib's inflate: over-subscribed codes, incomplete literal/length
// or distance codes (unless a single one-bit code), incomplete code-length
// codes, HLIT > 286, HDIST > 30, a missing end-of-block code, literal/length
// symbols 286/287, distance symbols 30/31, distances before the start of
// the stream, stored-block LEN/NLEN mismatch, input that ends before the
// final block and bytes after it (codec.py:125-127) are errors.
#include "nmk_common.cuh"

namespace nmk {

#ifndef NMK_INF_POS32
#define NMK_INF_POS32 1   // output positions in 32 bits (out_stride < 4 GiB - 64 KiB, checked by nmk_inflate): A/B on
                          // cfg2's 128 blocks 40.5 -> 39.4 ms (zlib streams), 48.4 -> 46.9 ms (GPU deflate's)
#endif
#ifndef NMK_INF_LITRUN
#define NMK_INF_LITRUN 0   // A/B: a check-free four-lookup literal run helps literal-heavy streams (the GPU deflate's:
                           // 48.4 -> 46.6 ms) but its repeated lookup at every match costs zlib's 40.5 -> 53.6 ms
#endif
constexpr int kInfWarps = 1;          // streams per CTA (one per SM for a block's worth of streams)
constexpr uint32_t kWin = 32768;      // DEFLATE's window: the last 32 KB of output, in shared memory
constexpr uint32_t kFlush = 1024;     // window -> global store granularity
constexpr int kLutBits = 12;   // 8 KB tables: zlib's distance codes mostly fit
constexpr int kLut = 1 << kLutBits;

enum InflateStatus : unsigned {
  kInfOk = 0,
  kInfBadBlockType = 1,
  kInfBadStored = 2,
  kInfBadHeader = 3,      // HLIT/HDIST out of range, bad repeat, no end-of-block code
  kInfBadCode = 4,        // over-subscribed / incomplete code, undecodable symbol
  kInfBadDistance = 5,    // distance symbol >= 30 or too far back
  kInfTruncated = 6,      // the input ended before the final block
  kInfTrailing = 7,       // bytes after the final block
  kInfOverflow = 8,       // the stream inflates past its output capacity
};

struct Huff {
  uint16_t lut[kLut];   // (len << 9) | sym for codes of <= kLutBits bits, 0 = slow path
  uint16_t count[16];
  uint16_t sym[288];
};

// Multi-literal table over the next kMBits bits: up to 4 literals whose
// codes fit (lo = the bytes, hi = n | bits << 4), or one length / end-of-
// block symbol (n = 0, lo = sym, bits = its length), or hi = 0: the slow path.
constexpr int kMBits = 12;
constexpr int kMLut = 1 << kMBits;

struct InfState {
  uint2 mlut[kMLut];
  Huff lit, dist;
  uint8_t lens[320];
  uint16_t offs[16];
  int status;
};

// bit reader (identical in every lane)
#ifndef NMK_INF_LOOKAHEAD
#define NMK_INF_LOOKAHEAD 0   // A/B: input words held two ahead in registers (a refill never waits for its own
                              // load) changes nothing: 40.5 -> 41.7 ms on cfg2's zlib streams -- the refill's loads
                              // hit L1; the decode is bound by its dependent ALU / shared-memory chain
#endif
struct Bits {
  const uint8_t* p;
  uint64_t len, pos;      // input bytes, next byte to load
  uint64_t buf;
  int cnt;
#if NMK_INF_LOOKAHEAD
  // the aligned 8-byte input words at wp, wp + 1, wp + 2 (wp: the word holding
  // byte `pos` at the last refill); loads never pass wlast (the buffer's pad)
  const uint64_t* wp;
  const uint64_t* wlast;
  uint64_t w0, w1, w2;
  __device__ __forceinline__ uint64_t ldw(const uint64_t* w) const { return __ldg(w < wlast ? w : wlast); }
  __device__ __forceinline__ void seek() {   // (re)load the window at pos
    wp = reinterpret_cast<const uint64_t*>((reinterpret_cast<uintptr_t>(p) + pos) & ~(uintptr_t)7);
    w0 = ldw(wp);
    w1 = ldw(wp + 1);
    w2 = ldw(wp + 2);
  }
#endif
  // to >= 57 bits: the next 8 input bytes from two aligned 8-byte words (the
  // input buffer is padded by 16 bytes on both sides), bytes at or past the
  // stream's end read as zero
  __device__ __forceinline__ void refill() {
    const int nb = (63 - cnt) >> 3;
    const uintptr_t a = reinterpret_cast<uintptr_t>(p) + pos;
    const uint64_t* w = reinterpret_cast<const uint64_t*>(a & ~(uintptr_t)7);
    const int sh = (int)(a & 7) * 8;
#if NMK_INF_LOOKAHEAD
    if (w != wp) {   // pos advances <= 8 bytes per refill: at most one word further
      w0 = w1;
      w1 = w2;
      wp = w;
      w2 = ldw(w + 2);   // needed two words (>= 8 bytes of input) from now
    }
    const uint64_t lo = w0, hi = w1;
#else
    const uint64_t lo = __ldg(w), hi = __ldg(w + 1);
#endif
    uint64_t v = sh ? (lo >> sh) | (hi << (64 - sh)) : lo;
    const uint64_t left = pos < len ? len - pos : 0;
    const int keep = (int)(left < (uint64_t)nb ? left : (uint64_t)nb);   // bytes of real input
    v = keep >= 8 ? v : (v & ((1ULL << (8 * keep)) - 1ULL));
    if (nb < 8) v &= (1ULL << (8 * nb)) - 1ULL;
    buf |= v << cnt;
    pos += nb;
    cnt += 8 * nb;
  }
  __device__ __forceinline__ uint32_t get(int n) {   // n <= 32
    if (cnt < n) refill();
    const uint32_t v = (uint32_t)(buf & ((1ULL << n) - 1ULL));
    buf >>= n;
    cnt -= n;
    return v;
  }
  // bits consumed so far > input size: the stream ran past its end
  __device__ __forceinline__ bool overrun() const { return pos * 8 - (uint64_t)cnt > len * 8; }
};

__device__ __forceinline__ uint32_t bitrev(uint32_t c, int n) { return __brev(c) >> (32 - n); }

// Build a canonical Huffman decoder from n code lengths in st.lens[first..].
// kind: 0 = code-length code (must be complete), 1 = literal/length or
// distance (complete, or a single one-bit code).  Returns false on a bad set.
__device__ bool huff_build(Huff& h, const uint8_t* lens, int n, int kind, InfState& st) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < kLut; i += 32) h.lut[i] = 0;
  __shared__ int s_ok[kInfWarps];
  const int w = threadIdx.x >> 5;
  if (lane == 0) {
    for (int l = 0; l < 16; ++l) h.count[l] = 0;
    for (int s = 0; s < n; ++s) h.count[lens[s]]++;
    int left = 1, maxl = 0;
    bool ok = true;
    for (int l = 1; l < 16; ++l) {
      left <<= 1;
      left -= h.count[l];
      if (left < 0) ok = false;   // over-subscribed
      if (h.count[l]) maxl = l;
    }
    if (ok && left > 0 && (kind == 0 || maxl != 1)) ok = false;   // incomplete (zlib inflate_table)
    if (h.count[0] == n) ok = kind != 0;                          // no codes: only allowed for distances
    st.offs[1] = 0;
    for (int l = 1; l < 15; ++l) st.offs[l + 1] = st.offs[l] + h.count[l];
    for (int s = 0; s < n; ++s)
      if (lens[s]) h.sym[st.offs[lens[s]]++] = (uint16_t)s;
    s_ok[w] = ok;
  }
  __syncwarp();
  // LUT: symbols in canonical order; code of the i-th symbol of length l is
  // first[l] + (i - index[l]).  Each lane fills the entries of a share of them.
  if (s_ok[w]) {
    int code = 0, index = 0;
    for (int l = 1; l <= kLutBits; ++l) {
      const int c = h.count[l];
      for (int i = lane; i < c; i += 32) {
        const uint32_t r = bitrev((uint32_t)(code + i), l);
        const uint16_t e = (uint16_t)((l << 9) | h.sym[index + i]);
        for (uint32_t j = r; j < (uint32_t)kLut; j += 1u << l) h.lut[j] = e;
      }
      code = (code + c) << 1;
      index += c;
    }
  }
  __syncwarp();
  return s_ok[w] != 0;
}

// mlut from the literal/length code's single-symbol table (all lanes)
__device__ void mlut_build(InfState& st) {
  const int lane = threadIdx.x & 31;
  for (int idx = lane; idx < kMLut; idx += 32) {
    uint32_t lo = 0, n = 0, used = 0, hi = 0;
    while (n < 4) {
      const uint16_t e = st.lit.lut[(idx >> used) & (kLut - 1)];
      const uint32_t l = e >> 9;
      if (!e || used + l > (uint32_t)kMBits) break;
      const uint32_t sym = e & 511;
      if (sym >= 256) {
        if (n == 0) hi = (l << 4), lo = sym;   // a lone length / end-of-block symbol
        break;
      }
      lo |= sym << (8 * n);
      ++n;
      used += l;
    }
    if (n) hi = n | (used << 4);
    st.mlut[idx] = make_uint2(lo, hi);
  }
  __syncwarp();
}

// one symbol; -1 when no code matches
__device__ __forceinline__ int huff_decode(const Huff& h, Bits& br) {
  if (br.cnt < 15) br.refill();
  const uint16_t e = h.lut[br.buf & (kLut - 1)];
  if (e) {
    const int l = e >> 9;
    br.buf >>= l;
    br.cnt -= l;
    return e & 511;
  }
  // canonical walk, one bit at a time (codes longer than kLutBits)
  int code = 0, first = 0, index = 0;
  for (int l = 1; l < 16; ++l) {
    code |= (int)(br.buf & 1ULL);
    br.buf >>= 1;
    br.cnt -= 1;
    const int c = h.count[l];
    if (code - c < first) return h.sym[index + (code - first)];
    index += c;
    first = (first + c) << 1;
    code <<= 1;
  }
  return -1;
}

__constant__ uint16_t c_lbase[29] = {3, 4, 5, 6, 7, 8, 9, 10, 11, 13, 15, 17, 19, 23, 27, 31,
                                     35, 43, 51, 59, 67, 83, 99, 115, 131, 163, 195, 227, 258};
__constant__ uint8_t c_lext[29] = {0, 0, 0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 3, 4, 4, 4, 4, 5, 5, 5, 5, 0};
__constant__ uint16_t c_dbase[30] = {1, 2, 3, 4, 5, 7, 9, 13, 17, 25, 33, 49, 65, 97, 129, 193,
                                     257, 385, 513, 769, 1025, 1537, 2049, 3073, 4097, 6145, 8193, 12289, 16385, 24577};
__constant__ uint8_t c_dext[30] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};
// c_mod[d][0] = 32 mod d, c_mod[d][1 + l] = l mod d (d < 32): the match copy's
// per-lane source offsets without integer division
struct ModTable {
  uint8_t v[32][33];
  constexpr ModTable() : v() {
    for (int d = 1; d < 32; ++d) {
      v[d][0] = (uint8_t)(32 % d);
      for (int l = 0; l < 32; ++l) v[d][1 + l] = (uint8_t)(l % d);
    }
  }
};
__constant__ ModTable c_modt = ModTable();
#define c_mod c_modt.v
__constant__ uint8_t c_clorder[19] = {16, 17, 18, 0, 8, 7, 9, 6, 10, 5, 11, 4, 12, 3, 13, 2, 14, 1, 15};

__global__ void __launch_bounds__(32 * kInfWarps)
k_inflate(const uint8_t* __restrict__ comp, const unsigned long long* __restrict__ comp_off, uint64_t nstreams,
          uint8_t* __restrict__ out, uint64_t out_stride, const unsigned long long* __restrict__ out_off,
          unsigned* __restrict__ status, unsigned long long* __restrict__ produced) {
  extern __shared__ __align__(16) uint8_t inf_smem[];   // InfState[kInfWarps], then the windows
  InfState* sst = reinterpret_cast<InfState*>(inf_smem);
  uint8_t* swin = inf_smem + sizeof(InfState) * kInfWarps;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t s = (uint64_t)blockIdx.x * kInfWarps + w;
  if (s >= nstreams) return;
  InfState& st = sst[w];
  Bits br;
  br.p = comp + comp_off[s];
  br.len = comp_off[s + 1] - comp_off[s];
  br.pos = 0;
  br.buf = 0;
  br.cnt = 0;
#if NMK_INF_LOOKAHEAD
  // the last whole 8-byte word inside the input's 16-byte tail pad
  br.wlast = reinterpret_cast<const uint64_t*>(
      (reinterpret_cast<uintptr_t>(comp) + comp_off[nstreams] + 8) & ~(uintptr_t)7);
  br.seek();
#endif
  uint8_t* dst = out + (out_off ? out_off[s] : s * out_stride);
  uint8_t* win = swin + (size_t)w * kWin;
  // output leaves through the window: every kFlush bytes the warp stores the
  // finished 128-byte pieces with coalesced 4-byte stores (dst and flushed
  // stay 16-byte aligned)
#if NMK_INF_POS32
  typedef uint32_t pos_t;
#else
  typedef uint64_t pos_t;
#endif
  pos_t flushed = 0;
  auto flush = [&](pos_t upto) {
    __syncwarp();
    for (; flushed + 128 <= upto; flushed += 128) {
      const uint32_t o = (uint32_t)(flushed + 4 * lane) & (kWin - 1);
      *reinterpret_cast<uint32_t*>(dst + flushed + 4 * lane) = *reinterpret_cast<const uint32_t*>(win + o);
    }
  };
  const pos_t cap = (pos_t)out_stride;
  pos_t pos = 0;
  unsigned err = kInfOk;
  bool final_seen = false;
  while (!err && !final_seen) {
    final_seen = br.get(1);
    const uint32_t type = br.get(2);
    if (type == 0) {   // stored: align to a byte, LEN, NLEN, raw bytes
      const int drop = br.cnt & 7;
      br.buf >>= drop;
      br.cnt -= drop;
      const uint32_t ln = br.get(16), nln = br.get(16);
      if (ln != (~nln & 0xffffu)) { err = kInfBadStored; break; }
      // the buffered whole bytes come first, then the input
      const uint64_t in0 = br.pos - (uint64_t)(br.cnt >> 3);
      if (in0 + ln > br.len) { err = kInfTruncated; break; }
      if (pos + ln > cap) { err = kInfOverflow; break; }
      for (uint32_t j = 0; j < ln; j += 32) {   // through the window in 32-byte pieces
        if (j + lane < ln) win[(uint32_t)(pos + j + lane) & (kWin - 1)] = __ldg(br.p + in0 + j + lane);
        __syncwarp();
        if (pos + j + 32 - flushed >= kFlush) flush(pos + min(j + 32, ln));
      }
      pos += ln;
      br.pos = in0 + ln;
      br.buf = 0;
      br.cnt = 0;
#if NMK_INF_LOOKAHEAD
      br.seek();
#endif
      __syncwarp();
      continue;
    }
    if (type == 3) { err = kInfBadBlockType; break; }
    if (type == 1) {   // fixed codes
      for (int i = lane; i < 288; i += 32) st.lens[i] = i < 144 ? 8 : i < 256 ? 9 : i < 280 ? 7 : 8;
      for (int i = lane; i < 30; i += 32) st.lens[288 + i] = 5;
      __syncwarp();
      huff_build(st.lit, st.lens, 288, 1, st);
      huff_build(st.dist, st.lens + 288, 30, 1, st);
      mlut_build(st);
    } else {           // dynamic
      const int hlit = (int)br.get(5) + 257, hdist = (int)br.get(5) + 1, hclen = (int)br.get(4) + 4;
      if (hlit > 286 || hdist > 30) { err = kInfBadHeader; break; }
      uint8_t cl[19];
      for (int i = 0; i < 19; ++i) cl[i] = 0;
      for (int i = 0; i < hclen; ++i) cl[c_clorder[i]] = (uint8_t)br.get(3);
      for (int i = lane; i < 19; i += 32) st.lens[i] = cl[i];
      __syncwarp();
      if (!huff_build(st.dist, st.lens, 19, 0, st)) { err = kInfBadCode; break; }   // dist table as scratch
      uint8_t l8[320];
      int i = 0;
      while (i < hlit + hdist && !err) {
        const int sym = huff_decode(st.dist, br);
        if (sym < 0) { err = kInfBadCode; break; }
        if (sym < 16) { l8[i++] = (uint8_t)sym; continue; }
        int rep, val = 0;
        if (sym == 16) {
          if (i == 0) { err = kInfBadHeader; break; }
          val = l8[i - 1];
          rep = 3 + (int)br.get(2);
        } else if (sym == 17) {
          rep = 3 + (int)br.get(3);
        } else {
          rep = 11 + (int)br.get(7);
        }
        if (i + rep > hlit + hdist) { err = kInfBadHeader; break; }
        while (rep--) l8[i++] = (uint8_t)val;
      }
      if (err) break;
      if (l8[256] == 0) { err = kInfBadHeader; break; }
      for (int j = lane; j < hlit + hdist; j += 32) st.lens[j] = l8[j];
      __syncwarp();
      if (!huff_build(st.lit, st.lens, hlit, 1, st)) { err = kInfBadCode; break; }
      mlut_build(st);
      __syncwarp();
      if (!huff_build(st.dist, st.lens + hlit, hdist, 1, st)) { err = kInfBadCode; break; }
    }
    // symbols: up to four literals per table lookup
    while (true) {
#if NMK_INF_LITRUN
      // literal run: four table lookups per refill (4 x kMBits <= the 57 bits a
      // refill guarantees) with no per-lookup capacity / refill / flush checks;
      // the first entry that is not a literal group leaves it to the general step
      if (pos + 16 <= cap) {
        if (br.cnt < 4 * kMBits) br.refill();
        bool run = true;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint2 e = st.mlut[br.buf & (kMLut - 1)];
          const uint32_t nl = e.y & 15u;
          if (!nl) { run = false; break; }
          const uint32_t used = e.y >> 4;
          br.buf >>= used;
          br.cnt -= (int)used;
          if ((uint32_t)lane < nl) win[(uint32_t)(pos + lane) & (kWin - 1)] = (uint8_t)(e.x >> (8 * lane));
          pos += nl;
        }
        if (pos - flushed >= kFlush) flush(pos);
        if (run) continue;
      }
#endif
      if (br.cnt < kMBits) br.refill();
      const uint2 me = st.mlut[br.buf & (kMLut - 1)];
      int sym;
      const uint32_t nlit = me.y & 15u;
      if (nlit) {
        if (pos + nlit > cap) { err = kInfOverflow; break; }
        const uint32_t used = me.y >> 4;
        br.buf >>= used;
        br.cnt -= (int)used;
        if ((uint32_t)lane < nlit) win[(uint32_t)(pos + lane) & (kWin - 1)] = (uint8_t)(me.x >> (8 * lane));
        pos += nlit;
        if (pos - flushed >= kFlush) flush(pos);
        continue;
      }
      if (me.y) {   // a lone length / end-of-block symbol
        const uint32_t used = me.y >> 4;
        br.buf >>= used;
        br.cnt -= (int)used;
        sym = (int)me.x;
      } else {
        sym = huff_decode(st.lit, br);
      }
      if (sym < 0 || sym > 285) { err = kInfBadCode; break; }
      if (sym < 256) {
        if (pos >= cap) { err = kInfOverflow; break; }
        if (lane == 0) win[pos & (kWin - 1)] = (uint8_t)sym;
        ++pos;
        if (pos - flushed >= kFlush) flush(pos);
        continue;
      }
      if (sym == 256) break;
      const int li = sym - 257;
      const uint32_t len = c_lbase[li] + br.get(c_lext[li]);
      const int ds = huff_decode(st.dist, br);
      if (ds < 0 || ds > 29) { err = kInfBadDistance; break; }
      const uint32_t dist = c_dbase[ds] + br.get(c_dext[ds]);
      if (dist > pos) { err = kInfBadDistance; break; }
      if (pos + len > cap) { err = kInfOverflow; break; }
      __syncwarp();   // earlier bytes (other lanes' window stores) are visible
      // lane j copies bytes j, j + 32, ...: source offset t = j mod dist,
      // advanced by 32 mod dist per round (sources all precede pos)
      if ((uint32_t)lane < len) {
        const uint32_t step = dist < 32 ? c_mod[dist][0] : 32u;   // 32 mod dist
        uint32_t t = dist < 32 ? c_mod[dist][lane + 1] : (uint32_t)lane;   // lane mod dist
        const uint32_t src = (uint32_t)(pos - dist);
        for (uint32_t j = lane; j < len; j += 32) {
          win[(uint32_t)(pos + j) & (kWin - 1)] = win[(src + t) & (kWin - 1)];
          t += step;
          if (t >= dist) t -= dist;
        }
      }
      __syncwarp();
      pos += len;
      if (pos - flushed >= kFlush) flush(pos);
    }
    if (!err && br.overrun()) err = kInfTruncated;
  }
  if (!err) {   // the unflushed tail (< 128 bytes)
    __syncwarp();
    for (pos_t j = flushed + lane; j < pos; j += 32) dst[j] = win[(uint32_t)j & (kWin - 1)];
  }
  if (!err) {
    // bytes consumed = ceil(bits / 8); anything after them is trailing data
    const uint64_t used = (br.pos * 8 - (uint64_t)br.cnt + 7) / 8;
    if (br.overrun()) err = kInfTruncated;
    else if (used < br.len) err = kInfTrailing;
  }
  if (lane == 0) {
    status[s] = err;
    produced[s] = pos;
  }
}

}  // namespace nmk

using namespace nmk;

extern "C" int nmk_inflate(const uint8_t* comp, const unsigned long long* comp_off, uint64_t nstreams, uint8_t* out,
                           uint64_t out_stride, const unsigned long long* out_off, unsigned* status,
                           unsigned long long* produced, void* stream) {
  if (nstreams == 0) return NMK_OK;
  if (!comp || !comp_off || !out || !status || !produced || out_stride == 0)
    return set_error(NMK_ERR_ARG, "nmk_inflate: bad argument");
  if (out_stride >= (1ULL << 32) - 65536) return set_error(NMK_ERR_ARG, "nmk_inflate: out_stride must be below 4 GiB");
  const uint64_t grid = (nstreams + kInfWarps - 1) / kInfWarps;
  constexpr size_t smem = (sizeof(InfState) + kWin) * kInfWarps;
  ensure_dyn_smem(k_inflate, smem);
  k_inflate<<<(unsigned)grid, 32 * kInfWarps, smem, (cudaStream_t)stream>>>(comp, comp_off, nstreams, out, out_stride,
                                                                         out_off, status, produced);
  return check_launch("k_inflate");
}
