/*
 * nmk_b200.h — C ABI of the B200 (sm_100a) NUMARCK hot path.
 *
 * The reference (arXiv 1703.02438 re-implementation, package `nmk`) is pure
 * Python; its hot path is the body of `pipeline.compress_pair` phases 1-4a
 * (pkg/src/nmk/pipeline.py:185-288) and the decode chain
 * `pipeline.decompress` -> `codec._decode_range` -> `codec.unpack_block` +
 * `core.reconstruct` (pipeline.py:327-340, codec.py:95-105,204-239,
 * core.py:158-208).  This library replaces exactly those phases.  The Python
 * mirror `paper_1703_02438_b200` binds these symbols through ctypes and keeps
 * the reference's public API (compress_pair / decompress / compress_series /
 * partial_decode) on top; see INTEGRATION.md for the binding.
 *
 * Conventions
 *  - All buffers are caller-owned DEVICE pointers unless named h_*; the
 *    stream is the last argument; every call is stream-ordered and returns
 *    0 (NMK_OK) or a negative NMK_ERR_* code with a thread-local message in
 *    nmk_last_error().  No call synchronises the stream.
 *  - dtype: NMK_F32 / NMK_F64, matching the container's dtype codes
 *    (container.py:28-31).
 *  - Element indices are 64-bit (n up to 4e9 per call).
 *  - Arithmetic is IEEE binary64 without contraction (built -fmad=false),
 *    bit-identical to the reference's numpy expressions.
 */
#ifndef NMK_B200_H
#define NMK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NMK_OK               0
#define NMK_ERR_ARG         -1   /* bad argument (ValueError in Python)            */
#define NMK_ERR_CUDA        -2   /* CUDA runtime / launch failure                   */
#define NMK_ERR_EMPTY_HIST  -6   /* no selectable bin: binning.py:145-146          */
#define NMK_ERR_NEEDS_SPARSE -7  /* sync-free path: span too wide for the dense
                                    histogram; rerun the sparse path             */

/* nmk_stats.reserved after nmk_hist_prep: the dense span, 0 when no ratio is
 * valid, NMK_SPAN_SPARSE when it exceeds the dense capacity. */
#define NMK_SPAN_SPARSE 0xffffffffffffffffULL

#define NMK_F32 0
#define NMK_F64 1

/* Device scalars produced by nmk_minmax (phase 1, pipeline.py:190-212).
 * For a multi-GPU run the caller all-reduces gmin (MIN), gmax (MAX) and
 * nvalid (SUM) before the histogram. */
typedef struct nmk_stats {
    double gmin;
    double gmax;
    unsigned long long nvalid;
    unsigned long long reserved;
} nmk_stats;

/* Device model header produced by nmk_select (phase 2 decisions,
 * pipeline.py:127-140,229; binning.py:142-206). */
typedef struct nmk_model {
    int32_t bits;          /* index length B                                    */
    int32_t k;             /* number of (quantised) centers                     */
    int32_t status;        /* 0 ok, NMK_ERR_EMPTY_HIST                          */
    int32_t m_selectable;  /* nonempty bins with a finite center                */
    double  tol_bin;       /* BinModel.tolerance: (2E)/2, or E when degenerate  */
    unsigned long long coverage[17]; /* auto-B: covered elements for B=2..16;
                                        [0], [1] = the two largest selectable
                                        bin counts                              */
} nmk_model;

/* Decode error word (device), checked by the caller after nmk_decode. */
typedef struct nmk_decode_err {
    unsigned int bad_index;        /* 1 if any code in [k, sentinel)            */
    unsigned int max_bad_index;    /* largest such code                         */
    unsigned int exhausted;        /* 1 if an exact value past the end was read */
    unsigned int reserved;
} nmk_decode_err;

/* Per-segment decode bookkeeping (device, written by nmk_decode). */
typedef struct nmk_segment_info {
    unsigned long long inc_before;   /* exact values before segment start,
                                        relative to the exact pointer passed   */
    unsigned long long n_sentinel;   /* sentinels inside the segment            */
} nmk_segment_info;

const char* nmk_last_error(void);
int nmk_version(void);

/* -- A1 standalone: ratio + validity (core.py:115-137) -------------------- */
int nmk_ratio(const void* base, const void* cur, uint64_t n, int dtype,
              double* ratios, uint8_t* valid, void* stream);

/* -- K1: fused ratio + min/max + valid count (pipeline.py:190-212) --------
 * keys (optional, 16-byte aligned float[n]): per-element f32 ratio key for
 * the histogram pass (NaN: invalid element, +inf: decide exactly). */
size_t nmk_minmax_ws_bytes(uint64_t n);
int nmk_minmax(const void* base, const void* cur, uint64_t n, int dtype,
               nmk_stats* stats, float* keys, void* ws, size_t ws_bytes, void* stream);

/* -- K2: histogram of floor((r - gmin) / width) over valid r
 *        (binning.py:110-116 via pipeline.py:214-224).
 * Dense: counts[q] for q in [0, nbins), nbins = floor((gmax-gmin)/width)+1;
 *        counts is zeroed by the call.
 * Sparse: sorted distinct keys (bit patterns of the non-negative double
 *        ordinal, -0 canonicalised) + counts + *nruns, for spans too wide to
 *        densify. */
int nmk_hist_dense(const void* base, const void* cur, uint64_t n, int dtype,
                   const nmk_stats* stats, double width, uint64_t nbins,
                   unsigned long long* counts, void* stream);
size_t nmk_hist_sparse_ws_bytes(uint64_t n);
int nmk_hist_sparse(const void* base, const void* cur, uint64_t n, int dtype,
                    const nmk_stats* stats, double width,
                    unsigned long long* keys, unsigned long long* counts,
                    unsigned long long* nruns, void* ws, size_t ws_bytes, void* stream);
/* Merge of gathered sparse histograms (binning.py:119-132): sort by key and
 * sum counts of equal keys. keys/counts hold n_in entries; output in place. */
size_t nmk_hist_merge_ws_bytes(uint64_t n_in);
int nmk_hist_merge(unsigned long long* keys, unsigned long long* counts, uint64_t n_in,
                   unsigned long long* nruns, void* ws, size_t ws_bytes, void* stream);

/* Histograms of a ratio ARRAY (binning.histogram_of / build_histogram,
 * binning.py:102-116; merge_histograms, binning.py:119-132) for callers that
 * already hold ratios.  ordinals/counts receive the sorted distinct ordinals
 * floor(RN(RN(r - origin) / width)) as f64 (np.unique order: -0 merged into
 * +0, NaN last, one NaN bin) and their counts; *nruns their number.
 * valid (nullable, u8[n]): elements with 0 are excluded.
 * nmk_hist_merge_values sorts and sums gathered (ordinal, count) pairs in
 * place (n_in entries) -- the device form of merge_histograms. */
size_t nmk_hist_values_ws_bytes(uint64_t n);
int nmk_hist_values(const double* ratios, const uint8_t* valid, uint64_t n, double origin, double width,
                    double* ordinals, unsigned long long* counts, unsigned long long* nruns,
                    void* ws, size_t ws_bytes, void* stream);
int nmk_hist_merge_values(double* ordinals, unsigned long long* counts, uint64_t n_in,
                          unsigned long long* nruns, void* ws, size_t ws_bytes, void* stream);

/* -- K3: single-CTA top-k + auto-B + quantisation + cuts
 *        (binning.py:135-152,155-206; pipeline.py:112-124,163-167,229).
 * keys == NULL selects the dense form (ordinal = array index, nbins = m_max);
 * counts then holds nbins + 1 entries, the last being K2's out-of-span
 * tripwire, which must be 0 (model->status = NMK_ERR_ARG otherwise).
 * nruns: device count for the sparse form (NULL for dense).
 * bits < 0 selects B automatically over [2, 16].
 * centers/cuts: capacity cap_k doubles; centers_t: cap_k elements of dtype. */
int nmk_select(const unsigned long long* keys, const unsigned long long* counts,
               uint64_t m_max, const unsigned long long* nruns,
               const nmk_stats* stats, double width, double tolerance,
               int bits, uint64_t n_total, int dtype,
               double* centers, double* cuts, void* centers_t, uint64_t cap_k,
               nmk_model* model, void* stream);

/* Coverage table of select_index_length (binning._coverage_by_bits,
 * binning.py:165-174): coverage[B - bits_lo] = total count of the
 * min(2^B - 1, m) most populous selectable bins, B in [bits_lo, bits_hi]
 * (2 <= lo <= hi <= 30).  Same histogram forms and stats as nmk_select
 * (stats->gmin = origin, stats->nvalid > 0); model is scratch (status
 * NMK_ERR_EMPTY_HIST and zero coverage when no bin is selectable). */
int nmk_coverage(const unsigned long long* keys, const unsigned long long* counts, uint64_t m_max,
                 const unsigned long long* nruns, const nmk_stats* stats, double width,
                 int bits_lo, int bits_hi, unsigned long long* coverage, nmk_model* model, void* stream);

/* Nearest center and compressibility on a ratio array (binning.nearest_center
 * / compressible_mask, binning.py:287-301,350-359): idx = searchsorted(cuts,
 * v, 'left') with cuts = RN(0.5*RN(c[i]+c[i+1])) (NaN -> k-1; k == 1 -> 0),
 * dist = |v - c[idx]|, flag = valid && dist <= tolerance.  centers: k
 * strictly increasing f64.  dist is nullable. */
int nmk_nearest_center(const double* values, uint64_t n, const double* centers, int k,
                       long long* idx, double* dist, void* stream);
int nmk_compressible_mask(const double* ratios, const uint8_t* valid, uint64_t n,
                          const double* centers, int k, double tolerance,
                          uint8_t* flags, long long* idx, void* stream);

/* -- K4: fused classify + round-trip filter + B-bit pack + stable compaction
 *        (binning.py:287-301,350-359; pipeline.py:143-160,238-288; codec.py:83-92)
 * Encodes the local element range [elem0, elem0 + n_local) of a global
 * stream of n_total elements.  Block b (global ordinal) of the packed index
 * stream lands at packed + (b - b0) * block_stride, b0 = elem0 / epb,
 * block_stride >= ceil(epb*bits/8) and a multiple of 16.
 * exact: n_local elements of capacity; prefix: local prefix per local block
 * (entry for a block whose start precedes elem0 is left untouched);
 * n_inc: device u64 total of local incompressible values.
 * recon (nullable, n_local elements of dtype): also write the decoder's
 * reconstruction of every local element -- T((1+c)*base) or the exact value
 * -- bit-identical to nmk_decode's output (compress_series). */
size_t nmk_encode_ws_bytes(uint64_t n_local, uint64_t elem0, uint64_t epb, int dtype);
int nmk_encode(const void* base, const void* cur, uint64_t n_local, uint64_t elem0,
               uint64_t n_total, int dtype, const double* centers, const double* cuts,
               int k, int bits, double tol_bin, double tolerance, uint64_t epb,
               uint8_t* packed, uint64_t block_stride, void* exact,
               unsigned long long* prefix, unsigned long long* n_inc, void* recon,
               void* ws, size_t ws_bytes, void* stream);

/* -- K5: fused unpack + sentinel scan + reconstruct, batched over segments
 *        (codec.py:95-105,204-239; core.py:158-208)
 * packed: blocks first_block .. at block_stride; prefix_rel[b - first_block]
 * = incompressible count before block b minus that before first_block; exact
 * points at the first exact value of first_block (n_exact available).
 * Segment s decodes [seg_start[s], seg_start[s]+seg_count[s]) (global element
 * indices) reading base[seg_out[s] + i] and writing out[seg_out[s] + i].
 * seg_* are HOST arrays of nseg entries. */
size_t nmk_decode_ws_bytes(const uint64_t* h_seg_start, const uint64_t* h_seg_count,
                           int nseg, uint64_t epb, uint64_t first_block);
int nmk_decode(const uint8_t* packed, uint64_t block_stride, uint64_t first_block,
               int bits, uint64_t epb, uint64_t n_total,
               const unsigned long long* prefix_rel, const double* centers, int k,
               const void* exact, uint64_t n_exact, const void* base, void* out, int dtype,
               const uint64_t* h_seg_start, const uint64_t* h_seg_count,
               const uint64_t* h_seg_out, int nseg,
               nmk_segment_info* seg_info, nmk_decode_err* err,
               void* ws, size_t ws_bytes, void* stream);

/* -- optional lossless stage on the GPU (codec.compress_block, codec.py:108-116)
 * Raw RFC 1951 stream per index block: block b's packed bytes (block_len,
 * last_len for the final block) at packed + b * block_stride.  Segments of
 * seg_bytes (multiple of 16, 64..65535) are LZ77 + fixed-Huffman coded
 * independently and joined by byte-aligning empty stored blocks, so any
 * inflater reproduces the input.  out (capacity nmk_deflate_bound) receives
 * the streams back to back; block_off[0..nblocks] (device) their offsets,
 * block_off[nblocks] = total bytes.  Not byte-equal to zlib's output. */
size_t nmk_deflate_ws_bytes(uint64_t nblocks, uint64_t block_len, uint32_t seg_bytes);
uint64_t nmk_deflate_bound(uint64_t nblocks, uint64_t block_len, uint32_t seg_bytes);
int nmk_deflate(const uint8_t* packed, uint64_t block_stride, uint64_t nblocks, uint64_t block_len,
                uint64_t last_len, uint32_t seg_bytes, uint8_t* out, unsigned long long* block_off,
                void* ws, size_t ws_bytes, void* stream);

/* -- lossless stage, decode half (codec.decompress_block, codec.py:119-128)
 * Inflates nstreams raw RFC 1951 streams -- stream s is comp[comp_off[s] ..
 * comp_off[s+1]) (comp_off: device, nstreams + 1 entries; comp 8-byte aligned
 * and readable 16 bytes past comp_off[nstreams]) -- into
 * out + out_off[s] (out_off: device, nullable = s * out_stride), capacity
 * out_stride bytes each, one warp per stream.  Any raw DEFLATE stream (zlib's or nmk_deflate's) is accepted.
 * status[s]: 0 ok, 1 bad block type, 2 stored LEN/NLEN mismatch, 3 bad
 * dynamic header, 4 bad Huffman code / symbol, 5 bad distance, 6 input ends
 * before the final block, 7 bytes after the final block, 8 output past
 * out_stride; produced[s]: bytes written. */
int nmk_inflate(const uint8_t* comp, const unsigned long long* comp_off, uint64_t nstreams, uint8_t* out,
                uint64_t out_stride, const unsigned long long* out_off, unsigned* status,
                unsigned long long* produced, void* stream);

/* -- sync-free (graph-capturable) variants ---------------------------------
 * Every decision scalar stays on the device, so a whole compress + decompress
 * step can be enqueued (or captured in a CUDA graph) without a host round
 * trip; the host reads stats/model/n_inc once at the end and reruns the
 * general path in the rare cases flagged there (NMK_ERR_NEEDS_SPARSE).
 *  - nmk_hist_prep: dense span from stats into stats->reserved, zero counts.
 *  - nmk_hist_dense_dev: K2 reading the span from stats->reserved; with
 *    `keys` from nmk_minmax it reads 4 bytes per element instead of both
 *    snapshots and re-reads (base, cur) only where a key cannot decide.
 *  - nmk_select with m_max == 0 and keys == NULL reads the span likewise
 *    (and sets model->status = NMK_ERR_NEEDS_SPARSE if it was too wide).
 *  - nmk_encode_dev: K4 reading k and tol_bin from `model`; k_cap bounds k
 *    (sizes shared memory); does nothing if model->status != 0.
 *  - nmk_decode_dev: K5 reading k from `model` and the exact-value count
 *    from the device scalar `n_exact`; segments are passed by value
 *    (nseg <= NMK_DEV_MAX_SEG), so nothing is copied from the host. */
#define NMK_DEV_MAX_SEG 4
int nmk_hist_prep(nmk_stats* stats, double width, uint64_t cap_bins,
                  unsigned long long* counts, void* stream);
int nmk_hist_dense_dev(const void* base, const void* cur, const float* keys, uint64_t n,
                       int dtype, const nmk_stats* stats, double width,
                       unsigned long long* counts, void* stream);
/* nmk_hist_dense_dev with hints from the previous step (span_hint: its dense
 * span, 0 = none; spread_hint: its two largest bins held under 3/4 of the
 * valid ratios, nmk_model.coverage[0..1] vs stats.nvalid): picks the launch shape and
 * counting policy -- a 512-thread CTA per SM with 96 KB of counters for
 * spans of 8K..24K bins, a no-hot-bin direct loop for spread fields.  The
 * counts never depend on the hints. */
int nmk_hist_dense_dev2(const void* base, const void* cur, const float* keys, uint64_t n,
                        int dtype, const nmk_stats* stats, double width,
                        unsigned long long* counts, uint64_t span_hint, int spread_hint, void* stream);
int nmk_encode_dev(const void* base, const void* cur, uint64_t n_local, uint64_t elem0,
                   uint64_t n_total, int dtype, const double* centers, const double* cuts,
                   const nmk_model* model, int k_cap, int bits, double tolerance, uint64_t epb,
                   uint8_t* packed, uint64_t block_stride, void* exact,
                   unsigned long long* prefix, unsigned long long* n_inc, void* recon,
                   void* ws, size_t ws_bytes, void* stream);
/* K4 keyed mode: as nmk_encode_dev, classifying from nmk_minmax's f32 ratio
 * keys (16-byte aligned float[n_local]) against the histogram bins of
 * `stats` (gmin, gmax, dense span from nmk_hist_prep) and `width` (= 2E), so
 * it reads 4 bytes per element; (base, cur) are re-read only where a key
 * cannot decide, for the incompressible values and for `recon`.  Falls back
 * to reading both snapshots when the centers are not on the bin grid.
 * Replaces the same reference phases as nmk_encode (pipeline.py:232-288). */
int nmk_encode_keyed_dev(const float* keys, const nmk_stats* stats, double width,
                         const void* base, const void* cur, uint64_t n_local, uint64_t elem0,
                         uint64_t n_total, int dtype, const double* centers, const double* cuts,
                         const nmk_model* model, int k_cap, int bits, double tolerance, uint64_t epb,
                         uint8_t* packed, uint64_t block_stride, void* exact,
                         unsigned long long* prefix, unsigned long long* n_inc, void* recon,
                         void* ws, size_t ws_bytes, void* stream);
int nmk_decode_dev(const uint8_t* packed, uint64_t block_stride, uint64_t first_block,
                   int bits, uint64_t epb, uint64_t n_total,
                   const unsigned long long* prefix_rel, const double* centers,
                   const nmk_model* model, const void* exact,
                   const unsigned long long* n_exact, const void* base, void* out, int dtype,
                   const uint64_t* h_seg_start, const uint64_t* h_seg_count,
                   const uint64_t* h_seg_out, int nseg, nmk_segment_info* seg_info,
                   nmk_decode_err* err, void* ws, size_t ws_bytes, void* stream);

/* Launch-count hints for a pipeline that repeats (one kernel fewer each in
 * the captured step); like K2's hints they come from the previous step's
 * host check and never change a result:
 *  - nmk_minmax_prep: nmk_minmax + nmk_hist_prep in one launch, for a
 *    single-rank pipeline (no exchange of the stats in between): every CTA
 *    clears its share of counts up front and the last CTA decides the span.
 *  - nmk_encode_keyed_dev2, keyed_hint = 1: the keyed kernel applied on the
 *    previous step (mode word 1 at nmk_encode_ws_mode_offset in ws), so the
 *    snapshot-reading fallback kernel is not launched; should the keyed mode
 *    not apply after all, the keyed kernel finishes on its exact per-element
 *    path (mode word 2: correct, slower -- drop the hint).
 *  - nmk_decode_dev2, ring_hint = nmk_decode_ring_for(n_exact, n_elems) of
 *    the previous step: only that TMA ring depth is launched (0: both, the
 *    device picks). */
int nmk_minmax_prep(const void* base, const void* cur, uint64_t n, int dtype, nmk_stats* stats,
                    float* keys, double width, uint64_t cap_bins, unsigned long long* counts,
                    void* ws, size_t ws_bytes, void* stream);
int nmk_encode_keyed_dev2(const float* keys, const nmk_stats* stats, double width,
                          const void* base, const void* cur, uint64_t n_local, uint64_t elem0,
                          uint64_t n_total, int dtype, const double* centers, const double* cuts,
                          const nmk_model* model, int k_cap, int bits, double tolerance, uint64_t epb,
                          uint8_t* packed, uint64_t block_stride, void* exact,
                          unsigned long long* prefix, unsigned long long* n_inc, void* recon,
                          int keyed_hint, void* ws, size_t ws_bytes, void* stream);
size_t nmk_encode_ws_mode_offset(uint64_t n_local, uint64_t elem0, uint64_t epb, int dtype);
int nmk_decode_dev2(const uint8_t* packed, uint64_t block_stride, uint64_t first_block,
                    int bits, uint64_t epb, uint64_t n_total,
                    const unsigned long long* prefix_rel, const double* centers,
                    const nmk_model* model, const void* exact,
                    const unsigned long long* n_exact, const void* base, void* out, int dtype,
                    const uint64_t* h_seg_start, const uint64_t* h_seg_count,
                    const uint64_t* h_seg_out, int nseg, nmk_segment_info* seg_info,
                    nmk_decode_err* err, int ring_hint, void* ws, size_t ws_bytes, void* stream);
int nmk_decode_ring_for(uint64_t n_exact, uint64_t n_elems);

/* -- 64-bit radix sort (k_sort.cu): the sort under nmk_hist_sparse / nmk_hist_merge
 * (np.unique / the sorted merge of binning.py:110-132), exposed for tests.
 * Stable, ascending; vals_in may be NULL (keys only); outputs must not alias inputs. */
size_t nmk_sort64_ws_bytes(uint64_t n, int with_vals);
int nmk_sort64(const unsigned long long* keys_in, unsigned long long* keys_out,
               const unsigned long long* vals_in, unsigned long long* vals_out, uint64_t n,
               void* ws, size_t ws_bytes, void* stream);

/* -- standalone codec kernels (codec.py:83-105) ---------------------------- */
int nmk_pack(const uint32_t* codes, uint64_t n, int bits, uint8_t* out, void* stream);
int nmk_unpack(const uint8_t* packed, uint64_t n, int bits, uint32_t* codes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* NMK_B200_H */
