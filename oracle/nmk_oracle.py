"""CPU oracle for the NUMARCK per-timestep hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference algorithm (the `nmk`
package under /root/reference/pkg/src/nmk) written for checking the CUDA path.
It is imported only by ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``.  The product path
(``paper_1703_02438_b200``) never imports it and has no CPU fallback.

Parity status: PINNED.  ``tests/test_oracle_golden.py`` checks every function
here against golden vectors produced by running the reference itself
(``tests/golden/make_golden.py``, committed together with its output).

Each function cites the reference file:line it restates.  The arithmetic is
IEEE-754 binary64 throughout, in the same operation order as the reference,
so results are bit-identical.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

SENTINEL_OF = lambda bits: (1 << bits) - 1  # noqa: E731  (pipeline.py:266, binning.py:95-97)


# ---------------------------------------------------------------------------
# Phase 1 — change ratios + min/max          core.py:115-137, pipeline.py:190-212
# ---------------------------------------------------------------------------

def ratios_of(base: np.ndarray, cur: np.ndarray):
    """Eq. 1 with the zero / non-finite rules (core.py:115-137).

    Returns (r float64[n], valid bool[n]); invalid slots carry +0.0.
    """
    b = np.asarray(base).astype(np.float64)
    x = np.asarray(cur).astype(np.float64)
    with np.errstate(all="ignore"):
        r = np.divide(np.subtract(x, b), b)
    ok = np.isfinite(r)
    ok &= np.isfinite(b)
    ok &= np.isfinite(x)
    zz = (b == 0.0) & (x == 0.0)
    r[zz] = 0.0          # 0/0 -> defined as "no change" (core.py:131-134)
    ok |= zz
    r[~ok] = 0.0         # invalid slots are zero-filled (core.py:135-136)
    return r, ok


def minmax_of(r: np.ndarray, valid: np.ndarray):
    """Global min/max over valid ratios, or None when none is valid
    (pipeline.py:194-197, 202-210)."""
    if not valid.any():
        return None
    v = r[valid]
    return float(v.min()), float(v.max())


# ---------------------------------------------------------------------------
# Phase 2 — histogram, top-k, B selection, quantisation
#           binning.py:100-206, pipeline.py:112-140, 214-229
# ---------------------------------------------------------------------------

def bin_ordinals(r: np.ndarray, origin: float, width: float) -> np.ndarray:
    """floor((r - origin) / width) as float64 (binning.py:113)."""
    with np.errstate(all="ignore"):
        return np.floor(np.divide(np.subtract(r, origin), width))


def histogram(r_valid: np.ndarray, origin: float, width: float):
    """Sparse histogram: sorted distinct ordinals + int64 counts
    (binning.py:110-116).  -0.0 and +0.0 ordinals merge (np.unique)."""
    q = bin_ordinals(r_valid, origin, width)
    keys, counts = np.unique(q, return_counts=True)
    return keys, counts.astype(np.int64)


def merge(parts):
    """Associative merge of sparse histograms (binning.py:119-132)."""
    if len(parts) == 1:
        return parts[0]
    keys = np.concatenate([p[0] for p in parts])
    cnts = np.concatenate([p[1] for p in parts])
    uk, inv = np.unique(keys, return_inverse=True)
    out = np.zeros(uk.size, dtype=np.int64)
    np.add.at(out, inv, cnts)
    return uk, out


def bin_centers(ordinals: np.ndarray, origin: float, width: float) -> np.ndarray:
    """origin + (m + 0.5) * width, add->mul->add, no FMA (binning.py:50-51)."""
    return np.add(origin, np.multiply(np.add(ordinals, 0.5), width))


def selectable(keys, counts, origin, width):
    """Drop bins whose center is not finite (binning.py:135-139)."""
    c = bin_centers(keys, origin, width)
    keep = np.isfinite(c)
    return keys[keep], counts[keep], c[keep]


def coverage(counts_sel: np.ndarray, lo: int = 2, hi: int = 16) -> dict:
    """Sum of the top min(2^B-1, m) counts per B (binning.py:170-179)."""
    desc = np.sort(counts_sel)[::-1]
    cum = np.cumsum(desc)
    out = {}
    for b in range(lo, hi + 1):
        k = min((1 << b) - 1, desc.size)
        out[b] = int(cum[k - 1]) if k > 0 else 0
    return out


def size_model(n: int, width: int, bits: int, n_inc: int) -> float:
    """Eq. 6 as evaluated by the reference, in Python float arithmetic
    (binning.py:155-167)."""
    return (1 << bits) * width + (n * bits) / 8 + n_inc * width


def auto_bits(counts_sel: np.ndarray, n: int, width: int, lo: int = 2, hi: int = 16) -> int:
    """argmin of the size model, ties to the smaller B (binning.py:182-206)."""
    cov = coverage(counts_sel, lo, hi)
    best, best_size = lo, None
    for b in range(lo, hi + 1):
        s = size_model(n, width, b, n - cov[b])
        if best_size is None or s < best_size:
            best, best_size = b, s
    return best


def top_k(keys, counts, origin, width, bits):
    """Top-k bins by (count desc, ordinal asc); sorted unique centers
    (binning.py:142-152).  Raises ValueError on an empty selection."""
    k_, c_, cen = selectable(keys, counts, origin, width)
    if k_.size == 0:
        raise ValueError("empty histogram")
    k = min((1 << bits) - 1, k_.size)
    order = np.lexsort((k_, -c_))[:k]
    return np.unique(cen[order])


def quantize(centers: np.ndarray, dtype) -> np.ndarray:
    """Round to the storage dtype and back, unique, finite, else [0.0]
    (pipeline.py:112-124)."""
    with np.errstate(all="ignore"):
        q = np.unique(centers.astype(dtype).astype(np.float64))
    q = q[np.isfinite(q)]
    return q if q.size else np.array([0.0])


# ---------------------------------------------------------------------------
# Phase 3 — nearest center + round-trip filter + block alignment
#           binning.py:287-301, 350-359; pipeline.py:143-160, 238-276; codec.py:28-59
# ---------------------------------------------------------------------------

def nearest(r: np.ndarray, centers: np.ndarray):
    """searchsorted over midpoint cuts, ties to the lower index
    (binning.py:287-301).  Returns (idx int64, |r - c[idx]|)."""
    with np.errstate(all="ignore"):
        if centers.size == 1:
            idx = np.zeros(r.size, dtype=np.int64)
        else:
            cuts = np.multiply(0.5, np.add(centers[:-1], centers[1:]))
            idx = np.searchsorted(cuts, r, side="left").astype(np.int64)
        return idx, np.abs(np.subtract(r, centers[idx]))


def classify(r, valid, base, cur, centers, tol_bin, tol):
    """compressible_mask + _roundtrip_filter (binning.py:350-359,
    pipeline.py:143-160).  Returns (flags, idx)."""
    idx, dist = nearest(r, centers)
    flags = valid & (dist <= tol_bin)
    if flags.any():
        b = np.asarray(base).astype(np.float64)
        x = np.asarray(cur).astype(np.float64)
        with np.errstate(all="ignore"):
            rec = np.multiply(np.add(1.0, centers[idx]), b)
            rec = rec.astype(np.asarray(base).dtype).astype(np.float64)
            flags &= np.abs(np.subtract(rec, x)) <= np.multiply(tol, np.abs(b))
    return flags, idx


def elements_per_block(block_bytes: int, bits: int) -> int:
    return (block_bytes * 8) // bits          # codec.py:40-42


def n_blocks(n: int, epb: int) -> int:
    return -(-n // epb)                        # codec.py:44-46


# ---------------------------------------------------------------------------
# Bit packing                                    codec.py:79-105
# ---------------------------------------------------------------------------

def pack(codes: np.ndarray, bits: int) -> bytes:
    """MSB-first B-bit packing, zero-padded to a byte (codec.py:83-92)."""
    codes = np.asarray(codes, dtype=np.uint64)
    if codes.size == 0:
        return b""
    sh = np.arange(bits - 1, -1, -1, dtype=np.uint64)
    bitmat = ((codes[:, None] >> sh) & np.uint64(1)).astype(np.uint8)
    return np.packbits(bitmat.reshape(-1)).tobytes()


def unpack(data: bytes, bits: int, count: int) -> np.ndarray:
    """Inverse of :func:`pack` (codec.py:95-105)."""
    if count == 0:
        return np.zeros(0, dtype=np.int64)
    raw = np.frombuffer(data, dtype=np.uint8, count=(count * bits + 7) // 8)
    bitmat = np.unpackbits(raw, count=count * bits).reshape(count, bits).astype(np.int64)
    w = np.left_shift(np.int64(1), np.arange(bits - 1, -1, -1, dtype=np.int64))
    return bitmat @ w


# ---------------------------------------------------------------------------
# Full encode (phases 1-4a) with the reference's shard/worker structure
# ---------------------------------------------------------------------------

def _shard_bounds(n: int, workers: int):
    edges = np.linspace(0, n, min(workers, n) + 1).astype(np.int64)   # pipeline.py:84-87
    return [(int(a), int(b)) for a, b in zip(edges[:-1], edges[1:])]


def encode(base: np.ndarray, cur: np.ndarray, tolerance: float = 1e-3,
           bits: int | None = None, block_bytes: int = 1 << 20, workers: int = 1):
    """Phases 1 -> 4a of compress_pair (pipeline.py:170-288), without zlib.

    Returns a dict with every intermediate the CUDA path must reproduce:
    gmin/gmax, hist (keys, counts), bits, centers (f64, quantised), epb,
    nblocks, flags, idx, codes, blocks (list of packed bytes per block),
    exact (incompressible values, element order), prefix (u64), n_inc.
    """
    base = np.ascontiguousarray(base)
    cur = np.ascontiguousarray(cur)
    n = base.shape[0]
    dt = base.dtype
    L = dt.itemsize
    shards = _shard_bounds(n, workers)
    pool = ThreadPoolExecutor(workers) if workers > 1 else None
    run = (lambda f, xs: list(pool.map(f, xs))) if pool else (lambda f, xs: [f(s) for s in xs])

    r = np.empty(n, dtype=np.float64)
    valid = np.empty(n, dtype=bool)

    def p1(sh):
        a, b_ = sh
        r[a:b_], valid[a:b_] = ratios_of(base[a:b_], cur[a:b_])
        return minmax_of(r[a:b_], valid[a:b_])

    ext = [e for e in run(p1, shards) if e is not None]
    out = {"n": n, "dtype": dt}
    if not ext:  # degenerate (pipeline.py:202-207, 163-167)
        out.update(gmin=None, gmax=None, hist=None)
        bits_ = bits if bits is not None else 2
        centers = np.array([0.0])
        tol_bin = float(tolerance)
    else:
        gmin = min(e[0] for e in ext)
        gmax = max(e[1] for e in ext)
        width = 2.0 * tolerance

        def p2(sh):
            a, b_ = sh
            v = valid[a:b_]
            return histogram(r[a:b_][v], gmin, width)

        parts = [p for p in run(p2, shards) if p[0].size]
        keys, counts = merge(parts)
        if bits is None:
            _, cs, _ = selectable(keys, counts, gmin, width)
            bits_ = auto_bits(cs, n, L)
        else:
            bits_ = bits
        centers = quantize(top_k(keys, counts, gmin, width, bits_), dt)
        tol_bin = width / 2.0
        out.update(gmin=gmin, gmax=gmax, hist=(keys, counts))

    flags = np.empty(n, dtype=bool)
    idx = np.empty(n, dtype=np.int64)

    def p3(sh):
        a, b_ = sh
        f, ix = classify(r[a:b_], valid[a:b_], base[a:b_], cur[a:b_], centers,
                         tol_bin, tolerance)
        flags[a:b_] = f
        idx[a:b_] = ix

    run(p3, shards)
    epb = elements_per_block(block_bytes, bits_)
    nb = n_blocks(n, epb)
    codes = np.where(flags, idx, SENTINEL_OF(bits_))
    inc_pos = np.flatnonzero(~flags)
    exact = cur[inc_pos]
    per_block = np.bincount(inc_pos // epb, minlength=nb)
    prefix = np.zeros(nb, dtype=np.uint64)
    prefix[1:] = np.cumsum(per_block[:-1])

    owners = [o for o in np.array_split(np.arange(nb), min(workers, nb)) if o.size]
    blocks = [None] * nb

    def p4(own):
        for b_ in own:
            lo = int(b_) * epb
            blocks[b_] = pack(codes[lo:min(lo + epb, n)], bits_)

    run(p4, owners)
    if pool:
        pool.shutdown()
    out.update(bits=bits_, centers=centers, epb=epb, nblocks=nb, flags=flags,
               idx=idx, codes=codes, blocks=blocks, exact=exact, prefix=prefix,
               n_inc=int(inc_pos.size))
    return out


# ---------------------------------------------------------------------------
# Decode                                core.py:158-208, codec.py:204-239
# ---------------------------------------------------------------------------

def reconstruct(base, centers, codes, exact, bits):
    """Inverse transform for one range (core.py:158-208)."""
    base = np.asarray(base)
    codes = np.asarray(codes)
    if codes.shape[0] != base.shape[0]:
        raise ValueError("indices and base cover different element counts")
    sent = SENTINEL_OF(bits)
    inc = codes == sent
    ci = codes[~inc]
    if ci.size and int(ci.max()) >= len(centers):
        raise ValueError(f"index {int(ci.max())} out of range for {len(centers)} centers")
    if ci.size and int(ci.min()) < 0:
        raise ValueError("negative bin index")
    need = int(inc.sum())
    exact = np.asarray(exact)
    if exact.shape[0] < need:
        raise ValueError(f"incompressible values exhausted: need {need}, have {exact.shape[0]}")
    if exact.shape[0] > need:
        raise ValueError(f"incompressible values not fully consumed: need {need}, have {exact.shape[0]}")
    out = np.empty(base.shape[0], dtype=base.dtype)
    if ci.size:
        c = np.asarray(centers, dtype=np.float64)[ci]
        b = base[~inc].astype(np.float64)
        out[~inc] = np.multiply(np.add(1.0, c), b).astype(base.dtype)
    if need:
        out[inc] = exact.astype(base.dtype, copy=False)
    return out


def decode_range(blocks, bits, epb, n, prefix, exact_all, centers, start, count, base):
    """Range decode from per-block packed bytes (codec.py:204-239)."""
    if start < 0 or count < 0 or start + count > n:
        raise ValueError(f"range [{start}, {start + count}) outside 0..{n}")
    base = np.asarray(base)
    if base.shape[0] != count:
        raise ValueError(f"base slice holds {base.shape[0]} elements, need {count}")
    if count == 0:
        return np.zeros(0, dtype=base.dtype)
    first, last = start // epb, (start + count - 1) // epb
    lo_el = first * epb
    parts = []
    for b_ in range(first, last + 1):
        s, e = b_ * epb, min((b_ + 1) * epb, n)
        parts.append(unpack(blocks[b_], bits, e - s))
    span = np.concatenate(parts)
    off = start - lo_el
    codes = span[off:off + count]
    sent = SENTINEL_OF(bits)
    before = int(prefix[first]) + int(np.count_nonzero(span[:off] == sent))
    need = int(np.count_nonzero(codes == sent))
    return reconstruct(base, centers.astype(np.float64), codes,
                       exact_all[before:before + need], bits)


def decode(enc: dict, base: np.ndarray, rng=None):
    """Full (rng=None) or range decode from an :func:`encode` result."""
    n = enc["n"]
    start, count = (0, n) if rng is None else rng
    centers = enc["centers"].astype(enc["dtype"]).astype(np.float64)
    return decode_range(enc["blocks"], enc["bits"], enc["epb"], n, enc["prefix"],
                        enc["exact"], centers, start, count, base)


def encode_series(snapshots, tolerance=1e-3, bits=None, block_bytes=1 << 20, workers=1):
    """Chain encode against the previous reconstruction (pipeline.py:343-372)."""
    recon = np.ascontiguousarray(snapshots[0]).copy()
    encs = []
    for snap in snapshots[1:]:
        e = encode(recon, snap, tolerance, bits, block_bytes, workers)
        encs.append(e)
        recon = decode(e, recon)
    return encs


def default_workers() -> int:
    return os.cpu_count() or 1
