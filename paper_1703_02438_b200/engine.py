"""Device-resident engine: the NUMARCK hot path on one GPU (or one rank's
element range of a multi-GPU run) over torch-owned HBM buffers.

    encode(base, cur, tolerance, bits, block_bytes)   -> DeviceEncoding
    decode(enc-like geometry, base, segments)          -> reconstructed values

Phases and the reference code they replace (pkg/src/nmk/...):
    K1 nmk_minmax      pipeline.py:190-212 + core.py:115-137
    K2 nmk_hist_*      pipeline.py:214-224 + binning.py:110-132
    K3 nmk_select      pipeline.py:127-140,229 + binning.py:135-206 + pipeline.py:112-124
    K4 nmk_encode      pipeline.py:232-288 (+ binning.py:287-301,350-359, codec.py:83-92)
    K5 nmk_decode      codec.py:204-239 + codec.py:95-105 + core.py:158-208

Host<->device traffic inside encode is three small reads (32 B of stats,
160 B of model header, 8 B of n_inc); everything else stays in HBM.  An
optional ``comm`` object inserts the three multi-GPU exchanges (min/max,
histogram, incompressible-count scan) between the phases.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N

DENSE_MAX_BINS = 1 << 22      # must match kGlobalBins in csrc/k_hist.cu
AUTO_BITS_HI = 16             # binning.DEFAULT_BITS_RANGE upper end
MIN_BITS, MAX_BITS = 2, 30


def _torch():
    return N.require_cuda()


def torch_dtype_code(t) -> int:
    import torch
    if t.dtype == torch.float64:
        return N.NMK_F64
    if t.dtype == torch.float32:
        return N.NMK_F32
    raise ValueError(f"unsupported snapshot dtype {t.dtype}")


def _p(t) -> int:
    return t.data_ptr()


def _stream(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def elements_per_block(block_bytes: int, bits: int) -> int:
    """codec.BlockLayout.elements_per_block (codec.py:40-42)."""
    return (block_bytes * 8) // bits


def block_stride(epb: int, bits: int) -> int:
    """Device stride between packed blocks: ceil(epb*B/8) rounded up to 16 B."""
    return ((epb * bits + 7) // 8 + 15) // 16 * 16


class Workspace:
    """Grow-only cache of device scratch buffers, one per (name)."""

    def __init__(self, device=None):
        import torch
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._bufs: dict[str, "torch.Tensor"] = {}

    def get(self, name: str, nbytes: int, zero: bool = False):
        import torch
        nbytes = max(int(nbytes), 256)
        t = self._bufs.get(name)
        if t is None or t.numel() < nbytes:
            cap = nbytes if t is None else max(nbytes, t.numel() + t.numel() // 4)
            t = (torch.zeros if zero else torch.empty)(cap, dtype=torch.uint8, device=self.device)
            self._bufs[name] = t
        return t

    def typed(self, name: str, count: int, dtype, zero: bool = False):
        import torch
        itemsize = torch.empty(0, dtype=dtype).element_size()
        return self.get(name, count * itemsize, zero)[: max(count, 1) * itemsize].view(dtype)[:count]


_default_ws: dict = {}


def default_workspace():
    import torch
    dev = torch.cuda.current_device()
    ws = _default_ws.get(dev)
    if ws is None:
        ws = _default_ws[dev] = Workspace(torch.device("cuda", dev))
    return ws


@dataclass
class DeviceEncoding:
    """Everything compress_pair's phases 1-4a produce, resident in HBM."""

    n: int                      # global element count
    elem0: int                  # first element of this range
    n_local: int
    dtype: np.dtype
    bits: int
    k: int
    epb: int
    nblocks: int                # global block count
    b0: int                     # first global block touched by this range
    stride: int
    centers: object             # torch f64 [k]
    centers_t: object           # torch T [k]  (what CompressedVariable stores)
    packed: object              # torch u8 [(b1-b0+1) * stride]
    exact: object               # torch T [n_inc]
    prefix: object              # torch i64 [b1-b0+1]  (u64 values)
    n_inc: int
    gmin: float | None
    gmax: float | None
    nvalid: int
    hist_form: str
    tol_bin: float
    phase_ms: dict = field(default_factory=dict)

    @property
    def sentinel(self) -> int:
        return (1 << self.bits) - 1

    def block_lengths(self) -> np.ndarray:
        """Packed bytes per block (codec.packed_size of each block's count)."""
        b = np.arange(self.b0, self.b0 + self.prefix.numel(), dtype=np.int64)
        cnt = np.minimum((b + 1) * self.epb, self.n) - b * self.epb
        return (cnt * self.bits + 7) // 8


def _read_struct(t, cls):
    raw = t.cpu().numpy().tobytes()
    return cls.from_buffer_copy(raw[: ctypes.sizeof(cls)])


class _PhaseClock:
    def __init__(self, enabled: bool, stream):
        import torch
        self.enabled = enabled
        self.stream = stream
        self.marks = []
        if enabled:
            self._ev = torch.cuda.Event

    def mark(self, name):
        if self.enabled:
            e = self._ev(enable_timing=True)
            e.record(self.stream)
            self.marks.append((name, e))

    def result(self) -> dict:
        if not self.enabled or len(self.marks) < 2:
            return {}
        self.marks[-1][1].synchronize()
        out = {}
        for (n0, e0), (n1, e1) in zip(self.marks[:-1], self.marks[1:]):
            out[n1] = out.get(n1, 0.0) + e0.elapsed_time(e1)
        return out


def encode(base, cur, tolerance: float, bits: int | None = None, block_bytes: int = 1 << 20,
           *, elem0: int = 0, n_total: int | None = None, comm=None, ws: Workspace | None = None,
           stream=None, timing: bool = False, recon=None, keyed: bool = True) -> DeviceEncoding:
    """Run K1..K4 on device tensors ``base``/``cur`` (1-D, same dtype, CUDA).

    ``keyed``: K1 stores f32 ratio keys; for a dense histogram K2 and K4 then
    read 4 bytes per element instead of both snapshots (same bytes out).

    ``elem0``/``n_total`` place this range inside a longer global stream (a
    multi-GPU shard); ``comm`` (see distributed.py) performs the exchanges.
    ``recon`` (a tensor like ``cur``) receives K4's reconstruction of every
    element, bit-identical to decoding the result.
    """
    torch = _torch()
    if base.device.type != "cuda" or cur.device.type != "cuda":
        raise ValueError("encode expects CUDA tensors")
    if base.dim() != 1 or cur.shape != base.shape or cur.dtype != base.dtype:
        raise ValueError("base/current must be 1-D tensors of equal shape and dtype")
    base = base.contiguous()
    cur = cur.contiguous()
    dt = torch_dtype_code(base)
    np_dt = np.dtype("<f8") if dt == N.NMK_F64 else np.dtype("<f4")
    L = np_dt.itemsize
    n_local = base.numel()
    n = n_total if n_total is not None else n_local
    if elem0 < 0 or elem0 + n_local > n or n < 1:
        raise ValueError("bad element range")
    if bits is not None and not MIN_BITS <= bits <= MAX_BITS:
        raise ValueError(f"bits must be in [{MIN_BITS}, {MAX_BITS}]")
    ws = ws or default_workspace()
    lib = N.lib()
    st = _stream(stream)
    s_obj = stream if stream is not None else torch.cuda.current_stream()
    clock = _PhaseClock(timing, s_obj)
    clock.mark("start")

    # ---- K1: ratio + min/max ------------------------------------------------
    stats = ws.typed("stats", 4, torch.int64)
    if n_local > 0:
        mm_bytes = lib.nmk_minmax_ws_bytes(n_local)
        mm_ws = ws.get("minmax", mm_bytes, zero=True)
        keys = ws.typed("ratio_keys", n_local + 4, torch.float32) if keyed else None
        N.check(lib.nmk_minmax(_p(base), _p(cur), n_local, dt, _p(stats), _p(keys) if keyed else None, _p(mm_ws),
                               mm_bytes, st))
    else:
        stats.copy_(torch.tensor([0x7FF0000000000000, -0x10000000000000, 0, 0], dtype=torch.int64))
    if comm is not None:
        comm.allreduce_stats(stats)
    clock.mark("change_ratio")
    sv = _read_struct(stats, N.NmkStats)
    nvalid = int(sv.nvalid)
    width = 2.0 * tolerance

    # ---- K2: histogram --------------------------------------------------------
    dummy = ws.typed("dummy", 2, torch.int64)
    bits_cap = bits if bits is not None else AUTO_BITS_HI
    keys_t = counts_t = nruns_t = None
    m_max = 1
    form = "none"
    if nvalid > 0:
        gmin, gmax = float(sv.gmin), float(sv.gmax)
        span = (gmax - gmin) / width
        dense = math.isfinite(span) and span < DENSE_MAX_BINS
        nbins = int(math.floor(span)) + 1 if dense else 0
        if comm is not None:
            dense = comm.agree_dense(dense)
        if dense:
            form = "dense"
            counts_t = ws.typed("hist_counts", nbins + 1, torch.int64)
            if n_local > 0 and keyed:
                # device span (same arithmetic as above) + K2 from the keys
                N.check(lib.nmk_hist_prep(_p(stats), width, DENSE_MAX_BINS, _p(counts_t), st))
                N.check(lib.nmk_hist_dense_dev2(_p(base), _p(cur), _p(keys), n_local, dt, _p(stats), width,
                                                _p(counts_t), nbins, 0, st))
            elif n_local > 0:
                N.check(lib.nmk_hist_dense(_p(base), _p(cur), n_local, dt, _p(stats), width, nbins,
                                           _p(counts_t), st))
            else:
                counts_t.zero_()
            if comm is not None:
                comm.allreduce_counts(counts_t)
            m_max = nbins
        else:
            form = "sparse"
            cap = max(n_local, 1)
            keys_t = ws.typed("hist_keys", cap, torch.int64)
            counts_t = ws.typed("hist_sp_counts", cap, torch.int64)
            nruns_t = ws.typed("hist_nruns", 1, torch.int64)
            if n_local > 0:
                sp_bytes = lib.nmk_hist_sparse_ws_bytes(n_local)
                sp_ws = ws.get("hist_sparse_ws", sp_bytes)
                N.check(lib.nmk_hist_sparse(_p(base), _p(cur), n_local, dt, _p(stats), width, _p(keys_t),
                                            _p(counts_t), _p(nruns_t), _p(sp_ws), sp_bytes, st))
            else:
                nruns_t.zero_()
            if comm is not None:
                keys_t, counts_t, nruns_t = comm.merge_sparse(keys_t, counts_t, nruns_t, ws)
            m_max = max(keys_t.numel(), 1)
    else:
        gmin = gmax = None

    # ---- K3: selection --------------------------------------------------------
    cap_k = max(1, min((1 << bits_cap) - 1, m_max))
    centers = ws.typed("centers", cap_k, torch.float64)
    cuts = ws.typed("cuts", cap_k, torch.float64)
    centers_t = ws.typed("centers_t", cap_k, base.dtype)
    model_t = ws.typed("model", ctypes.sizeof(N.NmkModel) // 8, torch.int64)
    N.check(lib.nmk_select(
        _p(keys_t) if keys_t is not None else None,
        _p(counts_t) if counts_t is not None else _p(dummy),
        m_max, _p(nruns_t) if nruns_t is not None else None,
        _p(stats), width, float(tolerance), -1 if bits is None else int(bits), n, dt,
        _p(centers), _p(cuts), _p(centers_t), cap_k, _p(model_t), st))
    clock.mark("binning")
    model = _read_struct(model_t, N.NmkModel)
    if model.status == N.NMK_ERR_EMPTY_HIST:
        raise N.NativeError(N.NMK_ERR_EMPTY_HIST, "empty histogram")
    if model.status == N.NMK_ERR_ARG and form == "dense":
        raise N.NativeError(N.NMK_ERR_ARG, "histogram ordinal beyond the dense span (K2 tripwire)")
    if model.status != 0:
        raise N.NativeError(model.status, "nmk_select failed")
    if form == "dense" and n_local > 0:
        trip = int(counts_t[m_max].item()) if counts_t.numel() > m_max else 0
        if trip:
            raise N.NativeError(N.NMK_ERR_ARG, f"histogram ordinal beyond the dense span ({trip})")
    B, k = int(model.bits), int(model.k)

    # ---- K4: encode -----------------------------------------------------------
    epb = elements_per_block(block_bytes, B)
    nblocks = -(-n // epb)
    stride = block_stride(epb, B)
    if n_local > 0:
        b0 = elem0 // epb
        b1 = (elem0 + n_local - 1) // epb
    else:
        b0 = b1 = 0
    nlb = b1 - b0 + 1
    packed = ws.typed("packed", nlb * stride, torch.uint8)
    exact = ws.typed("exact", max(n_local, 1), base.dtype)
    prefix = ws.typed("prefix", nlb, torch.int64)
    prefix.zero_()
    n_inc_t = ws.typed("n_inc", 1, torch.int64)
    if n_local > 0:
        e_bytes = lib.nmk_encode_ws_bytes(n_local, elem0, epb, dt)
        e_ws = ws.get("encode_ws", e_bytes)
        if recon is not None and (recon.shape != cur.shape or recon.dtype != cur.dtype or not recon.is_cuda):
            raise ValueError("recon must be a CUDA tensor like current")
        if keyed and form == "dense":
            N.check(lib.nmk_encode_keyed_dev(_p(keys), _p(stats), width, _p(base), _p(cur), n_local, elem0, n, dt,
                                             _p(centers), _p(cuts), _p(model_t), min(cap_k, (1 << B) - 1), B, float(tolerance), epb,
                                             _p(packed), stride, _p(exact), _p(prefix), _p(n_inc_t),
                                             _p(recon) if recon is not None else None, _p(e_ws), e_bytes, st))
        else:
            N.check(lib.nmk_encode(_p(base), _p(cur), n_local, elem0, n, dt, _p(centers), _p(cuts), k, B,
                                   float(model.tol_bin), float(tolerance), epb, _p(packed), stride, _p(exact),
                                   _p(prefix), _p(n_inc_t), _p(recon) if recon is not None else None, _p(e_ws),
                                   e_bytes, st))
    else:
        n_inc_t.zero_()
    clock.mark("assign_index")
    n_inc = int(n_inc_t.item())
    return DeviceEncoding(
        n=n, elem0=elem0, n_local=n_local, dtype=np_dt, bits=B, k=k, epb=epb, nblocks=nblocks, b0=b0,
        stride=stride, centers=centers[:k], centers_t=centers_t[:k], packed=packed, exact=exact[:n_inc],
        prefix=prefix, n_inc=n_inc, gmin=gmin, gmax=gmax, nvalid=nvalid, hist_form=form,
        tol_bin=float(model.tol_bin), phase_ms=clock.result())


@dataclass
class DecodeResult:
    out: object                     # torch T
    inc_before: np.ndarray          # per segment, relative to the exact pointer
    n_sentinel: np.ndarray          # per segment
    bad_index: bool
    max_bad_index: int
    exhausted: bool


def decode(packed, stride: int, first_block: int, bits: int, epb: int, n_total: int, prefix_rel,
           centers, exact, base, segments, out=None, *, ws: Workspace | None = None, stream=None,
           check: bool = True) -> DecodeResult:
    """K5 over ``segments`` = [(start, count, out_offset), ...] (global indices,
    empty segments not allowed).  ``base``/``out`` are laid out by out_offset;
    ``prefix_rel[b - first_block]`` is the incompressible count before block b
    minus the count before ``first_block``; ``exact`` starts at the first
    exact value of ``first_block``."""
    torch = _torch()
    ws = ws or default_workspace()
    lib = N.lib()
    st = _stream(stream)
    dt = torch_dtype_code(base)
    segs = [(int(a), int(c), int(o)) for a, c, o in segments]
    nseg = len(segs)
    if nseg == 0:
        raise ValueError("no segments")
    s_start = (ctypes.c_uint64 * nseg)(*[a for a, _, _ in segs])
    s_count = (ctypes.c_uint64 * nseg)(*[c for _, c, _ in segs])
    s_out = (ctypes.c_uint64 * nseg)(*[o for _, _, o in segs])
    total_out = max(o + c for _, c, o in segs)
    if out is None:
        out = torch.empty(total_out, dtype=base.dtype, device=base.device)
    k = centers.numel()
    d_bytes = lib.nmk_decode_ws_bytes(s_start, s_count, nseg, epb, first_block)
    d_ws = ws.get("decode_ws", d_bytes)
    info = ws.typed("seg_info", 2 * nseg, torch.int64)
    err = ws.typed("decode_err", 2, torch.int64)
    n_exact = exact.numel()
    exact_ptr = _p(exact) if n_exact else _p(ws.typed("dummy_exact", 1, base.dtype))
    N.check(lib.nmk_decode(_p(packed), stride, first_block, bits, epb, n_total, _p(prefix_rel), _p(centers), k,
                           exact_ptr, n_exact, _p(base), _p(out), dt, s_start, s_count, s_out, nseg,
                           _p(info), _p(err), _p(d_ws), d_bytes, st))
    if not check:
        return DecodeResult(out, None, None, False, 0, False)
    e = _read_struct(err, N.NmkDecodeErr)
    inf = info.cpu().numpy().view(np.uint64).reshape(nseg, 2)
    return DecodeResult(out, inf[:, 0].astype(np.int64), inf[:, 1].astype(np.int64), bool(e.bad_index),
                        int(e.max_bad_index), bool(e.exhausted))


def decode_encoding(enc: DeviceEncoding, base, out=None, *, ws=None, stream=None, check=True) -> DecodeResult:
    """Full decode of this rank's range straight from a DeviceEncoding."""
    # prefix[0] is 0 whether the range starts on a block boundary (count
    # before the block) or inside one (entry left untouched, zeroed); K4
    # zero-fills the packed bytes between the block start and the range.
    return decode(enc.packed, enc.stride, enc.b0, enc.bits, enc.epb, enc.n, enc.prefix, enc.centers,
                  enc.exact, base, [(enc.elem0, enc.n_local, 0)], out, ws=ws, stream=stream, check=check)


# ---------------------------------------------------------------------------
# Sync-free pipeline (explicit B): every decision scalar stays on the device
# ---------------------------------------------------------------------------

ASYNC_COMM_BINS = 1 << 16     # dense span all-reduced without a host round trip


class DevicePipeline:
    """compress (K1..K4) + full decompress (K5) of one element range with no
    host synchronisation: the dense span, k, tol_bin and the exact-value count
    are produced and consumed on the device (nmk_minmax_prep / *_dev entry
    points), all buffers are preallocated, so one step can be enqueued — or
    captured once in a CUDA graph and replayed.  ``check()`` reads the device
    scalars once and reports the rare cases that need the general path (span
    too wide for a dense histogram, empty histogram)."""

    def __init__(self, n_local: int, dtype, tolerance: float, bits: int, block_bytes: int = 1 << 20,
                 *, elem0: int = 0, n_total: int | None = None, comm=None, ws: Workspace | None = None,
                 comm_bins: int | None = None):
        torch = _torch()
        if bits is None or not MIN_BITS <= bits <= MAX_BITS:
            raise ValueError("the sync-free pipeline needs an explicit B in [2, 30]")
        self.torch_dtype = dtype
        self.dt = N.NMK_F64 if dtype == torch.float64 else N.NMK_F32
        self.np_dtype = np.dtype("<f8") if self.dt == N.NMK_F64 else np.dtype("<f4")
        self.n_local, self.elem0 = int(n_local), int(elem0)
        self.n = int(n_total) if n_total is not None else self.n_local
        self.tol, self.bits, self.block_bytes, self.comm = float(tolerance), int(bits), int(block_bytes), comm
        self.width = 2.0 * self.tol
        self.epb = elements_per_block(block_bytes, bits)
        self.nblocks = -(-self.n // self.epb)
        self.stride = block_stride(self.epb, bits)
        self.b0 = self.elem0 // self.epb
        self.nlb = (self.elem0 + self.n_local - 1) // self.epb - self.b0 + 1
        self.k_cap = (1 << bits) - 1
        # K2 launch shape follows the last observed dense span (check()); the
        # counts never depend on it
        self.span_hint = 0
        self.spread_hint = 0
        # launch-count hints, also from check(): the keyed K4 applied (its
        # fallback kernel is not launched) and the K5 ring depth that matched
        self.keyed_hint = 0
        self.ring_hint = 0
        # dense span capacity; with a comm it is also the all-reduced histogram
        # length (fit_comm_bins sizes it to the observed span)
        self.cap_bins = (comm_bins or ASYNC_COMM_BINS) if comm is not None else DENSE_MAX_BINS
        ws = ws or Workspace()
        self.ws = ws
        lib = N.lib()
        dev = ws.device
        self.stats = torch.zeros(4, dtype=torch.int64, device=dev)
        # K1 -> K2 f32 ratio keys: K2 reads 4 bytes per element, not 2L
        self.keys = torch.empty(max(self.n_local, 4), dtype=torch.float32, device=dev)
        self.counts = torch.zeros(self.cap_bins + 1, dtype=torch.int64, device=dev)
        self.centers = torch.zeros(self.k_cap, dtype=torch.float64, device=dev)
        self.cuts = torch.zeros(self.k_cap, dtype=torch.float64, device=dev)
        self.centers_t = torch.zeros(self.k_cap, dtype=dtype, device=dev)
        self.model = torch.zeros(ctypes.sizeof(N.NmkModel) // 8, dtype=torch.int64, device=dev)
        self.packed = torch.empty(self.nlb * self.stride, dtype=torch.uint8, device=dev)
        self.exact = torch.empty(max(self.n_local, 1), dtype=dtype, device=dev)
        self.prefix = torch.zeros(self.nlb, dtype=torch.int64, device=dev)
        self.n_inc = torch.zeros(1, dtype=torch.int64, device=dev)
        self.inc_offset = torch.zeros(1, dtype=torch.int64, device=dev)
        self.prefix_global = torch.zeros(self.nlb, dtype=torch.int64, device=dev)
        self.mm_bytes = lib.nmk_minmax_ws_bytes(self.n_local)
        self.mm_ws = torch.zeros(self.mm_bytes, dtype=torch.uint8, device=dev)
        self.e_bytes = lib.nmk_encode_ws_bytes(self.n_local, self.elem0, self.epb, self.dt)
        self.e_ws = torch.zeros(self.e_bytes, dtype=torch.uint8, device=dev)
        self.mode_off = lib.nmk_encode_ws_mode_offset(self.n_local, self.elem0, self.epb, self.dt)
        seg = (ctypes.c_uint64 * 1)
        self.s_start, self.s_count, self.s_out = seg(self.elem0), seg(self.n_local), seg(0)
        self.d_bytes = lib.nmk_decode_ws_bytes(self.s_start, self.s_count, 1, self.epb, self.b0)
        self.d_ws = torch.empty(self.d_bytes, dtype=torch.uint8, device=dev)
        self.seg_info = torch.zeros(2, dtype=torch.int64, device=dev)
        self.err = torch.zeros(2, dtype=torch.int64, device=dev)
        if comm is not None:
            self.gathered_inc = torch.zeros(comm.world, dtype=torch.int64, device=dev)

    def fit_comm_bins(self, nbins: int, headroom: float = 1.5, floor: int = 1024) -> int:
        """Size the all-reduced histogram to an observed dense span (e.g. the
        warm-up step's ``check()["nbins"]``) instead of ASYNC_COMM_BINS: the
        exchange then moves (cap + 1) * 8 bytes.  A later span above the cap
        is flagged on the device (NMK_ERR_NEEDS_SPARSE) and rerun through the
        general path, so the cap never changes a result.  Call before capture."""
        torch = _torch()
        cap = max(floor, 1 << max(0, math.ceil(math.log2(max(1, nbins) * headroom))))
        cap = min(cap, DENSE_MAX_BINS)
        if cap != self.cap_bins:
            self.cap_bins = cap
            self.counts = torch.zeros(cap + 1, dtype=torch.int64, device=self.counts.device)
        return cap

    # -- enqueue --------------------------------------------------------------
    def encode(self, base, cur, mark=None, recon=None):
        """Enqueue K1..K4 (+ the exchanges).  ``mark(name)`` is called after
        each phase (e.g. to record CUDA events); ``recon`` receives K4's
        reconstruction (= the decode of this encoding)."""
        lib, st = N.lib(), _stream()
        P = lambda t: t.data_ptr()  # noqa: E731
        mark = mark or (lambda name: None)
        if self.comm is None:
            # one rank: K1's last CTA decides the span and the histogram is
            # cleared inside K1 (no nmk_hist_prep launch)
            N.check(lib.nmk_minmax_prep(P(base), P(cur), self.n_local, self.dt, P(self.stats), P(self.keys),
                                        self.width, self.cap_bins, P(self.counts), P(self.mm_ws), self.mm_bytes, st))
            mark("K1_minmax")
        else:
            N.check(lib.nmk_minmax(P(base), P(cur), self.n_local, self.dt, P(self.stats), P(self.keys),
                                   P(self.mm_ws), self.mm_bytes, st))
            self.comm.allreduce_stats_device(self.stats)
            mark("K1_minmax")
            N.check(lib.nmk_hist_prep(P(self.stats), self.width, self.cap_bins, P(self.counts), st))
        N.check(lib.nmk_hist_dense_dev2(P(base), P(cur), P(self.keys), self.n_local, self.dt, P(self.stats),
                                        self.width, P(self.counts), self.span_hint, self.spread_hint, st))
        if self.comm is not None:
            self.comm.allreduce_counts(self.counts)
        mark("K2_histogram")
        N.check(lib.nmk_select(None, P(self.counts), 0, None, P(self.stats), self.width, self.tol, self.bits, self.n,
                               self.dt, P(self.centers), P(self.cuts), P(self.centers_t), self.k_cap, P(self.model),
                               st))
        mark("K3_select")
        # K4 classifies from the keys (4 bytes per element instead of 2L)
        N.check(lib.nmk_encode_keyed_dev2(P(self.keys), P(self.stats), self.width, P(base), P(cur), self.n_local,
                                          self.elem0, self.n, self.dt, P(self.centers), P(self.cuts), P(self.model),
                                          self.k_cap, self.bits, self.tol, self.epb, P(self.packed), self.stride,
                                          P(self.exact), P(self.prefix), P(self.n_inc),
                                          P(recon) if recon is not None else None, self.keyed_hint, P(self.e_ws),
                                          self.e_bytes, st))
        mark("K4_encode")
        if self.comm is not None:
            # global positions of this rank's exact values / block prefixes;
            # the local prefix stays as the decoder's rank anchor
            self.comm.exscan_device(self.n_inc, self.inc_offset, self.prefix, self.prefix_global)

    def decode(self, base, out):
        lib, st = N.lib(), _stream()
        P = lambda t: t.data_ptr()  # noqa: E731
        N.check(lib.nmk_decode_dev2(P(self.packed), self.stride, self.b0, self.bits, self.epb, self.n, P(self.prefix),
                                    P(self.centers), P(self.model), P(self.exact), P(self.n_inc), P(base), P(out),
                                    self.dt, self.s_start, self.s_count, self.s_out, 1, P(self.seg_info),
                                    P(self.err), self.ring_hint, P(self.d_ws), self.d_bytes, st))

    def step(self, base, cur, out, mark=None):
        self.encode(base, cur, mark)
        self.decode(base, out)
        if mark:
            mark("K5_decode")

    def capture(self, base, cur, out, warmup: int = 1):
        """Record step() once into a CUDA graph (buffers are fixed)."""
        torch = _torch()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(warmup):
                self.step(base, cur, out)
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.step(base, cur, out)
        return g

    # -- host view (one synchronisation) --------------------------------------
    def check(self) -> dict:
        sv = _read_struct(self.stats, N.NmkStats)
        model = _read_struct(self.model, N.NmkModel)
        e = _read_struct(self.err, N.NmkDecodeErr)
        n_inc = int(self.n_inc.item())
        trip = int(self.counts[min(int(sv.reserved), self.cap_bins)].item()) \
            if 0 < sv.reserved <= self.cap_bins else 0
        if 0 < sv.reserved <= self.cap_bins and model.status == 0:
            self.span_hint = int(sv.reserved)
            # spread field: a hot pair of bins would hold under 3/4 of the valid
            # ratios (K3 leaves the two largest selectable counts in coverage[0..1])
            top2 = int(model.coverage[0]) + int(model.coverage[1])
            self.spread_hint = int(4 * top2 < 3 * int(sv.nvalid))
        # K4's mode word: 1 = the keyed kernel applied (skip the fallback
        # launch next time), 2 = it ran on its exact path only (stale hint), 0 =
        # the snapshot-reading kernel did the work
        k4_mode = int(self.e_ws[self.mode_off:self.mode_off + 4].view(_torch().int32).item())
        self.keyed_hint = int(model.status == 0 and k4_mode == 1)
        if model.status == 0:
            self.ring_hint = int(N.lib().nmk_decode_ring_for(
                n_inc, self.n_local + self.elem0 - self.b0 * self.epb))
        return {"status": int(model.status), "bits": int(model.bits), "k": int(model.k), "n_inc": n_inc,
                "gmin": float(sv.gmin), "gmax": float(sv.gmax), "nvalid": int(sv.nvalid), "nbins": int(sv.reserved),
                "tripwire": trip, "bad_index": bool(e.bad_index), "exhausted": bool(e.exhausted), "k4_mode": k4_mode,
                "n_sentinel": int(self.seg_info[1].item())}

    def encoding(self) -> DeviceEncoding:
        """The finished encode as a DeviceEncoding (after check() passed)."""
        c = self.check()
        if c["status"] != 0:
            raise N.NativeError(c["status"], "sync-free pipeline could not complete: rerun engine.encode")
        k = c["k"]
        return DeviceEncoding(
            n=self.n, elem0=self.elem0, n_local=self.n_local, dtype=self.np_dtype, bits=self.bits, k=k,
            epb=self.epb, nblocks=self.nblocks, b0=self.b0, stride=self.stride, centers=self.centers[:k],
            centers_t=self.centers_t[:k], packed=self.packed, exact=self.exact[:c["n_inc"]], prefix=self.prefix,
            n_inc=c["n_inc"], gmin=c["gmin"], gmax=c["gmax"], nvalid=c["nvalid"], hist_form="dense",
            tol_bin=float(_read_struct(self.model, N.NmkModel).tol_bin))
