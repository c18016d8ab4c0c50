"""Compression pipeline — the reference's drop-in API on the B200.

Mirrors pkg/src/nmk/pipeline.py: same names, arguments, outputs and error
behaviour (`PipelineConfig`, `PhaseTimings`, `PipelineError`,
`compress_pair`, `decompress`, `compress_series`).  Phases 1-4a run as the
four CUDA kernels of engine.encode; phase 4b (per-block DEFLATE) stays on the
host as in the reference and is timed separately in `PhaseTimings.zlib`.
Output bytes are identical to the reference's for every input and config.
"""

from __future__ import annotations

import ctypes
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import codec, container, engine, staging
from .core import TemporalPair, Tolerance

DEFAULT_TOLERANCE = 1e-3
STRATEGIES = ("top_k", "equal_width", "log_scale", "kmeans")   # binning.py:18
MIN_BITS, MAX_BITS = 2, 30
ACCELERATED_STRATEGIES = ("top_k",)


class PipelineError(Exception):
    """Failure inside a pipeline phase; ``phase`` names where."""

    def __init__(self, phase: str, message: str):
        super().__init__(f"phase {phase}: {message}")
        self.phase = phase


@dataclass(frozen=True)
class PipelineConfig:
    """Knobs for one compression run (pipeline.py:36-58)."""

    workers: int = 1
    tolerance: float = DEFAULT_TOLERANCE
    strategy: str = "top_k"
    bits: int | None = None
    block_bytes: int = codec.DEFAULT_BLOCK_BYTES
    deflate_level: int = codec.DEFAULT_DEFLATE_LEVEL
    # lossless stage: "host" = stdlib zlib exactly as the reference (default,
    # byte-identical .nmk files); "gpu" = k_deflate.cu (valid raw DEFLATE,
    # different bytes; deflate_level is ignored)
    deflate: str = "host"

    def __post_init__(self) -> None:
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.block_bytes < codec.MIN_BLOCK_BYTES:
            raise ValueError(f"block_bytes must be >= {codec.MIN_BLOCK_BYTES}")
        if self.strategy not in STRATEGIES:
            raise ValueError(f"unknown strategy {self.strategy!r}")
        if self.bits is not None and not MIN_BITS <= self.bits <= MAX_BITS:
            raise ValueError(f"bits must be in [{MIN_BITS}, {MAX_BITS}]")
        if not 0 <= self.deflate_level <= 9:
            raise ValueError("deflate level must be in 0..9")
        if self.deflate not in ("host", "gpu"):
            raise ValueError(f"deflate must be 'host' or 'gpu', got {self.deflate!r}")
        Tolerance(self.tolerance)


@dataclass
class PhaseTimings:
    """Seconds per pipeline phase (pipeline.py:61-81).

    GPU phases are CUDA-event times: change_ratio = H2D + K1, binning = K2+K3,
    assign_index = K4 (which also performs index_alignment and bits_packing,
    fused), bits_packing = D2H of the packed stream; zlib = host DEFLATE.
    """

    change_ratio: float = 0.0
    binning: float = 0.0
    assign_index: float = 0.0
    index_alignment: float = 0.0
    bits_packing: float = 0.0
    zlib: float = 0.0
    io: float = 0.0

    PHASES = ("change_ratio", "binning", "assign_index", "index_alignment", "bits_packing", "zlib", "io")

    def total(self) -> float:
        return sum(getattr(self, p) for p in self.PHASES)

    def records(self) -> list[str]:
        return [f"timing.{p}={getattr(self, p):.6f}" for p in self.PHASES]


# ---------------------------------------------------------------------------
# host <-> device staging
# ---------------------------------------------------------------------------

_pinned: dict = {}


def _pinned_buf(key: str, nbytes: int):
    import torch
    t = _pinned.get(key)
    if t is None or t.numel() < nbytes:
        t = torch.empty(max(nbytes, 1 << 16), dtype=torch.uint8, pin_memory=True)
        _pinned[key] = t
    return t


def to_device(a: np.ndarray, key: str = "h2d"):
    """numpy -> CUDA tensor (staging.h2d: threaded fills of two pinned chunks
    overlapped with their DMA)."""
    return staging.h2d(a)


def _to_host(t, key: str) -> np.ndarray:
    """CUDA tensor -> fresh numpy array (staging.d2h)."""
    return staging.d2h(t)


def _encoding_to_host(enc: engine.DeviceEncoding):
    """Packed blocks (list of bytes), exact values, prefix, stored centers."""
    packed = _to_host(enc.packed[: enc.prefix.numel() * enc.stride], "d2h_packed")
    lens = enc.block_lengths()
    blocks = [packed[i * enc.stride: i * enc.stride + int(lens[i])].tobytes() for i in range(len(lens))]
    exact = _to_host(enc.exact, "d2h_exact").view(enc.dtype) if enc.n_inc else np.zeros(0, dtype=enc.dtype)
    prefix = enc.prefix.cpu().numpy().view(np.uint64).copy()
    centers = enc.centers_t.cpu().numpy().astype(enc.dtype, copy=False).copy()
    return blocks, exact, prefix, centers


def _deflate(blocks, config: PipelineConfig) -> list[bytes]:
    """Phase 4b, per-block raw DEFLATE on the host (pipeline.py:290-304).
    ``codec.compress_block`` is looked up at call time (monkeypatchable)."""
    fn = lambda b: codec.compress_block(b, config.deflate_level)  # noqa: E731
    try:
        if config.workers > 1 and len(blocks) > 1:
            with ThreadPoolExecutor(max_workers=config.workers) as ex:
                return list(ex.map(fn, blocks))
        return [fn(b) for b in blocks]
    except PipelineError:
        raise
    except Exception as exc:
        raise PipelineError("zlib", str(exc)) from exc


def assemble_variable(enc: engine.DeviceEncoding, config: PipelineConfig, name: str,
                      timings: PhaseTimings | None = None) -> container.CompressedVariable:
    """Device encoding -> CompressedVariable (pipeline.py:290-324)."""
    t0 = time.perf_counter()
    if getattr(config, "deflate", "host") == "gpu":   # the reference's PipelineConfig has no such field
        # the packed stream never comes to the host: only the DEFLATE output
        try:
            deflated = codec.gpu_deflate_blocks(enc.packed, enc.stride, enc.block_lengths())
        except N.NativeError as exc:
            raise PipelineError("zlib", str(exc)) from exc
        tz = time.perf_counter()
        exact = _to_host(enc.exact, "d2h_exact").view(enc.dtype) if enc.n_inc else np.zeros(0, dtype=enc.dtype)
        prefix = enc.prefix.cpu().numpy().view(np.uint64).copy()
        centers = enc.centers_t.cpu().numpy().astype(enc.dtype, copy=False).copy()
        t1 = time.perf_counter()
        zlib_s, pack_s = tz - t0, t1 - tz
    else:
        blocks, exact, prefix, centers = _encoding_to_host(enc)
        t1 = time.perf_counter()
        deflated = _deflate(blocks, config)
        pack_s, zlib_s = t1 - t0, time.perf_counter() - t1
    sizes = np.fromiter((len(b) for b in deflated), dtype=np.uint64, count=len(deflated))
    offsets = np.zeros(len(deflated), dtype=np.uint64)
    np.cumsum(sizes[:-1], out=offsets[1:])
    if timings is not None:
        timings.bits_packing += pack_s
        timings.zlib += zlib_s
    variable = container.CompressedVariable(
        name=name, dtype_code=container.dtype_code_for(enc.dtype), n=enc.n, bits=enc.bits,
        tolerance=float(config.tolerance), elements_per_block=enc.epb, nblocks=enc.nblocks,
        n_incompressible=enc.n_inc, centers=centers, index_offsets=offsets,
        incompressible_prefix=prefix, index_table=b"".join(deflated), incompressible_table=exact)
    variable.validate()
    return variable


def _check_strategy(config: PipelineConfig) -> None:
    if config.strategy not in ACCELERATED_STRATEGIES:
        raise NotImplementedError(
            f"strategy {config.strategy!r} is outside the B200 hot path (top_k binning only)")


def _encode_device(base_d, cur_d, config: PipelineConfig, timing: bool = True, recon=None):
    try:
        return engine.encode(base_d, cur_d, config.tolerance, config.bits, config.block_bytes, timing=timing,
                             recon=recon)
    except N.NativeError as exc:
        if exc.code == N.NMK_ERR_EMPTY_HIST:
            raise PipelineError("binning", "empty histogram") from exc
        raise


def compress_pair(pair: TemporalPair, config: PipelineConfig, name: str = "var0"):
    """Compress ``pair.current`` against ``pair.base`` on the GPU.

    Returns ``(CompressedVariable, PhaseTimings)``; the variable is byte-for-
    byte the reference's for the same input and config (pipeline.py:170-324).
    """
    _check_strategy(config)
    N.require_cuda()
    timings = PhaseTimings()
    t0 = time.perf_counter()
    base_d = to_device(pair.base, "h2d_base")
    cur_d = to_device(pair.current, "h2d_cur")
    h2d = time.perf_counter() - t0
    enc = _encode_device(base_d, cur_d, config)
    ms = enc.phase_ms
    timings.change_ratio = h2d + ms.get("change_ratio", 0.0) / 1e3
    timings.binning = ms.get("binning", 0.0) / 1e3
    timings.assign_index = ms.get("assign_index", 0.0) / 1e3
    variable = assemble_variable(enc, config, name, timings)
    return variable, timings


def decompress(variable: container.CompressedVariable, base_reconstructed, rng=None) -> np.ndarray:
    """Reconstruct the full variable or the slice ``rng = (start, count)``
    (pipeline.py:327-340)."""
    if rng is None:
        start, count = 0, variable.n
    else:
        start, count = rng
    base = np.asarray(base_reconstructed)
    if rng is None and base.shape[0] != variable.n:
        raise ValueError("base snapshot length mismatch")
    return codec.partial_decode(variable, start, count, base)


@dataclass
class HostEncoding:
    """Pre-deflate outputs of phases 1-4a on the host (what phase 4b and the
    container consume).  Arrays alias reusable pinned buffers: they stay valid
    until the next encode_host call."""

    n: int
    dtype: np.dtype
    bits: int
    k: int
    epb: int
    nblocks: int
    stride: int
    b0: int
    packed: np.ndarray      # u8, block b at (b - b0) * stride
    exact: np.ndarray
    prefix: np.ndarray      # u64 per local block
    centers: np.ndarray     # stored dtype
    n_inc: int

    def block(self, b: int) -> memoryview:
        ln = packed_len(self, b)
        i = b - self.b0
        return memoryview(self.packed)[i * self.stride: i * self.stride + ln]


def packed_len(h, b: int) -> int:
    cnt = min((b + 1) * h.epb, h.n) - b * h.epb
    return (cnt * h.bits + 7) // 8


def _host_tensor(a, key):
    """numpy array or CPU tensor -> pinned CPU tensor (no copy if pinned)."""
    import torch
    if isinstance(a, torch.Tensor):
        if a.is_pinned():
            return a
        a = a.numpy()
    a = np.ascontiguousarray(a)
    st = _pinned_buf(key, a.nbytes)
    st[: a.nbytes].numpy()[:] = a.view(np.uint8).reshape(-1)
    tdt = torch.float64 if a.dtype.itemsize == 8 else torch.float32
    return st[: a.nbytes].view(tdt)


def _d2h_pinned(t, key: str) -> np.ndarray:
    import torch
    nbytes = t.numel() * t.element_size()
    st = _pinned_buf(key, nbytes)
    if nbytes:
        st[:nbytes].copy_(t.reshape(-1).view(torch.uint8), non_blocking=True)
    return st[:nbytes].numpy()


def encode_host(base, current, config: PipelineConfig, *, elem0: int = 0, n_total: int | None = None,
                comm=None) -> HostEncoding:
    """Phases 1-4a from HOST buffers to HOST buffers: H2D of both snapshots,
    K1..K4, D2H of the packed stream, exact values and prefix table.  This is
    the reference-facing call the e2e benchmark times (zlib excluded)."""
    import torch
    from . import distributed
    _check_strategy(config)
    N.require_cuda()
    hb = _host_tensor(base, "e2e_base")
    hc = _host_tensor(current, "e2e_cur")
    db = hb.to("cuda", non_blocking=True)
    dc = hc.to("cuda", non_blocking=True)
    try:
        enc, _, _ = distributed.encode_shard(db, dc, elem0, n_total if n_total is not None else db.numel(),
                                             config.tolerance, config.bits, config.block_bytes, comm=comm)
    except N.NativeError as exc:
        if exc.code == N.NMK_ERR_EMPTY_HIST:
            raise PipelineError("binning", "empty histogram") from exc
        raise
    nlb = enc.prefix.numel()
    packed = _d2h_pinned(enc.packed[: nlb * enc.stride], "e2e_packed")
    exact = _d2h_pinned(enc.exact, "e2e_exact").view(enc.dtype)
    prefix = _d2h_pinned(enc.prefix, "e2e_prefix").view(np.uint64)
    centers = _d2h_pinned(enc.centers_t, "e2e_centers").view(enc.dtype)
    torch.cuda.current_stream().synchronize()
    return HostEncoding(enc.n, enc.dtype, enc.bits, enc.k, enc.epb, enc.nblocks, enc.stride, enc.b0, packed,
                        exact, prefix, centers, enc.n_inc)


def decode_host(h: HostEncoding, base, *, elem0: int = 0, count: int | None = None) -> np.ndarray:
    """Full (or [elem0, elem0+count) of this encoding's range) reconstruction
    from HOST buffers: H2D of packed stream, exact values, prefix, centers
    and base, K5, D2H of the output.  Returns a view of a pinned buffer."""
    import torch
    N.require_cuda()
    count = h.n - elem0 if count is None else count
    dev = torch.device("cuda", torch.cuda.current_device())
    d_packed = torch.from_numpy(h.packed).to(dev, non_blocking=True)
    d_exact = torch.from_numpy(h.exact).to(dev, non_blocking=True)
    d_prefix = torch.from_numpy(h.prefix.view(np.int64)).to(dev, non_blocking=True)
    d_centers = torch.from_numpy(h.centers.astype(np.float64)).to(dev, non_blocking=True)
    hb = _host_tensor(base, "e2e_dbase")
    d_base = hb.to(dev, non_blocking=True)
    res = engine.decode(d_packed, h.stride, h.b0, h.bits, h.epb, h.n, d_prefix, d_centers, d_exact, d_base,
                        [(elem0, count, 0)], check=False)
    out = _d2h_pinned(res.out, "e2e_out").view(h.dtype)
    torch.cuda.current_stream().synchronize()
    return out


class StreamCompressor:
    """Compress + reconstruct a stream of HOST timestep pairs, overlapping the
    host->device copy of step i+1 with the kernels of step i and the
    device->host copy of step i-1 (three CUDA streams, ``depth`` device slots).

    ``submit(base, cur)`` takes pinned host tensors and returns a ticket;
    ``result(ticket)`` waits and returns ``(HostEncoding, reconstruction)``,
    both views of pinned host buffers owned by the ticket's slot.  Call
    ``result(t)`` before ``submit`` reuses the slot (``depth`` submissions
    later).  The kernels are the sync-free device pipeline (explicit B); the
    exact values (alpha*n of them, unknown at enqueue time) are read back in
    ``result``."""

    def __init__(self, n: int, dtype, config: PipelineConfig, depth: int = 2, *, elem0: int = 0,
                 n_total: int | None = None, comm=None):
        """``n`` elements per step on this rank; with ``comm`` (multi-GPU) the
        rank holds [elem0, elem0+n) of an ``n_total``-element variable."""
        import torch
        _check_strategy(config)
        if config.bits is None:
            raise ValueError("StreamCompressor needs an explicit B (PipelineConfig.bits)")
        N.require_cuda()
        self.n, self.config, self.depth = int(n), config, int(depth)
        self.elem0, self.n_total, self.comm = int(elem0), (int(n_total) if n_total is not None else int(n)), comm
        self.torch_dtype = torch.float64 if np.dtype(dtype).itemsize == 8 else torch.float32
        self.np_dtype = np.dtype("<f8") if self.torch_dtype == torch.float64 else np.dtype("<f4")
        self.s_h2d, self.s_cmp, self.s_d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        self.s_x = torch.cuda.Stream()   # exact-value readback: must not queue behind the next step's D2H
        self.slots = []
        for _ in range(self.depth):
            pipe = engine.DevicePipeline(self.n, self.torch_dtype, config.tolerance, config.bits,
                                         config.block_bytes, elem0=elem0, n_total=n_total, comm=comm,
                                         ws=engine.Workspace())
            sl = {
                "pipe": pipe,
                "base": torch.empty(self.n, dtype=self.torch_dtype, device="cuda"),
                "cur": torch.empty(self.n, dtype=self.torch_dtype, device="cuda"),
                "out": torch.empty(self.n, dtype=self.torch_dtype, device="cuda"),
                "h_packed": torch.empty(pipe.packed.numel(), dtype=torch.uint8, pin_memory=True),
                "h_exact": torch.empty(max(self.n // 64, 1), dtype=self.torch_dtype, pin_memory=True),
                "h_prefix": torch.empty(pipe.prefix.numel(), dtype=torch.int64, pin_memory=True),
                # stats | model | n_inc | decode err word | segment info (inc_before, n_sentinel)
                "h_scal": torch.empty(4 + pipe.model.numel() + 1 + 2 + 2, dtype=torch.int64, pin_memory=True),
                "h_centers": torch.empty(pipe.k_cap, dtype=self.torch_dtype, pin_memory=True),
                "h_out": torch.empty(self.n, dtype=self.torch_dtype, pin_memory=True),
                "ev_in": torch.cuda.Event(), "ev_cmp": torch.cuda.Event(), "ev_out": torch.cuda.Event(),
                "busy": False,
            }
            self.slots.append(sl)
        self.count = 0

    def submit(self, base, cur) -> int:
        import torch
        t = self.count
        sl = self.slots[t % self.depth]
        if sl["busy"]:
            sl["ev_out"].synchronize()          # slot reuse: its last D2H must be done
        sl["busy"] = True
        with torch.cuda.stream(self.s_h2d):
            self.s_h2d.wait_event(sl["ev_cmp"])  # device inputs no longer read
            sl["base"].copy_(base, non_blocking=True)
            sl["cur"].copy_(cur, non_blocking=True)
            sl["ev_in"].record(self.s_h2d)
        with torch.cuda.stream(self.s_cmp):
            self.s_cmp.wait_event(sl["ev_in"])
            self.s_cmp.wait_event(sl["ev_out"])  # previous D2H of this slot's outputs
            sl["pipe"].step(sl["base"], sl["cur"], sl["out"])
            sl["ev_cmp"].record(self.s_cmp)
        with torch.cuda.stream(self.s_d2h):
            self.s_d2h.wait_event(sl["ev_cmp"])
            p = sl["pipe"]
            sl["h_packed"].copy_(p.packed, non_blocking=True)
            sl["h_prefix"].copy_(p.prefix, non_blocking=True)
            sl["h_scal"][:4].copy_(p.stats, non_blocking=True)
            sl["h_scal"][4:4 + p.model.numel()].copy_(p.model, non_blocking=True)
            m = 4 + p.model.numel()
            sl["h_scal"][m:m + 1].copy_(p.n_inc, non_blocking=True)
            sl["h_scal"][m + 1:m + 3].copy_(p.err, non_blocking=True)
            sl["h_scal"][m + 3:m + 5].copy_(p.seg_info, non_blocking=True)
            sl["h_centers"].copy_(p.centers_t, non_blocking=True)
            sl["h_out"].copy_(sl["out"], non_blocking=True)
            sl["ev_out"].record(self.s_d2h)
        self.count += 1
        return t

    def result(self, ticket: int):
        import torch
        sl = self.slots[ticket % self.depth]
        sl["ev_out"].synchronize()
        p = sl["pipe"]
        scal = sl["h_scal"].numpy()
        m = 4 + p.model.numel()
        n_inc = int(scal[m])
        if n_inc > sl["h_exact"].numel():
            sl["h_exact"] = torch.empty(n_inc, dtype=self.torch_dtype, pin_memory=True)
        if n_inc:
            with torch.cuda.stream(self.s_x):
                sl["h_exact"][:n_inc].copy_(p.exact[:n_inc], non_blocking=True)
            self.s_x.synchronize()
        self.last_d2h_bytes = (p.packed.numel() + n_inc * self.np_dtype.itemsize + p.prefix.numel() * 8
                               + sl["h_scal"].numel() * 8 + p.k_cap * self.np_dtype.itemsize
                               + self.n * self.np_dtype.itemsize)
        model = N.NmkModel.from_buffer_copy(scal[4:m].tobytes()[: ctypes.sizeof(N.NmkModel)])
        if model.status == N.NMK_ERR_NEEDS_SPARSE:
            return self._general_path(sl)
        if model.status == N.NMK_ERR_ARG:
            raise PipelineError("binning", "histogram ordinal beyond the dense span (K2 tripwire)")
        if model.status != 0:
            raise PipelineError("binning", f"sync-free pipeline status {model.status}")
        err = N.NmkDecodeErr.from_buffer_copy(scal[m + 1:m + 3].tobytes())
        n_sent = int(scal[m + 4])
        if err.bad_index or err.exhausted or n_sent != n_inc:
            raise PipelineError("assign_index", f"decode of the fresh encoding disagrees with it: bad_index="
                                f"{err.bad_index} exhausted={err.exhausted} sentinels={n_sent} n_inc={n_inc}")
        k = int(model.k)
        enc = HostEncoding(self.n, self.np_dtype, p.bits, k, p.epb, p.nblocks, p.stride, p.b0,
                           sl["h_packed"].numpy(), sl["h_exact"].numpy()[:n_inc],
                           sl["h_prefix"].numpy().view(np.uint64), sl["h_centers"].numpy()[:k], n_inc)
        return enc, sl["h_out"].numpy()

    def _general_path(self, sl):
        """A span too wide for the dense device histogram: rerun this slot's
        step (its device inputs are intact until the slot is resubmitted)
        through engine.encode's sort-based path, with K4's fused
        reconstruction standing in for the decode."""
        import torch
        p = sl["pipe"]
        with torch.cuda.stream(self.s_x):
            try:
                enc = engine.encode(sl["base"], sl["cur"], self.config.tolerance, self.config.bits,
                                    self.config.block_bytes, elem0=self.elem0, n_total=self.n_total, comm=self.comm,
                                    recon=sl["out"])
            except N.NativeError as exc:
                raise PipelineError("binning", str(exc)) from exc
            nb = enc.prefix.numel() * enc.stride
            sl["h_packed"][:nb].copy_(enc.packed[:nb], non_blocking=True)
            if enc.n_inc > sl["h_exact"].numel():
                sl["h_exact"] = torch.empty(enc.n_inc, dtype=self.torch_dtype, pin_memory=True)
            if enc.n_inc:
                sl["h_exact"][: enc.n_inc].copy_(enc.exact, non_blocking=True)
            sl["h_prefix"][: enc.prefix.numel()].copy_(enc.prefix, non_blocking=True)
            sl["h_centers"][: enc.k].copy_(enc.centers_t, non_blocking=True)
            sl["h_out"].copy_(sl["out"], non_blocking=True)
        self.s_x.synchronize()
        self.last_d2h_bytes = nb + enc.n_inc * self.np_dtype.itemsize + enc.prefix.numel() * 8 + \
            enc.k * self.np_dtype.itemsize + self.n * self.np_dtype.itemsize
        h = HostEncoding(self.n, self.np_dtype, enc.bits, enc.k, enc.epb, enc.nblocks, enc.stride, enc.b0,
                         sl["h_packed"].numpy(), sl["h_exact"].numpy()[: enc.n_inc],
                         sl["h_prefix"].numpy().view(np.uint64), sl["h_centers"].numpy()[: enc.k], enc.n_inc)
        assert p.stride == enc.stride and p.epb == enc.epb
        return h, sl["h_out"].numpy()

    def h2d_bytes(self) -> int:
        """Host->device bytes per step (both snapshots)."""
        return 2 * self.n * self.np_dtype.itemsize


class SeriesStreamCompressor:
    """compress_series for a stream of HOST snapshots where only x_t crosses
    PCIe: the base of step t is K4's fused reconstruction of step t-1, which
    never leaves HBM (pipeline.py:364-372 without the decode pass).

    ``start(x0)`` uploads the first snapshot; ``submit(x_t)`` (pinned host
    tensor) enqueues H2D of x_t, K1..K4 against the resident reconstruction,
    and D2H of the packed stream, prefix, centers and scalars, returning a
    ticket; ``result(ticket)`` returns the step's HostEncoding (views of
    pinned buffers owned by the ticket's slot, valid until ``depth`` later
    submissions).  The H2D of step t+1 overlaps the kernels of step t."""

    def __init__(self, n: int, dtype, config: PipelineConfig, depth: int = 2):
        import torch
        _check_strategy(config)
        if config.bits is None:
            raise ValueError("SeriesStreamCompressor needs an explicit B (PipelineConfig.bits)")
        N.require_cuda()
        self.n, self.config, self.depth = int(n), config, int(depth)
        self.torch_dtype = torch.float64 if np.dtype(dtype).itemsize == 8 else torch.float32
        self.np_dtype = np.dtype("<f8") if self.torch_dtype == torch.float64 else np.dtype("<f4")
        self.s_h2d, self.s_cmp, self.s_d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        self.s_x = torch.cuda.Stream()   # exact-value readback: must not queue behind the next step's D2H
        self.recon = [torch.empty(self.n, dtype=self.torch_dtype, device="cuda") for _ in range(2)]
        self.ev_recon = torch.cuda.Event()
        self.slots = []
        for _ in range(self.depth):
            pipe = engine.DevicePipeline(self.n, self.torch_dtype, config.tolerance, config.bits,
                                         config.block_bytes, ws=engine.Workspace())
            self.slots.append({
                "pipe": pipe, "cur": torch.empty(self.n, dtype=self.torch_dtype, device="cuda"),
                "h_packed": torch.empty(pipe.packed.numel(), dtype=torch.uint8, pin_memory=True),
                "h_exact": torch.empty(max(self.n // 64, 1), dtype=self.torch_dtype, pin_memory=True),
                "h_prefix": torch.empty(pipe.prefix.numel(), dtype=torch.int64, pin_memory=True),
                "h_scal": torch.empty(4 + pipe.model.numel() + 1, dtype=torch.int64, pin_memory=True),
                "h_centers": torch.empty(pipe.k_cap, dtype=self.torch_dtype, pin_memory=True),
                "ev_in": torch.cuda.Event(), "ev_cmp": torch.cuda.Event(), "ev_out": torch.cuda.Event(),
                "busy": False,
            })
        self.count = 0

    def start(self, first) -> None:
        """Begin a chain at snapshot ``first`` (collect the previous chain's
        results first).  No host synchronisation for a pinned ``first``: the
        upload is ordered behind the previous chain's kernels and in front of
        the next step's on the device."""
        import torch
        self.s_h2d.wait_stream(self.s_cmp)       # recon[0] may still be read by the last step
        with torch.cuda.stream(self.s_h2d):
            self.recon[0].copy_(torch.as_tensor(first), non_blocking=True)
        self.s_cmp.wait_stream(self.s_h2d)
        self.count = 0

    def submit(self, cur) -> int:
        import torch
        t = self.count
        sl = self.slots[t % self.depth]
        if sl["busy"]:
            sl["ev_out"].synchronize()
        sl["busy"] = True
        with torch.cuda.stream(self.s_h2d):
            self.s_h2d.wait_event(sl["ev_cmp"])
            sl["cur"].copy_(cur, non_blocking=True)
            sl["ev_in"].record(self.s_h2d)
        base, nxt = self.recon[t % 2], self.recon[(t + 1) % 2]
        with torch.cuda.stream(self.s_cmp):
            self.s_cmp.wait_event(sl["ev_in"])
            self.s_cmp.wait_event(sl["ev_out"])
            sl["pipe"].encode(base, sl["cur"], recon=nxt)
            sl["ev_cmp"].record(self.s_cmp)
        with torch.cuda.stream(self.s_d2h):
            self.s_d2h.wait_event(sl["ev_cmp"])
            p = sl["pipe"]
            m = 4 + p.model.numel()
            sl["h_packed"].copy_(p.packed, non_blocking=True)
            sl["h_prefix"].copy_(p.prefix, non_blocking=True)
            sl["h_scal"][:4].copy_(p.stats, non_blocking=True)
            sl["h_scal"][4:m].copy_(p.model, non_blocking=True)
            sl["h_scal"][m:m + 1].copy_(p.n_inc, non_blocking=True)
            sl["h_centers"].copy_(p.centers_t, non_blocking=True)
            sl["ev_out"].record(self.s_d2h)
        self.count += 1
        return t

    def result(self, ticket: int) -> HostEncoding:
        import torch
        sl = self.slots[ticket % self.depth]
        sl["ev_out"].synchronize()
        p = sl["pipe"]
        scal = sl["h_scal"].numpy()
        m = 4 + p.model.numel()
        n_inc = int(scal[m])
        model = N.NmkModel.from_buffer_copy(scal[4:m].tobytes()[: ctypes.sizeof(N.NmkModel)])
        if model.status != 0:
            raise PipelineError("binning", f"series step {ticket}: sync-free pipeline status {model.status} "
                                "(use compress_series for spans beyond the dense histogram)")
        if n_inc > sl["h_exact"].numel():
            sl["h_exact"] = torch.empty(n_inc, dtype=self.torch_dtype, pin_memory=True)
        if n_inc:
            # own stream: s_d2h already holds the next step's copies, which wait for its kernels
            with torch.cuda.stream(self.s_x):
                sl["h_exact"][:n_inc].copy_(p.exact[:n_inc], non_blocking=True)
            self.s_x.synchronize()
        self.last_d2h_bytes = (p.packed.numel() + n_inc * self.np_dtype.itemsize + p.prefix.numel() * 8
                               + sl["h_scal"].numel() * 8 + p.k_cap * self.np_dtype.itemsize)
        k = int(model.k)
        return HostEncoding(self.n, self.np_dtype, p.bits, k, p.epb, p.nblocks, p.stride, p.b0,
                            sl["h_packed"].numpy(), sl["h_exact"].numpy()[:n_inc],
                            sl["h_prefix"].numpy().view(np.uint64), sl["h_centers"].numpy()[:k], n_inc)

    def h2d_bytes(self) -> int:
        """Host->device bytes per step: the new snapshot only."""
        return self.n * self.np_dtype.itemsize


def compress_series(snapshots, config: PipelineConfig, name: str = "var0"):
    """Compress a snapshot chain (pipeline.py:343-372).

    Snapshot i is encoded against the reconstruction of snapshot i-1.  The
    reconstruction never leaves the GPU: K4 writes it while encoding (the
    decoder's arithmetic on the same codes and exact values), so
    the chain equals the reference's decompress-then-encode loop without a
    decode pass per step.
    """
    _check_strategy(config)
    snapshots = [np.ascontiguousarray(s) for s in snapshots]
    if len(snapshots) < 2:
        raise ValueError("a series needs at least two snapshots")
    n = snapshots[0].shape[0]
    for i, s in enumerate(snapshots[1:], start=1):
        if s.shape[0] != n:
            raise ValueError(f"snapshot {i} length {s.shape[0]} != {n}")
        if s.dtype != snapshots[0].dtype:
            raise ValueError(f"snapshot {i} dtype differs")
    TemporalPair(snapshots[0], snapshots[1])  # dtype / shape validation
    N.require_cuda()
    first = snapshots[0].copy()
    import torch
    recon = to_device(first, "h2d_base")
    nxt = torch.empty_like(recon)
    variables = []
    for i, snap in enumerate(snapshots[1:], start=1):
        cur = to_device(snap, "h2d_cur")
        enc = _encode_device(recon, cur, config, timing=False, recon=nxt)
        variables.append(assemble_variable(enc, config, f"{name}.{i:04d}"))
        recon, nxt = nxt, recon
    return first, variables
