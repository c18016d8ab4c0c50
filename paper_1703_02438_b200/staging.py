"""Host <-> device staging for the reference-facing API (numpy in, numpy out).

The reference's entry points take and return pageable numpy arrays
(pipeline.py:170-340).  A pageable cudaMemcpy runs at a fraction of the PCIe
rate, and a single-threaded copy into pinned memory at ~10 GB/s, so both
directions go through two pinned chunks: several host threads fill (or
drain) one chunk while the DMA engine moves the other.  Not thread-safe (one
set of chunks per process), like the rest of the module-level workspaces."""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor, wait

import numpy as np

CHUNK_BYTES = 32 << 20
SMALL_BYTES = 16 << 20         # up to this one thread copies (<= 1.6 ms; no pool dispatch jitter on small ranges)
_WORKERS = max(1, min(8, os.cpu_count() or 1))

_executor = None
_slots = None


def _pool() -> ThreadPoolExecutor:
    global _executor
    if _executor is None:
        _executor = ThreadPoolExecutor(max_workers=_WORKERS, thread_name_prefix="nmk-stage")
    return _executor


def _chunks():
    """Two pinned chunks per device, each with the event of the last DMA that
    used it (events belong to the device they were created on)."""
    global _slots
    import torch
    if _slots is None:
        _slots = {}
    dev = torch.cuda.current_device()
    if dev not in _slots:
        sl = []
        for _ in range(2):
            t = torch.empty(CHUNK_BYTES, dtype=torch.uint8, pin_memory=True)
            sl.append({"t": t, "np": t.numpy(), "ev": torch.cuda.Event()})
        _slots[dev] = sl
    return _slots[dev]


def _par_copy(dst: np.ndarray, src: np.ndarray) -> None:
    """dst[:] = src for 1-D uint8 views, split over the host threads (numpy's
    copy releases the GIL; a fresh destination's page faults spread too)."""
    n = dst.shape[0]
    if n <= SMALL_BYTES or _WORKERS == 1:
        np.copyto(dst, src)
        return
    piece = -(-n // _WORKERS)
    piece = -(-piece // 4096) * 4096
    futs = [_pool().submit(np.copyto, dst[o:o + piece], src[o:o + piece]) for o in range(0, n, piece)]
    wait(futs)
    for f in futs:
        f.result()


def _torch_dtype(dt: np.dtype):
    import torch
    if dt.kind == "f" and dt.itemsize == 8:
        return torch.float64
    if dt.kind == "f" and dt.itemsize == 4:
        return torch.float32
    return None


def h2d(a: np.ndarray, device=None):
    """numpy array -> CUDA tensor (float32 / float64 keep their dtype, anything
    else arrives as uint8 bytes), enqueued on the current stream."""
    import torch
    a = np.ascontiguousarray(a)
    nbytes = a.nbytes
    dev = torch.empty(nbytes, dtype=torch.uint8, device=device or "cuda")
    src = a.reshape(-1).view(np.uint8)
    stream = torch.cuda.current_stream()
    for k, off in enumerate(range(0, nbytes, CHUNK_BYTES)):
        ln = min(CHUNK_BYTES, nbytes - off)
        sl = _chunks()[k % 2]
        sl["ev"].synchronize()                      # the chunk's previous DMA is done
        _par_copy(sl["np"][:ln], src[off:off + ln])
        dev[off:off + ln].copy_(sl["t"][:ln], non_blocking=True)
        sl["ev"].record(stream)
    tdt = _torch_dtype(a.dtype)
    return dev.view(tdt) if tdt is not None else dev


def d2h(t) -> np.ndarray:
    """CUDA tensor -> fresh numpy array of the same dtype (uint8 for byte
    tensors); synchronises the current stream for the chunks it reads."""
    import torch
    flat = t.reshape(-1)
    np_dt = {torch.float64: np.dtype("<f8"), torch.float32: np.dtype("<f4"), torch.int64: np.dtype("<i8"),
             torch.uint8: np.dtype("u1")}[flat.dtype]
    src = flat.view(torch.uint8)
    nbytes = src.numel()
    out = np.empty(nbytes, dtype=np.uint8)
    stream = torch.cuda.current_stream()
    pending = None
    for k, off in enumerate(range(0, nbytes, CHUNK_BYTES)):
        ln = min(CHUNK_BYTES, nbytes - off)
        sl = _chunks()[k % 2]
        sl["ev"].synchronize()                      # an earlier upload from this chunk is done
        sl["t"][:ln].copy_(src[off:off + ln], non_blocking=True)
        sl["ev"].record(stream)
        if pending is not None:                     # drain the other chunk while this DMA runs
            psl, poff, pln = pending
            psl["ev"].synchronize()
            _par_copy(out[poff:poff + pln], psl["np"][:pln])
        pending = (sl, off, ln)
    if pending is not None:
        psl, poff, pln = pending
        psl["ev"].synchronize()
        _par_copy(out[poff:poff + pln], psl["np"][:pln])
    return out.view(np_dt)
