"""Domain types and the numeric kernel surface (mirror of nmk.core).

Types and validation follow pkg/src/nmk/core.py:13-112 so callers and error
behaviour are unchanged; the numeric work (ratio_arrays, reconstruct) runs
on the B200 through libnmkgpu.so — there is no numpy implementation here.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N

SUPPORTED_DTYPES = {4: np.dtype("<f4"), 8: np.dtype("<f8")}


def dtype_for_width(width: int) -> np.dtype:
    """Element dtype for a byte width of 4 or 8 (core.py:16-21)."""
    try:
        return SUPPORTED_DTYPES[width]
    except KeyError:
        raise ValueError(f"unsupported element width {width}, expected 4 or 8") from None


@dataclass(frozen=True)
class Tolerance:
    """Relative error bound per element (core.py:24-34)."""

    value: float

    def __post_init__(self) -> None:
        v = float(self.value)
        if not np.isfinite(v) or v <= 0.0:
            raise ValueError(f"tolerance must be finite and > 0, got {self.value}")
        object.__setattr__(self, "value", v)


class TemporalPair:
    """Two aligned 1-D float snapshots (core.py:37-76): ``base`` is the
    earlier one, ``current`` the one being compressed."""

    __slots__ = ("base", "current")

    def __init__(self, base, current):
        base = np.ascontiguousarray(base)
        current = np.ascontiguousarray(current)
        if base.ndim != 1 or current.ndim != 1:
            raise ValueError("snapshots must be 1-D arrays")
        if base.shape != current.shape:
            raise ValueError(f"snapshot lengths differ: {base.shape[0]} vs {current.shape[0]}")
        if base.shape[0] < 1:
            raise ValueError("snapshots must hold at least one element")
        if base.dtype.itemsize not in SUPPORTED_DTYPES or base.dtype.kind != "f":
            raise ValueError(f"unsupported snapshot dtype {base.dtype}")
        if base.dtype != current.dtype:
            raise ValueError(f"snapshot dtypes differ: {base.dtype} vs {current.dtype}")
        self.base = base
        self.current = current

    @property
    def n(self) -> int:
        return self.base.shape[0]

    @property
    def width(self) -> int:
        return self.base.dtype.itemsize

    @property
    def dtype(self) -> np.dtype:
        return self.base.dtype


@dataclass
class ChangeRatioField:
    """Element-wise ratios + validity + global bounds (core.py:79-100)."""

    ratios: np.ndarray
    valid: np.ndarray
    min_ratio: float
    max_ratio: float

    @property
    def n(self) -> int:
        return self.ratios.shape[0]

    def valid_ratios(self) -> np.ndarray:
        if self.valid.all():
            return self.ratios
        return self.ratios[self.valid]


def _to_device(a: np.ndarray):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def ratio_arrays(base: np.ndarray, current: np.ndarray):
    """Eq. 1 with the zero / non-finite rules on the GPU (core.py:115-137).

    Returns host ``(ratios float64, valid bool)``."""
    import torch
    N.require_cuda()
    base = np.ascontiguousarray(base)
    current = np.ascontiguousarray(current)
    n = base.shape[0]
    if n == 0:
        return np.zeros(0), np.zeros(0, dtype=bool)
    b, c = _to_device(base), _to_device(current)
    r = torch.empty(n, dtype=torch.float64, device=b.device)
    v = torch.empty(n, dtype=torch.uint8, device=b.device)
    N.check(N.lib().nmk_ratio(b.data_ptr(), c.data_ptr(), n, N.dtype_code(base.dtype), r.data_ptr(),
                              v.data_ptr(), torch.cuda.current_stream().cuda_stream))
    return r.cpu().numpy(), v.cpu().numpy().astype(bool)


def compute_change_ratios(pair: TemporalPair) -> ChangeRatioField:
    """Ratios plus min/max over the valid ones (core.py:140-155); min/max
    come from the fused K1 kernel."""
    import torch
    from . import engine
    ratios, valid = ratio_arrays(pair.base, pair.current)
    b, c = _to_device(pair.base), _to_device(pair.current)
    ws = engine.default_workspace()
    stats = ws.typed("stats", 4, torch.int64)
    lib = N.lib()
    nb = lib.nmk_minmax_ws_bytes(pair.n)
    mm = ws.get("minmax", nb, zero=True)
    N.check(lib.nmk_minmax(b.data_ptr(), c.data_ptr(), pair.n, N.dtype_code(pair.dtype), stats.data_ptr(),
                           None, mm.data_ptr(), nb, torch.cuda.current_stream().cuda_stream))
    sv = engine._read_struct(stats, N.NmkStats)
    if sv.nvalid == 0:
        raise ValueError("no element has a well-defined change ratio")
    return ChangeRatioField(ratios=ratios, valid=valid, min_ratio=float(sv.gmin), max_ratio=float(sv.gmax))


def reconstruct(base_reconstructed, centers, indices, incompressible_values, bits: int) -> np.ndarray:
    """Inverse transform for one element range (core.py:158-208) on the GPU:
    the ids are bit-packed into one block and decoded by K5."""
    from . import codec
    base = np.asarray(base_reconstructed)
    idx = np.asarray(indices)
    if idx.shape[0] != base.shape[0]:
        raise ValueError("indices and base cover different element counts")
    sentinel = (1 << bits) - 1
    k = len(centers)
    if idx.size:
        if int(idx.min()) < 0:
            comp = idx[idx != sentinel]
            if comp.size and int(comp.max()) >= k:
                raise ValueError(f"index {int(comp.max())} out of range for {k} centers")
            raise ValueError("negative bin index")
        if int(idx.max()) > sentinel:
            comp = idx[idx != sentinel]
            raise ValueError(f"index {int(comp.max())} out of range for {k} centers")
    n_inc = int(np.count_nonzero(idx == sentinel))
    inc = np.asarray(incompressible_values)
    if base.shape[0] == 0:
        if inc.shape[0] > 0:
            raise ValueError(f"incompressible values not fully consumed: need 0, have {inc.shape[0]}")
        return np.empty(0, dtype=base.dtype)
    packed = codec.pack_block(idx, bits)
    out, need, have, bad, maxbad = codec._gpu_decode_blocks(
        [packed], bits, epb=base.shape[0], n=base.shape[0], prefix=np.zeros(1, dtype=np.uint64),
        centers64=np.asarray(centers, dtype=np.float64), exact=inc.astype(base.dtype, copy=False),
        exact_offset=0, start=0, count=base.shape[0], base=base)
    if bad:
        raise ValueError(f"index {maxbad} out of range for {k} centers")
    if inc.shape[0] < n_inc:
        raise ValueError(f"incompressible values exhausted: need {n_inc}, have {inc.shape[0]}")
    if inc.shape[0] > n_inc:
        raise ValueError(f"incompressible values not fully consumed: need {n_inc}, have {inc.shape[0]}")
    return out
