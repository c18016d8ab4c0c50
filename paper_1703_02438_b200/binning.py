"""Binning-level API on the B200 (mirror of the top-k part of nmk.binning,
pkg/src/nmk/binning.py).

The fused pipeline (engine.encode) never materialises these objects; this
module serves callers that hold a ratio array or a ``Histogram`` -- the
reference's binning functions and its tests -- with the same kernels:

* ``histogram_of`` / ``build_histogram``  -> ``nmk_hist_values``
  (floor((r - origin)/width), sort, run-length; binning.py:102-116)
* ``merge_histograms``                     -> ``nmk_hist_merge_values`` (binning.py:119-132)
* ``top_k_bins``                           -> K3 ``nmk_select`` (binning.py:142-152)
* ``select_index_length`` / ``incompressible_ratio``
                                            -> ``nmk_coverage`` (binning.py:165-206)
* ``nearest_center`` / ``compressible_mask`` -> ``nmk_nearest_center`` /
  ``nmk_compressible_mask`` (binning.py:287-301,350-359)

``Histogram`` and ``BinModel`` restate the reference's data types and their
validation (binning.py:27-97) so results are interchangeable with the
reference's.  The other dictionary strategies (equal-width, log-scale,
k-means) and dp_optimal_coverage are outside the accelerated path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .core import ChangeRatioField, Tolerance

STRATEGIES = ("top_k", "equal_width", "log_scale", "kmeans")
MIN_BITS = 2
MAX_BITS = 30
DEFAULT_BITS_RANGE = (2, 16)
_DENSE_CAP = 10_000_000


@dataclass
class Histogram:
    """Counts of change ratios over width-``width`` bins anchored at ``origin``;
    only nonempty bins are stored, ``ordinals`` as integer-valued float64
    (binning.py:27-62)."""

    origin: float
    width: float
    ordinals: np.ndarray
    counts: np.ndarray

    @property
    def total(self) -> int:
        return int(self.counts.sum())

    @property
    def nonempty(self) -> int:
        return len(self.ordinals)

    def centers_of(self, ordinals: np.ndarray) -> np.ndarray:
        return self.origin + (ordinals + 0.5) * self.width

    def dense_counts(self) -> np.ndarray:
        if self.nonempty == 0:
            return np.zeros(0, dtype=np.int64)
        last = self.ordinals[-1]
        if not np.isfinite(last) or last + 1 > _DENSE_CAP:
            raise ValueError("histogram spans too many bins to densify")
        dense = np.zeros(int(last) + 1, dtype=np.int64)
        dense[self.ordinals.astype(np.int64)] = self.counts
        return dense


@dataclass
class BinModel:
    """Selected centers + index length + tolerance (binning.py:65-97)."""

    centers: np.ndarray
    bits: int
    tolerance: Tolerance
    strategy: str

    def __post_init__(self) -> None:
        self.centers = np.asarray(self.centers, dtype=np.float64)
        if self.strategy not in STRATEGIES:
            raise ValueError(f"unknown strategy {self.strategy!r}")
        if not MIN_BITS <= self.bits <= MAX_BITS:
            raise ValueError(f"index length {self.bits} outside [{MIN_BITS}, {MAX_BITS}]")
        k = len(self.centers)
        if k < 1:
            raise ValueError("a bin model needs at least one center")
        if k > (1 << self.bits) - 1:
            raise ValueError(f"{k} centers exceed the {(1 << self.bits) - 1} usable ids at B={self.bits}")
        if k > 1 and not (np.diff(self.centers) > 0).all():
            raise ValueError("centers must be strictly increasing")

    @property
    def k(self) -> int:
        return len(self.centers)

    @property
    def sentinel(self) -> int:
        return (1 << self.bits) - 1


# ---------------------------------------------------------------------------
# device helpers
# ---------------------------------------------------------------------------

def _stream() -> int:
    import torch
    return torch.cuda.current_stream().cuda_stream


def _dev(a: np.ndarray, dtype):
    import torch
    a = np.ascontiguousarray(a, dtype=dtype)
    return torch.from_numpy(a.copy() if not a.flags.writeable else a).cuda()


def _stats_tensor(origin: float, nvalid: int):
    """An nmk_stats record on the device: gmin = origin (K3's center origin)."""
    import torch
    rec = np.zeros(4, dtype=np.int64)
    rec[0] = np.float64(origin).view(np.int64)
    rec[1] = np.float64(origin).view(np.int64)
    rec[2] = nvalid
    return torch.from_numpy(rec).cuda()


def _read(t, dtype) -> np.ndarray:
    return t.cpu().numpy().view(dtype)


# ---------------------------------------------------------------------------
# histograms (binning.py:102-132)
# ---------------------------------------------------------------------------

def _histogram_device(ratios: np.ndarray, valid, origin: float, width: float) -> Histogram:
    import torch
    torch_ = N.require_cuda()
    r = np.asarray(ratios, dtype=np.float64)
    n = r.shape[0]
    if n == 0:
        return Histogram(origin=origin, width=width, ordinals=np.zeros(0), counts=np.zeros(0, dtype=np.int64))
    lib = N.lib()
    d_r = _dev(r, np.float64)
    d_v = _dev(np.asarray(valid, dtype=np.uint8), np.uint8) if valid is not None else None
    ords = torch_.empty(n, dtype=torch.float64, device="cuda")
    cnts = torch_.empty(n, dtype=torch.int64, device="cuda")
    nruns = torch_.zeros(1, dtype=torch.int64, device="cuda")
    wsb = lib.nmk_hist_values_ws_bytes(n)
    ws = torch_.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
    N.check(lib.nmk_hist_values(d_r.data_ptr(), d_v.data_ptr() if d_v is not None else None, n, float(origin),
                                float(width), ords.data_ptr(), cnts.data_ptr(), nruns.data_ptr(), ws.data_ptr(), wsb,
                                _stream()))
    m = int(nruns.item())
    return Histogram(origin=origin, width=width, ordinals=ords[:m].cpu().numpy(),
                     counts=cnts[:m].cpu().numpy().astype(np.int64))


def histogram_of(ratios: np.ndarray, origin: float, width: float) -> Histogram:
    """Histogram of a raw ratio slice against a fixed origin/width grid
    (binning.py:110-116) on the GPU: ordinal per element, radix sort,
    run-length.  Negative, infinite and NaN ordinals follow np.unique."""
    return _histogram_device(ratios, None, origin, width)


def build_histogram(field: ChangeRatioField, tolerance: Tolerance) -> Histogram:
    """Histogram of the valid ratios in bins of width 2E anchored at the
    minimum (binning.py:102-107); the validity mask is applied on the device."""
    valid = np.asarray(field.valid, dtype=bool)
    if field.ratios.shape[0] == 0 or not valid.any():
        raise ValueError("no valid change ratios to histogram")
    return _histogram_device(field.ratios, None if valid.all() else valid, field.min_ratio,
                             2.0 * tolerance.value)


def merge_histograms(parts: list) -> Histogram:
    """Element-wise sum of per-shard histograms (binning.py:119-132): the
    gathered (ordinal, count) pairs are sorted and summed on the device."""
    import torch
    if not parts:
        raise ValueError("nothing to merge")
    first = parts[0]
    if len(parts) == 1:
        return first
    torch_ = N.require_cuda()
    ords = np.concatenate([np.asarray(p.ordinals, dtype=np.float64) for p in parts])
    cnts = np.concatenate([np.asarray(p.counts, dtype=np.int64) for p in parts])
    n = ords.shape[0]
    if n == 0:
        return Histogram(origin=first.origin, width=first.width, ordinals=np.zeros(0),
                         counts=np.zeros(0, dtype=np.int64))
    lib = N.lib()
    d_o = _dev(ords, np.float64)
    d_c = _dev(cnts, np.int64)
    nruns = torch_.zeros(1, dtype=torch.int64, device="cuda")
    wsb = lib.nmk_hist_merge_ws_bytes(n)
    ws = torch_.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
    N.check(lib.nmk_hist_merge_values(d_o.data_ptr(), d_c.data_ptr(), n, nruns.data_ptr(), ws.data_ptr(), wsb,
                                      _stream()))
    m = int(nruns.item())
    return Histogram(origin=first.origin, width=first.width, ordinals=d_o[:m].cpu().numpy(),
                     counts=d_c[:m].cpu().numpy().astype(np.int64))


# ---------------------------------------------------------------------------
# selection (binning.py:135-206)
# ---------------------------------------------------------------------------

def top_k_bins(hist, bits: int) -> BinModel:
    """The most populous bins, ties toward the lower ordinal (binning.py:142-152),
    selected by K3's radix select over the sparse histogram.

    K3 treats a zero count as an empty bin; the reference's ``_selectable``
    keeps zero-count bins with a finite center (a hand-built Histogram may
    hold them).  Every count is therefore passed as count + 1, which keeps
    the (count desc, ordinal asc) order and makes those bins selectable last,
    exactly as lexsort ranks them."""
    import torch
    if not MIN_BITS <= bits <= MAX_BITS:
        raise ValueError(f"index length {bits} outside [{MIN_BITS}, {MAX_BITS}]")
    torch_ = N.require_cuda()
    ords = np.ascontiguousarray(hist.ordinals, dtype=np.float64)
    m = ords.shape[0]
    if m == 0:
        raise ValueError("empty histogram")
    lib = N.lib()
    keys = _dev(ords, np.float64).view(torch.int64)
    counts = _dev(np.asarray(hist.counts, dtype=np.int64) + 1, np.int64)
    nruns = torch_.tensor([m], dtype=torch.int64, device="cuda")
    stats = _stats_tensor(hist.origin, 1)
    cap_k = max(1, min((1 << bits) - 1, m))
    centers = torch_.empty(cap_k, dtype=torch.float64, device="cuda")
    cuts = torch_.empty(cap_k, dtype=torch.float64, device="cuda")
    centers_t = torch_.empty(cap_k, dtype=torch.float64, device="cuda")
    model_t = torch_.zeros(ctypes.sizeof(N.NmkModel) // 8, dtype=torch.int64, device="cuda")
    width = float(hist.width)
    N.check(lib.nmk_select(keys.data_ptr(), counts.data_ptr(), m, nruns.data_ptr(), stats.data_ptr(), width,
                           width / 2.0, int(bits), 0, N.NMK_F64, centers.data_ptr(), cuts.data_ptr(),
                           centers_t.data_ptr(), cap_k, model_t.data_ptr(), _stream()))
    model = N.NmkModel.from_buffer_copy(model_t.cpu().numpy().tobytes()[: ctypes.sizeof(N.NmkModel)])
    if model.status == N.NMK_ERR_EMPTY_HIST:
        raise ValueError("empty histogram")
    if model.status != 0:
        raise N.NativeError(model.status, "nmk_select failed")
    chosen = centers[: int(model.k)].cpu().numpy()
    return BinModel(centers=chosen, bits=bits, tolerance=Tolerance(hist.width / 2.0), strategy="top_k")


def estimate_file_size(n: int, width: int, bits: int, n_incompressible: int) -> float:
    """Modeled compressed size in bytes (binning.py:155-162, Eq. 6)."""
    return (1 << bits) * width + (n * bits) / 8 + n_incompressible * width


def _coverage_by_bits(hist, bits_range) -> dict[int, int]:
    """Elements covered by the top 2^B - 1 selectable bins per B
    (binning.py:165-174), from K3's multi-slot radix select."""
    import torch
    lo, hi = int(bits_range[0]), int(bits_range[1])
    ords = np.ascontiguousarray(hist.ordinals, dtype=np.float64)
    m = ords.shape[0]
    if m == 0:
        return {b: 0 for b in range(lo, hi + 1)}
    torch_ = N.require_cuda()
    lib = N.lib()
    keys = _dev(ords, np.float64).view(torch.int64)
    counts = _dev(np.asarray(hist.counts, dtype=np.int64), np.int64)
    nruns = torch_.tensor([m], dtype=torch.int64, device="cuda")
    stats = _stats_tensor(hist.origin, 1)
    cov = torch_.zeros(hi - lo + 1, dtype=torch.int64, device="cuda")
    model_t = torch_.zeros(ctypes.sizeof(N.NmkModel) // 8, dtype=torch.int64, device="cuda")
    N.check(lib.nmk_coverage(keys.data_ptr(), counts.data_ptr(), m, nruns.data_ptr(), stats.data_ptr(),
                             float(hist.width), lo, hi, cov.data_ptr(), model_t.data_ptr(), _stream()))
    c = cov.cpu().numpy()
    return {lo + i: int(c[i]) for i in range(hi - lo + 1)}


def incompressible_ratio(hist, n: int, bits: int) -> float:
    """Fraction of the n elements outside the top 2^bits - 1 bins (binning.py:177-180)."""
    covered = _coverage_by_bits(hist, (bits, bits))[bits]
    return (n - covered) / n


def select_index_length(hist, n: int, width: int, bits_range: tuple[int, int] = DEFAULT_BITS_RANGE):
    """Index length minimising the modeled file size, ties to the smaller B
    (binning.py:182-206); the coverage table comes from the device."""
    lo, hi = bits_range
    if lo < MIN_BITS or hi > MAX_BITS or lo > hi:
        raise ValueError(f"bits range {bits_range} outside [{MIN_BITS}, {MAX_BITS}]")
    coverage = _coverage_by_bits(hist, bits_range)
    sizes: dict[int, float] = {}
    best_bits, best_size = lo, None
    for bits in range(lo, hi + 1):
        size = estimate_file_size(n, width, bits, n - coverage[bits])
        sizes[bits] = size
        if best_size is None or size < best_size:
            best_size, best_bits = size, bits
    return best_bits, sizes


# ---------------------------------------------------------------------------
# classification (binning.py:287-301,350-359)
# ---------------------------------------------------------------------------

def nearest_center(values: np.ndarray, centers: np.ndarray):
    """Nearest center by the midpoint cuts, ties to the lower index
    (binning.py:287-301), on the GPU.  Returns ``(indices, distances)``."""
    import torch
    v = np.asarray(values, dtype=np.float64)
    c = np.asarray(centers, dtype=np.float64)
    n = v.shape[0]
    if n == 0:
        return np.zeros(0, dtype=np.int64), np.zeros(0, dtype=np.float64)
    torch_ = N.require_cuda()
    d_v, d_c = _dev(v, np.float64), _dev(c, np.float64)
    idx = torch_.empty(n, dtype=torch.int64, device="cuda")
    dist = torch_.empty(n, dtype=torch.float64, device="cuda")
    N.check(N.lib().nmk_nearest_center(d_v.data_ptr(), n, d_c.data_ptr(), len(c), idx.data_ptr(), dist.data_ptr(),
                                       _stream()))
    return idx.cpu().numpy(), dist.cpu().numpy()


def compressible_mask(field: ChangeRatioField, model):
    """Per-element compressibility flags and nearest-center indices
    (binning.py:350-359), on the GPU."""
    import torch
    r = np.asarray(field.ratios, dtype=np.float64)
    n = r.shape[0]
    if n == 0:
        return np.zeros(0, dtype=bool), np.zeros(0, dtype=np.int64)
    torch_ = N.require_cuda()
    c = np.asarray(model.centers, dtype=np.float64)
    d_r, d_c = _dev(r, np.float64), _dev(c, np.float64)
    d_v = _dev(np.asarray(field.valid, dtype=np.uint8), np.uint8)
    flags = torch_.empty(n, dtype=torch.uint8, device="cuda")
    idx = torch_.empty(n, dtype=torch.int64, device="cuda")
    N.check(N.lib().nmk_compressible_mask(d_r.data_ptr(), d_v.data_ptr(), n, d_c.data_ptr(), len(c),
                                          float(model.tolerance.value), flags.data_ptr(), idx.data_ptr(),
                                          _stream()))
    return flags.cpu().numpy().astype(bool), idx.cpu().numpy()
