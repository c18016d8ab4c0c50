"""The binning-level and ratio-level public API on the GPU against the oracle
(oracle/nmk_oracle.py, pinned to the reference's golden vectors):

* core.ratio_arrays / compute_change_ratios   (core.py:115-155)
* binning.histogram_of / build_histogram / merge_histograms (binning.py:102-132)
* binning.top_k_bins                           (binning.py:142-152)
* binning.select_index_length / incompressible_ratio (binning.py:165-206)
* binning.nearest_center / compressible_mask   (binning.py:287-301,350-359)

on inputs far larger than the reference's own unit tests, with the edge
values those tests plant (zeros, signed zeros, infinities, NaN, denormals,
ties on cuts).
"""

import numpy as np
import pytest

import nmk_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1703_02438_b200 as nmk  # noqa: E402
from paper_1703_02438_b200 import binning, core, workloads  # noqa: E402


def _edge_pair(n, dtype, seed):
    rng = np.random.default_rng(seed)
    base = rng.lognormal(0.0, 1.0, n)
    cur = base * (1.0 + rng.normal(0.0, 0.01, n))
    specials = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324, 1e308, -1e308, 1.0, -1.0, 2.0 ** -149])
    k = n // 50
    pos = rng.choice(n, size=2 * k, replace=False)
    base[pos[:k]] = rng.choice(specials, size=k)
    cur[pos[k:]] = rng.choice(specials, size=k)
    same = rng.choice(n, size=k, replace=False)
    cur[same] = base[same]                           # unchanged (incl. -0 bases: ratio -0.0)
    return base.astype(dtype), cur.astype(dtype)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_ratio_arrays_and_change_field(dtype):
    base, cur = _edge_pair(1_000_003, dtype, seed=1)
    r, v = core.ratio_arrays(base, cur)
    ro, vo = O.ratios_of(base, cur)
    assert r.view(np.uint64).tobytes() == ro.view(np.uint64).tobytes()
    assert np.array_equal(v, vo)
    f = core.compute_change_ratios(core.TemporalPair(base, cur))
    mm = O.minmax_of(ro, vo)
    assert (f.min_ratio, f.max_ratio) == mm
    assert f.ratios.tobytes() == ro.tobytes() and np.array_equal(f.valid, vo)


def test_compute_change_ratios_no_valid_raises():
    base = np.array([0.0, 0.0, 1.0])
    cur = np.array([1.0, np.nan, np.inf])
    with pytest.raises(ValueError):
        core.compute_change_ratios(core.TemporalPair(base, cur))


def _np_hist(r, origin, width):
    with np.errstate(all="ignore"):
        q = np.floor((r - origin) / width)
    return np.unique(q, return_counts=True)


@pytest.mark.parametrize("seed", [0, 1])
def test_histogram_of_matches_unique(seed):
    rng = np.random.default_rng(seed)
    r = np.concatenate([rng.normal(0, 0.01, 400_000), rng.uniform(-50, 50, 10_000),
                        np.array([0.0, -0.0, np.inf, -np.inf, np.nan, np.nan, 1e300, -1e300])])
    rng.shuffle(r)
    origin = -0.013     # not the minimum: negative ordinals occur
    h = binning.histogram_of(r, origin, 2e-3)
    k, c = _np_hist(r, origin, 2e-3)
    assert h.ordinals.view(np.uint64).tobytes() == k.view(np.uint64).tobytes()
    assert np.array_equal(h.counts, c)


def test_build_histogram_and_merge_match_oracle():
    base, cur = workloads.cfg5_host(1 << 20, seed=2)
    f = core.compute_change_ratios(core.TemporalPair(base, cur))
    tol = core.Tolerance(1e-4)
    h = binning.build_histogram(f, tol)
    ro, vo = O.ratios_of(base, cur)
    k, c = O.histogram(ro[vo], f.min_ratio, 2e-4)
    assert h.ordinals.tobytes() == k.tobytes() and np.array_equal(h.counts, c)
    parts = [binning.histogram_of(ch, f.min_ratio, 2e-4) for ch in np.array_split(ro[vo], 7)]
    m = binning.merge_histograms(parts)
    assert m.ordinals.tobytes() == k.tobytes() and np.array_equal(m.counts, c)


@pytest.mark.parametrize("bits", [2, 4, 8, 10, 12])
def test_top_k_and_index_length_match_oracle(bits):
    base, cur = workloads.cfg5_host(1 << 20, seed=3)
    ro, vo = O.ratios_of(base, cur)
    gmin = float(ro[vo].min())
    keys, counts = O.histogram(ro[vo], gmin, 2e-4)
    h = binning.Histogram(origin=gmin, width=2e-4, ordinals=keys, counts=counts)
    model = binning.top_k_bins(h, bits)
    want = O.top_k(keys, counts, gmin, 2e-4, bits)
    assert model.centers.tobytes() == want.tobytes()
    assert model.k == len(want) and model.tolerance.value == 1e-4
    _, cs, _ = O.selectable(keys, counts, gmin, 2e-4)
    cov = O.coverage(cs, 2, 30)
    assert binning._coverage_by_bits(h, (2, 30)) == cov
    best, sizes = binning.select_index_length(h, base.size, 8)
    assert best == O.auto_bits(cs, base.size, 8)
    assert binning.incompressible_ratio(h, base.size, bits) == (base.size - cov[bits]) / base.size


def test_top_k_ties_and_zero_count_bins():
    # ties broken toward the lower ordinal; zero-count bins stay selectable last
    h = binning.Histogram(origin=0.0, width=0.002, ordinals=np.arange(6, dtype=np.float64),
                          counts=np.array([3, 0, 3, 5, 0, 3], dtype=np.int64))
    m = binning.top_k_bins(h, 2)        # k = 3: bins 3, 0, 2
    assert np.array_equal(m.centers, h.centers_of(np.array([0.0, 2.0, 3.0])))
    m = binning.top_k_bins(h, 3)        # k = 6 > 4 nonzero: all six (zero counts included)
    assert np.array_equal(m.centers, h.centers_of(np.arange(6, dtype=np.float64)))


def test_nearest_center_and_mask_match_oracle():
    rng = np.random.default_rng(4)
    centers = np.unique(rng.normal(0, 0.02, 300))
    cuts = 0.5 * (centers[:-1] + centers[1:])
    v = np.concatenate([rng.normal(0, 0.03, 500_000), cuts, centers, np.nextafter(cuts, np.inf),
                        np.nextafter(cuts, -np.inf), [np.nan, np.inf, -np.inf, 0.0, -0.0]])
    idx, dist = binning.nearest_center(v, centers)
    wi, wd = O.nearest(v, centers)
    assert np.array_equal(idx, wi)
    assert dist.view(np.uint64).tobytes() == np.asarray(wd).view(np.uint64).tobytes()
    valid = rng.uniform(size=v.size) < 0.9
    f = core.ChangeRatioField(ratios=v, valid=valid, min_ratio=0.0, max_ratio=0.0)
    model = binning.BinModel(centers=centers, bits=10, tolerance=core.Tolerance(1e-3), strategy="top_k")
    flags, idx2 = binning.compressible_mask(f, model)
    assert np.array_equal(idx2, wi)
    assert np.array_equal(flags, valid & (np.asarray(wd) <= 1e-3))


def test_package_exports_binning_api():
    for name in ("Histogram", "BinModel", "build_histogram", "top_k_bins", "compressible_mask",
                 "select_index_length", "merge_histograms", "nearest_center"):
        assert hasattr(nmk, name)


@pytest.mark.parametrize("n", [1, 31, 32, 33, 511, 512, 4095, 4096, 4097, 100_003, 1_500_001])
@pytest.mark.parametrize("with_vals", [False, True])
def test_radix_sort64_matches_numpy(n, with_vals):
    """k_sort.cu (the sort under the sparse histogram and its merge): stable
    ascending order of 64-bit keys, values carried along, at sizes around the
    warp, warp-run and tile edges; keys with few and with many distinct values."""
    import torch
    from paper_1703_02438_b200 import _native as N
    lib = N.lib()
    rng = np.random.default_rng(n + int(with_vals))
    for kind in ("wide", "narrow", "bitpatterns"):
        if kind == "wide":
            keys = rng.integers(0, np.iinfo(np.uint64).max, n, dtype=np.uint64)
        elif kind == "narrow":
            keys = rng.integers(0, 7, n, dtype=np.uint64) << np.uint64(40)      # many equal keys: stability matters
        else:
            keys = np.abs(rng.normal(0, 1e6, n)).astype(np.float64).view(np.uint64)   # ordinal bit patterns
        vals = np.arange(n, dtype=np.uint64)
        d_k, d_v = torch.from_numpy(keys.view(np.int64)).cuda(), torch.from_numpy(vals.view(np.int64)).cuda()
        o_k, o_v = torch.empty_like(d_k), torch.empty_like(d_v)
        wsb = lib.nmk_sort64_ws_bytes(n, int(with_vals))
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
        N.check(lib.nmk_sort64(d_k.data_ptr(), o_k.data_ptr(), d_v.data_ptr() if with_vals else None,
                               o_v.data_ptr() if with_vals else None, n, ws.data_ptr(), wsb, None))
        order = np.argsort(keys, kind="stable")
        assert np.array_equal(o_k.cpu().numpy().view(np.uint64), keys[order]), kind
        assert np.array_equal(d_k.cpu().numpy().view(np.uint64), keys)          # input untouched
        if with_vals:
            assert np.array_equal(o_v.cpu().numpy().view(np.uint64), vals[order]), kind
