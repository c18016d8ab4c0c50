"""K4's keyed mode (classification from K1's f32 ratio keys, k_encode.cuh
setup_keyed / classify_key) must give the exact path's bits: ratios planted
at cuts, at c +- E and at bin edges, f32 round-trip rejections, magnitudes
at the edges of the keys' safe range, and the keyed/unkeyed engines
compared byte for byte (packed stream, exact values, prefix, recon)."""

import numpy as np
import pytest

import nmk_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1703_02438_b200 import _native as N, engine  # noqa: E402


def _blocks(enc):
    nlb = enc.prefix.numel()
    packed = enc.packed[: nlb * enc.stride].cpu().numpy()
    lens = enc.block_lengths()
    return [packed[i * enc.stride: i * enc.stride + int(lens[i])].tobytes() for i in range(nlb)]


def _run_all(b, c, E, bits, bb=1 << 16):
    """oracle vs engine(keyed) vs engine(unkeyed) vs DevicePipeline (keyed)."""
    o = O.encode(b, c, E, bits, bb)
    dec = O.decode(o, b).tobytes()
    base, cur = torch.from_numpy(b).cuda(), torch.from_numpy(c).cuda()
    outs = []
    for keyed in (True, False):
        rec = torch.full_like(cur, float("nan"))
        enc = engine.encode(base, cur, E, bits, bb, recon=rec, keyed=keyed, ws=engine.Workspace())
        assert enc.n_inc == o["n_inc"]
        assert _blocks(enc) == o["blocks"], f"packed stream differs (keyed={keyed})"
        assert enc.exact.cpu().numpy().tobytes() == o["exact"].tobytes()
        assert enc.prefix.cpu().numpy().astype(np.uint64).tobytes() == o["prefix"].astype(np.uint64).tobytes()
        assert rec.cpu().numpy().tobytes() == dec, f"fused reconstruction differs (keyed={keyed})"
        outs.append(enc)
    if bits is not None:
        pipe = engine.DevicePipeline(base.numel(), base.dtype, E, bits, bb)
        out = torch.empty_like(base)
        pipe.step(base, cur, out)
        chk = pipe.check()
        if chk["status"] == 0:
            enc = pipe.encoding()
            assert _blocks(enc) == o["blocks"]
            assert enc.exact.cpu().numpy().tobytes() == o["exact"].tobytes()
            assert out.cpu().numpy().tobytes() == dec
            rec = torch.full_like(cur, float("nan"))
            pipe.encode(base, cur, recon=rec)
            assert rec.cpu().numpy().tobytes() == dec
    return o


def _plant(rng, targets, n, dtype, lo=0.5, hi=2.0):
    t = rng.choice(targets, n)
    t = t + np.spacing(np.abs(t) + 1e-300) * rng.integers(-8, 9, n)
    b = rng.uniform(lo, hi, n) * np.where(rng.uniform(size=n) < 0.3, -1.0, 1.0)
    return b.astype(dtype), (b * (1.0 + t)).astype(dtype)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("E,shift", [(1e-3, 0.0), (1e-4, 0.0), (2e-4, 1.5), (1e-5, -0.3)])
def test_keyed_cuts_tolerance_and_bin_edges(dtype, E, shift):
    rng = np.random.default_rng(41)
    n = 150_000
    b = rng.lognormal(0.0, 1.0, n)
    c = b * (1.0 + shift + np.where(rng.uniform(size=n) < 0.8, rng.normal(0, 4 * E, n),
                                    rng.uniform(-60 * E, 60 * E, n)))
    b, c = b.astype(dtype), c.astype(dtype)
    o = O.encode(b, c, E, 8, 1 << 16)
    cen = o["centers"].astype(np.float64)
    r, v = O.ratios_of(b, c)
    gmin = float(r[v].min())
    edges = gmin + np.arange(1, 200) * (2 * E)
    targets = np.concatenate([0.5 * (cen[:-1] + cen[1:]), cen + E, cen - E, cen + E * (1 - 1e-9),
                              cen - E * (1 + 1e-9), cen + E * (1 - 3e-8), edges])
    pb, px = _plant(rng, targets, n, dtype)
    _run_all(np.concatenate([b, pb]), np.concatenate([c, px]), E, 8)


@pytest.mark.parametrize("scale", [1.0, 1e3, 3e5])
def test_keyed_f32_roundtrip_rejections(scale):
    """f32 values where T((1+c)b) misses by a rounding: the filter must reject
    exactly the oracle's elements (pipeline.py:143-160)."""
    rng = np.random.default_rng(42)
    n = 200_000
    E = 2e-6
    b = (rng.uniform(0.5, 2.0, n) * scale).astype(np.float32)
    c = (b.astype(np.float64) * (1.0 + rng.normal(0, 3 * E, n))).astype(np.float32)
    o = _run_all(b, c, E, 10, 1 << 15)
    assert o["n_inc"] > 0


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_keyed_safe_range_edges(dtype):
    """Bases and currents straddling the keys' safe range (2^-900..2^901 for
    f64, 2^-100..2^101 for f32) and b = x = 0 pairs."""
    rng = np.random.default_rng(43)
    lo, hi = (-900, 901) if dtype == np.float64 else (-100, 101)
    n = 60_000
    e = rng.choice(np.r_[lo - 3:lo + 4, hi - 4:hi + 3, -2:3], n)
    b = np.ldexp(rng.uniform(1.0, 2.0, n), e) * np.where(rng.uniform(size=n) < 0.5, -1, 1)
    c = b * (1.0 + np.where(rng.uniform(size=n) < 0.5, rng.normal(0, 0.002, n), rng.uniform(-0.04, 0.04, n)))
    z = rng.uniform(size=n) < 0.01
    b[z] = 0.0
    c[z] = 0.0
    with np.errstate(over="ignore"):
        b, c = b.astype(dtype), c.astype(dtype)
    _run_all(b, c, 1e-3, 8, 1 << 14)


def test_keyed_all_invalid_and_tiny():
    rng = np.random.default_rng(44)
    b = np.zeros(5000)
    c = rng.uniform(1, 2, 5000)
    _run_all(b, c, 1e-3, 4, 4096)            # no valid ratio: degenerate model
    for n in (1, 7, 300, 1025):
        b = rng.lognormal(0, 1, n)
        c = b * (1 + rng.normal(0, 0.002, n))
        _run_all(b, c, 1e-3, 8, 4096)


def _dense_counts(pipe, nbins):
    return pipe.counts[: nbins + 1].cpu().numpy()


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("E,shift,sigma", [(1e-3, 0.0, 3e-4), (1e-3, 2e-4, 2e-4), (1e-4, 0.0, 1e-4),
                                           (5e-3, 0.7, 1e-3)])
def test_keyed_histogram_hot_bins_exact(dtype, E, shift, sigma):
    """K2's hot-bin f32 test (k_hist.cu hot_params) against the oracle's
    np.unique histogram: a dominant narrow bin whose edge sits near the bulk
    of the ratios, planted ratios within a few ulps of its edges, outliers."""
    rng = np.random.default_rng(45)
    n = 400_000
    b = rng.uniform(0.5, 2.0, n) * np.where(rng.uniform(size=n) < 0.3, -1.0, 1.0)
    r = shift + rng.normal(0, sigma, n)
    out = rng.uniform(size=n) < 0.03
    r[out] = rng.laplace(0, 0.1, out.sum())
    c = b * (1.0 + r)
    b, c = b.astype(dtype), c.astype(dtype)
    rr, v = O.ratios_of(b, c)
    gmin = float(rr[v].min())
    e0 = gmin + np.floor((shift - gmin) / (2 * E)) * (2 * E)      # edges around the bulk
    edges = e0 + np.arange(-3, 4) * (2 * E)
    pb, px = _plant(rng, edges, 100_000, dtype)
    base = np.concatenate([b, pb]).astype(dtype)
    cur = np.concatenate([c, px]).astype(dtype)
    bt, ct = torch.from_numpy(base).cuda(), torch.from_numpy(cur).cuda()
    pipe = engine.DevicePipeline(bt.numel(), bt.dtype, E, 10, 1 << 16)
    out_t = torch.empty_like(bt)
    pipe.step(bt, ct, out_t)
    chk = pipe.check()
    assert chk["status"] == 0 and chk["tripwire"] == 0
    rr, v = O.ratios_of(base, cur)
    keys, counts = O.histogram(rr[v], chk["gmin"], 2 * E)
    dense = np.zeros(chk["nbins"], dtype=np.int64)
    dense[keys.astype(np.int64)] = counts
    got = _dense_counts(pipe, chk["nbins"])
    np.testing.assert_array_equal(got[: chk["nbins"]], dense)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("bits", [12, 13, 11])
def test_keyed_misaligned_blocks(dtype, bits):
    """Index blocks of epb % 4 != 0 elements (B = 12: 43690 per 64 KiB block,
    B = 13 / 11: odd epb) start keys at every shift mod 4: the keyed kernel's
    shifted pair copies and the unaligned single chunks must match the oracle."""
    rng = np.random.default_rng(46 + bits)
    n = 700_001
    b = rng.lognormal(0.0, 1.0, n)
    c = b * (1.0 + np.where(rng.uniform(size=n) < 0.9, rng.normal(0, 0.002, n), rng.uniform(-0.05, 0.05, n)))
    b[rng.uniform(size=n) < 0.003] = 0.0
    _run_all(b.astype(dtype), c.astype(dtype), 1e-3, bits)


def test_keyed_wide_table_u16():
    """B <= 15 keeps a u16 ordinal table of 16384 rows: selected centers
    spread over more than 8192 histogram bins (uniform ratios over ~12000
    bins, B = 12 takes the 4095 fullest) must still take the keyed path and
    match the oracle."""
    rng = np.random.default_rng(47)
    n = 600_000
    E = 5e-5
    b = rng.uniform(0.5, 2.0, n)
    c = b * (1.0 + rng.uniform(-0.6, 0.6, n))
    o = _run_all(b, c, E, 12)
    cen = o["centers"]
    assert (cen[-1] - cen[0]) / (2 * E) > 8192   # the table really is wider than the u32 one


def _f32_boundary_pair(rng, n):
    """f32 pairs around K1's f32 fast path edges (k_ratio.cu mm_visit32):
    |d| near |b| / 4, |b| near 2^-60 and 2^60, x == b, sign flips, zeros,
    ratios that straddle the running extremes."""
    mag = np.exp2(rng.uniform(-64.0, 64.0, n))
    edge = rng.choice([2.0 ** -60, 2.0 ** 60, 1.0], n) * (1.0 + rng.integers(-3, 4, n) * 2.0 ** -23)
    b = np.where(rng.uniform(size=n) < 0.3, edge, mag) * np.where(rng.uniform(size=n) < 0.4, -1.0, 1.0)
    b = b.astype(np.float32)
    r = rng.choice([0.25, -0.25, 0.0, 1e-3, -1e-3, 0.7, -0.9, 3.0], n)
    r = r + rng.integers(-4, 5, n) * 2.0 ** -24
    x = (b.astype(np.float64) * (1.0 + r)).astype(np.float32)
    x[rng.uniform(size=n) < 0.01] = 0.0
    b[rng.uniform(size=n) < 0.005] = 0.0
    return b, x


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_f32_keys_contract_and_extremes(seed):
    """K1's f32 keys satisfy |key - r| <= |key| 2^-23 (r the reference's f64
    ratio, core.py:126-136); invalid elements get NaN, keys outside the safe
    range +inf; gmin / gmax / nvalid equal numpy's exactly."""
    from paper_1703_02438_b200 import _native as N
    rng = np.random.default_rng(seed)
    n = (1 << 18) + 37
    b, x = _f32_boundary_pair(rng, n)
    base, cur = torch.from_numpy(b).cuda(), torch.from_numpy(x).cuda()
    lib = N.lib()
    stats = torch.zeros(4, dtype=torch.int64, device="cuda")
    keys = torch.empty(n + 4, dtype=torch.float32, device="cuda")
    wsb = lib.nmk_minmax_ws_bytes(n)
    ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda")
    N.check(lib.nmk_minmax(base.data_ptr(), cur.data_ptr(), n, N.NMK_F32, stats.data_ptr(), keys.data_ptr(),
                           ws.data_ptr(), wsb, torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    bd, xd = b.astype(np.float64), x.astype(np.float64)
    with np.errstate(all="ignore"):
        r = (xd - bd) / bd
    valid = np.isfinite(r) & np.isfinite(bd) & np.isfinite(xd)
    both0 = (bd == 0) & (xd == 0)
    r[both0] = 0.0
    valid |= both0
    st = stats.cpu().numpy()
    assert st[2] == valid.sum()
    assert np.float64(st[0:1].view(np.float64)[0]) == r[valid].min()
    assert np.float64(st[1:2].view(np.float64)[0]) == r[valid].max()
    k = keys[:n].cpu().numpy().astype(np.float64)
    assert np.isnan(k[~valid]).all()
    fin = valid & np.isfinite(k)
    assert np.all(np.abs(k[fin] - r[fin]) <= np.abs(k[fin]) * 2.0 ** -23)
    assert np.all(np.isposinf(k[valid & ~np.isfinite(k)]))
    # most elements with |r| < 1/4 and moderate |b| take the f32 fast path and
    # must carry a finite key
    mid = valid & (np.abs(r) < 0.2) & (np.abs(bd) > 2.0 ** -50) & (np.abs(bd) < 2.0 ** 50)
    assert np.isfinite(k[mid]).all()


@pytest.mark.parametrize("bits", [8, 10])
def test_f32_boundary_pairs_bit_exact(bits):
    rng = np.random.default_rng(11 + bits)
    b, x = _f32_boundary_pair(rng, (1 << 16) + 5)
    _run_all(b, x, 1e-3, bits)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("E,kind", [(1e-3, "bimodal"), (1e-2, "bimodal"), (2e-3, "uniform"), (1e-3, "narrow")])
def test_histogram_forms_exact(dtype, E, kind):
    """All three forms of K2's key histogram against np.unique at sizes where
    every warp runs several tiles: lane-private counters (span <= 63 bins:
    "narrow"), the hot pair, and the out-of-line direct tiles a spread field
    switches to (cfg5's bimodal mixture, uniform ratios over ~10^3 bins)."""
    rng = np.random.default_rng(7)
    n = (1 << 23) + 1234
    b = rng.lognormal(0.0, 1.0, n)
    if kind == "bimodal":
        m = rng.uniform(size=n)
        r = np.where(m < 0.4, rng.normal(-0.02, 0.004, n), rng.normal(0.03, 0.006, n))
        out = m > 0.8
        r[out] = rng.uniform(-1.0, 1.0, out.sum())
    elif kind == "uniform":
        r = rng.uniform(-1.0, 1.0, n)
    else:
        r = rng.normal(0.0, 0.008, n)
    c = b * (1.0 + r)
    b[rng.uniform(size=n) < 0.003] = 0.0
    b, c = b.astype(dtype), c.astype(dtype)
    bt, ct = torch.from_numpy(b).cuda(), torch.from_numpy(c).cuda()
    pipe = engine.DevicePipeline(bt.numel(), bt.dtype, E, 8)
    out_t = torch.empty_like(bt)
    pipe.step(bt, ct, out_t)
    chk = pipe.check()
    assert chk["status"] == 0 and chk["tripwire"] == 0
    rr, v = O.ratios_of(b, c)
    keys, counts = O.histogram(rr[v], chk["gmin"], 2 * E)
    dense = np.zeros(chk["nbins"], dtype=np.int64)
    dense[keys.astype(np.int64)] = counts
    got = _dense_counts(pipe, chk["nbins"])
    np.testing.assert_array_equal(got[: chk["nbins"]], dense)
    if kind == "narrow":
        assert chk["nbins"] <= 63


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("E,kind", [(1e-4, "bimodal"), (1e-3, "bimodal"), (1e-2, "bimodal"), (1e-3, "narrow"),
                                    (2e-5, "uniform"), (1e-3, "concentrated")])
@pytest.mark.parametrize("span_hint,spread_hint", [(0, 0), (1116, 1), (10000, 1), (20000, 0), (3, 1)])
def test_histogram_launch_shapes_exact(dtype, E, kind, span_hint, spread_hint):
    """K2's launch shapes (hot-pair / spread replicas / wide 1024-thread
    replicas) and counting policies, chosen by the previous step's span and
    spread hints, give the same exact counts whatever the hint -- including
    hints that do not match the data (a stale hint costs speed only).
    Spans: bimodal at E = 1e-4 -> 10^4 bins (the wide shape), uniform at
    E = 2e-5 -> 5*10^4 bins (beyond every replica: the global fallback)."""
    rng = np.random.default_rng(11)
    n = (1 << 22) + 4321
    b = rng.lognormal(0.0, 1.0, n)
    if kind == "bimodal":
        m = rng.uniform(size=n)
        r = np.where(m < 0.4, rng.normal(-0.02, 0.004, n), rng.normal(0.03, 0.006, n))
        out = m > 0.8
        r[out] = rng.uniform(-1.0, 1.0, out.sum())
    elif kind == "uniform":
        r = rng.uniform(-1.0, 1.0, n)
    elif kind == "concentrated":
        r = np.where(rng.uniform(size=n) < 0.95, rng.normal(0.0, 1e-4, n), rng.normal(0.0, 0.05, n))
    else:
        r = rng.normal(0.0, 0.008, n)
    c = b * (1.0 + r)
    b, c = b.astype(dtype), c.astype(dtype)
    bt, ct = torch.from_numpy(b).cuda(), torch.from_numpy(c).cuda()
    pipe = engine.DevicePipeline(bt.numel(), bt.dtype, E, 8)
    pipe.span_hint, pipe.spread_hint = span_hint, spread_hint
    out_t = torch.empty_like(bt)
    pipe.encode(bt, ct)
    torch.cuda.synchronize()
    sv = engine._read_struct(pipe.stats, N.NmkStats)
    nbins = int(sv.reserved)
    rr, v = O.ratios_of(b, c)
    keys, counts = O.histogram(rr[v], float(sv.gmin), 2 * E)
    dense = np.zeros(nbins, dtype=np.int64)
    dense[keys.astype(np.int64)] = counts
    got = _dense_counts(pipe, nbins)
    np.testing.assert_array_equal(got[:nbins], dense)
    assert int(pipe.counts[nbins].item()) == 0   # tripwire
    if kind == "bimodal" and E == 1e-4:
        assert 8192 < nbins + 1 <= 20480       # the wide shape's range
    if kind == "uniform":
        assert nbins + 1 > 20480
