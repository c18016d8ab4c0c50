"""The sync-free device pipeline (engine.DevicePipeline: device-decided span,
model scalars read on the device, optional CUDA-graph replay) must produce
exactly the general path's bytes, and flag the cases it cannot handle."""

import numpy as np
import pytest

import nmk_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_1703_02438_b200 import _native as N, engine, workloads  # noqa: E402


def _host_blocks(enc):
    nlb = enc.prefix.numel()
    packed = enc.packed[: nlb * enc.stride].cpu().numpy()
    lens = enc.block_lengths()
    return [packed[i * enc.stride: i * enc.stride + int(lens[i])].tobytes() for i in range(nlb)]


def _special_mix(n, seed, dtype, spread, shift=0.0):
    """Ragged n, ratios spread over many bins, plus zeros / NaN / inf."""
    rng = np.random.default_rng(seed)
    b = rng.uniform(0.5, 2.0, n) * np.where(rng.uniform(size=n) < 0.4, -1.0, 1.0)
    c = b * (1.0 + shift + rng.uniform(-spread, spread, n))
    m = rng.uniform(size=n)
    c[m < 0.01] = np.nan
    b[(m >= 0.01) & (m < 0.02)] = 0.0
    c[(m >= 0.015) & (m < 0.02)] = 0.0
    c[(m >= 0.02) & (m < 0.025)] = np.inf
    return b.astype(dtype), c.astype(dtype)


@pytest.mark.parametrize("case", ["cfg1", "cfg2", "cfg5_b10", "cfg5_b12_e4", "f32", "many_bins", "many_bins_f32",
                                  "offset_f32", "offset_f32_far", "ragged_small"])
@pytest.mark.parametrize("graph", [False, True])
def test_pipeline_matches_general_path(case, graph):
    if case == "cfg1":
        b, c = workloads.cfg1_host(1 << 20, seed=2); E, bits, bb = 1e-3, 8, 1 << 20
    elif case == "cfg2":
        b, c = workloads.cfg2_host(64, seed=1); E, bits, bb = 1e-3, 8, 1 << 16
    elif case == "cfg5_b10":
        b, c = workloads.cfg5_host(1 << 19, seed=4); E, bits, bb = 1e-3, 10, 1 << 16
    elif case == "cfg5_b12_e4":
        b, c = workloads.cfg5_host(1 << 19, seed=5); E, bits, bb = 1e-4, 12, 1 << 17
    elif case == "f32":
        s = workloads.cfg3_host(shape=(4, 96, 192), steps=2, seed=3)
        b, c = s[0], s[1]; E, bits, bb = 5e-3, 10, 1 << 15
    elif case == "many_bins":     # ~6000 bins, hot bins never cover a tile
        b, c = _special_mix(1_000_003, 31, np.float64, 0.3); E, bits, bb = 5e-5, 12, 1 << 16
    elif case == "many_bins_f32":
        b, c = _special_mix(777_777, 32, np.float32, 0.1); E, bits, bb = 2e-5, 11, 1 << 15
    elif case == "offset_f32":    # centers away from 0: f32 quantisation offsets (direct grid)
        b, c = _special_mix(500_001, 33, np.float32, 0.01, shift=3.0); E, bits, bb = 5e-5, 9, 1 << 14
    elif case == "offset_f32_far":   # offsets too large for the direct grid: cut search
        b, c = _special_mix(500_001, 35, np.float32, 0.002, shift=30.0); E, bits, bb = 1e-5, 9, 1 << 14
    else:
        b, c = _special_mix(1_001, 34, np.float64, 0.01); E, bits, bb = 1e-3, 6, 4096
    base = torch.from_numpy(b).cuda()
    cur = torch.from_numpy(c).cuda()
    rec_general = torch.full_like(cur, float("nan"))
    ref = engine.encode(base, cur, E, bits, bb, recon=rec_general, keyed=False)   # snapshot-reading K2/K4
    ref_blocks, ref_exact = _host_blocks(ref), ref.exact.cpu().numpy().copy()
    ref_prefix = ref.prefix.cpu().numpy().copy()
    ref_out = engine.decode_encoding(ref, base).out.cpu().numpy()
    # K4's fused reconstruction is the decoder's output, bit for bit
    assert rec_general.cpu().numpy().tobytes() == ref_out.tobytes()
    pipe = engine.DevicePipeline(base.numel(), base.dtype, E, bits, bb)
    out = torch.empty_like(base)
    if graph:
        g = pipe.capture(base, cur, out)
        out.zero_()
        g.replay()
        g.replay()
    else:
        pipe.step(base, cur, out)
    chk = pipe.check()
    assert chk["status"] == 0 and not chk["bad_index"] and not chk["exhausted"]
    assert chk["n_sentinel"] == chk["n_inc"] == ref.n_inc
    enc = pipe.encoding()
    assert enc.k == ref.k and enc.gmin == ref.gmin and enc.gmax == ref.gmax
    assert enc.centers.cpu().numpy().tobytes() == ref.centers.cpu().numpy().tobytes()
    assert _host_blocks(enc) == ref_blocks
    assert enc.exact.cpu().numpy().tobytes() == ref_exact.tobytes()
    assert enc.prefix.cpu().numpy().tobytes() == ref_prefix.tobytes()
    assert out.cpu().numpy().tobytes() == ref_out.tobytes()
    # and against the oracle
    o = O.encode(b, c, E, bits, bb)
    assert enc.n_inc == o["n_inc"] and _host_blocks(enc) == o["blocks"]
    # sync-free encode with the fused reconstruction
    rec = torch.full_like(cur, float("nan"))
    pipe.encode(base, cur, recon=rec)
    assert rec.cpu().numpy().tobytes() == ref_out.tobytes()


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("E,shift", [(1e-3, 0.0), (1e-4, 0.0), (1e-4, 2.5), (5e-5, -0.7), (2e-3, 40.0)])
def test_pipeline_keys_exact_at_bin_edges(dtype, E, shift):
    """K1's f32 ratio keys drive K2 (all-f32 ordinals with an f64 and an
    exact fallback); ratios planted within 8 ulps of every bin edge, around
    zero and around an offset, must still land in the oracle's bins."""
    rng = np.random.default_rng(21)
    n = 200_000
    b = rng.uniform(0.5, 2.0, n)
    c = b * (1.0 + shift + rng.uniform(-0.02, 0.03, n))
    r, v = O.ratios_of(b.astype(dtype), c.astype(dtype))
    gmin = float(r[v].min())
    edges = gmin + np.arange(1, int(0.04 / (2 * E))) * (2 * E)
    t = rng.choice(edges, n) + np.spacing(np.abs(edges).max()) * rng.integers(-8, 9, n)
    b2 = rng.uniform(0.5, 2.0, n) * np.where(rng.uniform(size=n) < 0.3, -1.0, 1.0)
    base = np.concatenate([b, b2]).astype(dtype)
    cur = np.concatenate([c, b2 * (1.0 + t)]).astype(dtype)
    bt, ct = torch.from_numpy(base).cuda(), torch.from_numpy(cur).cuda()
    pipe = engine.DevicePipeline(bt.numel(), bt.dtype, E, 12, 1 << 16)
    out = torch.empty_like(bt)
    pipe.step(bt, ct, out)
    enc = pipe.encoding()
    o = O.encode(base, cur, E, 12, 1 << 16)
    assert enc.centers.cpu().numpy().tobytes() == o["centers"].tobytes()
    assert _host_blocks(enc) == o["blocks"]
    assert enc.exact.cpu().numpy().tobytes() == o["exact"].tobytes()
    assert out.cpu().numpy().tobytes() == O.decode(o, base).tobytes()


def test_pipeline_flags_wide_span():
    b, c = workloads.outlier_pair(50_000, seed=3)   # 5e8-bin span: sparse path needed
    base, cur = torch.from_numpy(b).cuda(), torch.from_numpy(c).cuda()
    pipe = engine.DevicePipeline(base.numel(), base.dtype, 1e-3, 2)
    out = torch.empty_like(base)
    pipe.step(base, cur, out)
    assert pipe.check()["status"] == N.NMK_ERR_NEEDS_SPARSE
    with pytest.raises(N.NativeError):
        pipe.encoding()


def test_pipeline_degenerate():
    base = torch.zeros(10_000, dtype=torch.float64, device="cuda")
    cur = torch.ones_like(base)
    pipe = engine.DevicePipeline(base.numel(), base.dtype, 1e-3, 4)
    out = torch.empty_like(base)
    pipe.step(base, cur, out)
    chk = pipe.check()
    assert chk["status"] == 0 and chk["k"] == 1 and chk["n_inc"] == 10_000
    assert torch.equal(out, cur)


@pytest.mark.parametrize("n", [1, 3, 8, 255, 256, 257, 511, 4097, 70_001])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_pipeline_small_and_ragged(n, dtype):
    """Sizes below / around the chunk (256), key tile (512) and vector widths."""
    b, c = workloads.cfg5_host(n, seed=n)
    b, c = b.astype(dtype), c.astype(dtype)
    base, cur = torch.from_numpy(b).cuda(), torch.from_numpy(c).cuda()
    pipe = engine.DevicePipeline(n, base.dtype, 1e-3, 8, 4096)
    out = torch.empty_like(base)
    pipe.step(base, cur, out)
    chk = pipe.check()
    assert chk["status"] == 0 and not chk["bad_index"] and not chk["exhausted"]
    o = O.encode(b, c, 1e-3, 8, 4096)
    enc = pipe.encoding()
    assert _host_blocks(enc) == o["blocks"]
    assert enc.exact.cpu().numpy().tobytes() == o["exact"].tobytes()
    assert out.cpu().numpy().tobytes() == O.decode(o, b).tobytes()


def _pipeline_bytes(pipe, base, cur):
    out = torch.empty_like(base)
    pipe.step(base, cur, out)
    chk = pipe.check()
    assert chk["status"] == 0 and not chk["bad_index"] and not chk["exhausted"] and chk["tripwire"] == 0
    enc = pipe.encoding()
    return (chk, _host_blocks(enc), enc.exact.cpu().numpy().tobytes(), enc.prefix.cpu().numpy().tobytes(),
            out.cpu().numpy().tobytes())


@pytest.mark.parametrize("case", ["keyed", "keyed_f32", "not_keyed"])
def test_pipeline_launch_hints_never_change_bytes(case):
    """The launch-count hints (keyed K4 without its fallback launch, a single
    K5 ring depth) are speed-only: every forced combination -- including a
    keyed hint on a field where the keyed mode does not apply, which runs the
    keyed kernel on its exact path -- gives the oracle's bytes."""
    if case == "keyed":
        b, c = workloads.cfg5_host(300_001, seed=8); E, bits, bb = 1e-3, 8, 1 << 15
    elif case == "keyed_f32":
        b, c = _special_mix(250_003, 36, np.float32, 0.05); E, bits, bb = 1e-3, 9, 1 << 14
    else:   # top bins scattered over ~50 000 bins: wider than the keyed table
        rng = np.random.default_rng(37)
        b = rng.uniform(0.5, 2.0, 400_003)
        c = b * (1.0 + rng.uniform(-1.0, 1.0, b.size))
        E, bits, bb = 2e-5, 8, 1 << 15
    base, cur = torch.from_numpy(b).cuda(), torch.from_numpy(c).cuda()
    o = O.encode(b, c, E, bits, bb)
    want_out = O.decode(o, b).tobytes()
    pipe = engine.DevicePipeline(base.numel(), base.dtype, E, bits, bb)
    chk, blocks, exact, prefix, out = _pipeline_bytes(pipe, base, cur)     # no hints: every kernel launched
    assert blocks == o["blocks"] and exact == o["exact"].tobytes() and out == want_out
    assert chk["k4_mode"] == (0 if case == "not_keyed" else 1)
    assert pipe.keyed_hint == (0 if case == "not_keyed" else 1) and pipe.ring_hint in (1, 2)
    for keyed_hint in (0, 1):
        for ring_hint in (0, 1, 2):
            pipe.keyed_hint, pipe.ring_hint = keyed_hint, ring_hint
            chk2, blocks2, exact2, prefix2, out2 = _pipeline_bytes(pipe, base, cur)
            assert (blocks2, exact2, prefix2, out2) == (blocks, exact, prefix, out), (keyed_hint, ring_hint)
            if case == "not_keyed":
                assert chk2["k4_mode"] == (2 if keyed_hint else 0)   # 2: the keyed kernel's exact path
                assert pipe.keyed_hint == 0                          # check() drops the stale hint
    # hinted pipeline captured in a graph
    g = pipe.capture(base, cur, torch.empty_like(base))
    g.replay()
    assert _host_blocks(pipe.encoding()) == o["blocks"]


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_minmax_prep_clears_wide_histograms(dtype):
    """nmk_minmax_prep = nmk_minmax + nmk_hist_prep in one launch: a span wider
    than the slots every CTA clears up front (65 537) is finished by the last
    CTA; stale counts from a previous, different step must not survive."""
    rng = np.random.default_rng(41)
    n = 600_001
    b = rng.uniform(0.5, 2.0, n)
    c = b * (1.0 + rng.uniform(-0.5, 0.5, n))
    b, c = b.astype(dtype), c.astype(dtype)
    E = 2e-6                                   # ~250 000 bins
    base, cur = torch.from_numpy(b).cuda(), torch.from_numpy(c).cuda()
    pipe = engine.DevicePipeline(n, base.dtype, E, 8, 1 << 15)
    pipe.counts.fill_(7)                       # garbage the fused prep has to clear
    out = torch.empty_like(base)
    pipe.step(base, cur, out)
    chk = pipe.check()
    assert chk["status"] == 0 and chk["tripwire"] == 0 and chk["nbins"] > 65_537
    r, v = O.ratios_of(b, c)
    ordinals, counts = O.histogram(r[v], float(r[v].min()), 2 * E)
    got = pipe.counts[: chk["nbins"]].cpu().numpy()
    dense = np.zeros(chk["nbins"], dtype=np.int64)
    dense[np.asarray(ordinals, dtype=np.int64)] = counts
    assert np.array_equal(got, dense)
    assert int(got.sum()) == chk["nvalid"]
    o = O.encode(b, c, E, 8, 1 << 15)
    assert _host_blocks(pipe.encoding()) == o["blocks"]
    assert out.cpu().numpy().tobytes() == O.decode(o, b).tobytes()


@pytest.mark.parametrize("nchunks", [1, 2, 511, 512, 513, 1024, 1025, 2049])
@pytest.mark.parametrize("tail", [-1, 0, 1])
def test_finalize_tile_boundaries(nchunks, tail):
    """k_enc_finalize takes tiles of 512 chunks with a look-back across tiles:
    element counts around every tile edge, with a few incompressible values in
    every chunk, against the oracle."""
    n = nchunks * 256 + tail
    if n <= 0:
        pytest.skip("empty")
    rng = np.random.default_rng(1000 + nchunks)
    b = rng.uniform(0.5, 2.0, n)
    c = b * (1.0 + rng.normal(0.0, 2e-3, n))
    wild = rng.uniform(size=n) < 0.01          # ~2.5 exact values per chunk
    c[wild] = b[wild] * rng.uniform(2.0, 3.0, int(wild.sum()))
    base, cur = torch.from_numpy(b).cuda(), torch.from_numpy(c).cuda()
    pipe = engine.DevicePipeline(n, base.dtype, 1e-3, 6, 4096 * 3)   # blocks of 16384 elements: 64 chunks each
    chk, blocks, exact, prefix, out = _pipeline_bytes(pipe, base, cur)
    o = O.encode(b, c, 1e-3, 6, 4096 * 3)
    assert chk["n_inc"] == o["n_inc"] and blocks == o["blocks"]
    assert exact == o["exact"].tobytes() and prefix == o["prefix"].tobytes()
    assert out == O.decode(o, b).tobytes()


@pytest.mark.parametrize("nbins_target", [65535, 65536, 65537, 65538, 131075])
def test_minmax_prep_span_boundaries(nbins_target):
    """The fused span decision clears 65 537 histogram slots up front and the
    rest in K1's last CTA: spans right at that edge, on a dirty buffer."""
    E = 1e-3
    n = 200_000
    rng = np.random.default_rng(nbins_target)
    b = np.ones(n)
    r = rng.uniform(0.0, 1.0, n) * (nbins_target - 1) * 2 * E
    r[0], r[1] = 0.0, (nbins_target - 0.5) * 2 * E          # gmin = 0, gmax inside the last bin
    c = b * (1.0 + r)
    base, cur = torch.from_numpy(b).cuda(), torch.from_numpy(c).cuda()
    pipe = engine.DevicePipeline(n, base.dtype, E, 8, 1 << 15)
    pipe.counts.fill_(3)
    out = torch.empty_like(base)
    pipe.step(base, cur, out)
    chk = pipe.check()
    assert chk["status"] == 0 and chk["tripwire"] == 0
    rr, v = O.ratios_of(b, c)
    ordinals, counts = O.histogram(rr[v], float(rr[v].min()), 2 * E)
    assert chk["nbins"] == int(ordinals.max()) + 1
    dense = np.zeros(chk["nbins"], dtype=np.int64)
    dense[np.asarray(ordinals, dtype=np.int64)] = counts
    assert np.array_equal(pipe.counts[: chk["nbins"]].cpu().numpy(), dense)
    o = O.encode(b, c, E, 8, 1 << 15)
    assert _host_blocks(pipe.encoding()) == o["blocks"]
