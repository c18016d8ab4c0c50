"""GPU parity: the CUDA path (through libnmkgpu.so) against the golden vectors
produced by the reference itself and against the pinned CPU oracle.

Bar: bit-exact for every integer / byte / index output (bins, histogram,
centers, packed codes, incompressible set, prefix table) and bit-exact
reconstruction.
"""

import hashlib
import io

import numpy as np
import pytest

import nmk_oracle as O
from conftest import golden_bits, golden_blocks, golden_names, load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1703_02438_b200 as nmk  # noqa: E402
from paper_1703_02438_b200 import _native as N, codec, container, engine, workloads  # noqa: E402


def _variable_blocks(var):
    return [codec.decompress_block(codec._block_bytes_of(var, b)) for b in range(var.nblocks)]


def _sha(var):
    return hashlib.sha256(container.to_bytes([var])).hexdigest()


def _compress(base, cur, E, bits, block_bytes=1 << 20, name="v"):
    cfg = nmk.PipelineConfig(tolerance=E, bits=bits, block_bytes=block_bytes)
    var, _ = nmk.compress_pair(nmk.TemporalPair(base, cur), cfg, name=name)
    return var


# ---------------------------------------------------------------------------
# golden vectors from the reference
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", golden_names())
def test_golden_compress_decompress(name):
    g = load_golden(name)
    var = _compress(g["base"], g["cur"], float(g["E"]), golden_bits(g), int(g["block_bytes"]))
    assert var.bits == int(g["bits"])
    assert var.centers.tobytes() == g["centers"].tobytes()
    assert var.elements_per_block == int(g["epb"]) and var.nblocks == int(g["nblocks"])
    assert var.n_incompressible == int(g["n_inc"])
    assert var.incompressible_prefix.tobytes() == g["prefix"].tobytes()
    assert var.incompressible_table.tobytes() == g["exact"].tobytes()
    assert _variable_blocks(var) == golden_blocks(g)
    assert _sha(var) == str(g["nmk_sha256"]), ".nmk bytes differ from the reference's"
    out = nmk.decompress(var, g["base"])
    assert out.tobytes() == g["decoded"].tobytes()
    pos = 0
    for s, c in g["ranges"]:
        s, c = int(s), int(c)
        part = nmk.decompress(var, g["base"][s:s + c], rng=(s, c))
        assert part.tobytes() == g["range_out"][pos:pos + c].tobytes()
        pos += c


@pytest.mark.parametrize("name", golden_names())
def test_golden_phase_intermediates(name):
    """K1 (gmin/gmax/nvalid) and K2 (histogram) against the reference's own
    compute_change_ratios / build_histogram."""
    g = load_golden(name)
    b = torch.from_numpy(g["base"]).cuda()
    c = torch.from_numpy(g["cur"]).cuda()
    enc = engine.encode(b, c, float(g["E"]), golden_bits(g), int(g["block_bytes"]))
    assert enc.nvalid == int(g["nvalid"])
    if enc.nvalid:
        assert np.float64(enc.gmin).tobytes() == g["gmin"].tobytes()
        assert np.float64(enc.gmax).tobytes() == g["gmax"].tobytes()
        keys, counts = _device_histogram(b, c, float(g["E"]), enc)
        np.testing.assert_array_equal(keys, g["hist_keys"])
        np.testing.assert_array_equal(counts, g["hist_counts"])


def _device_histogram(b, c, E, enc):
    """Run K2 again and return (sorted nonempty ordinals, counts)."""
    lib = N.lib()
    ws = engine.default_workspace()
    stats = torch.tensor([np.float64(enc.gmin).view(np.int64), np.float64(enc.gmax).view(np.int64),
                          enc.nvalid, 0], dtype=torch.int64, device="cuda")
    dt = engine.torch_dtype_code(b)
    width = 2.0 * E
    st = torch.cuda.current_stream().cuda_stream
    if enc.hist_form == "dense":
        nbins = int(np.floor((enc.gmax - enc.gmin) / width)) + 1
        counts = torch.empty(nbins + 1, dtype=torch.int64, device="cuda")
        N.check(lib.nmk_hist_dense(b.data_ptr(), c.data_ptr(), b.numel(), dt, stats.data_ptr(), width, nbins,
                                   counts.data_ptr(), st))
        cn = counts.cpu().numpy()
        assert cn[nbins] == 0
        nz = np.flatnonzero(cn[:nbins])
        return nz.astype(np.float64), cn[nz]
    n = b.numel()
    keys = torch.empty(n, dtype=torch.int64, device="cuda")
    counts = torch.empty(n, dtype=torch.int64, device="cuda")
    nruns = torch.zeros(1, dtype=torch.int64, device="cuda")
    nb = lib.nmk_hist_sparse_ws_bytes(n)
    wsb = torch.empty(nb, dtype=torch.uint8, device="cuda")
    N.check(lib.nmk_hist_sparse(b.data_ptr(), c.data_ptr(), n, dt, stats.data_ptr(), width, keys.data_ptr(),
                                counts.data_ptr(), nruns.data_ptr(), wsb.data_ptr(), nb, st))
    m = int(nruns.item())
    return keys[:m].cpu().numpy().view(np.float64), counts[:m].cpu().numpy()


@pytest.mark.parametrize("name", ["series_drift_f32", "series_cfg3_b10"])
def test_golden_series(name):
    g = load_golden(name)
    snaps = [g[f"snap{i}"] for i in range(int(g["nsteps"]))]
    cfg = nmk.PipelineConfig(tolerance=float(g["E"]), bits=golden_bits(g), block_bytes=int(g["block_bytes"]))
    first, variables = nmk.compress_series(snaps, cfg, name="s")
    assert first.tobytes() == snaps[0].tobytes()
    recon = first
    for i, v in enumerate(variables, start=1):
        assert v.name == f"s.{i:04d}"
        assert v.bits == int(g[f"bits{i}"])
        assert v.centers.tobytes() == g[f"centers{i}"].tobytes()
        assert b"".join(_variable_blocks(v)) == g[f"packed{i}"].tobytes()
        assert v.incompressible_table.tobytes() == g[f"exact{i}"].tobytes()
        assert _sha(v) == str(g[f"sha{i}"])
        recon = nmk.decompress(v, recon)
        assert recon.tobytes() == g[f"recon{i}"].tobytes()


# ---------------------------------------------------------------------------
# oracle parity on the BASELINE configurations (reduced sizes)
# ---------------------------------------------------------------------------

def _check_against_oracle(base, cur, E, bits, block_bytes=1 << 20, ranges=()):
    ref = O.encode(base, cur, E, bits, block_bytes, workers=4)
    var = _compress(base, cur, E, bits, block_bytes)
    assert var.bits == ref["bits"]
    assert var.centers.tobytes() == ref["centers"].astype(base.dtype).tobytes()
    assert var.n_incompressible == ref["n_inc"]
    assert var.incompressible_prefix.tobytes() == ref["prefix"].tobytes()
    assert var.incompressible_table.tobytes() == ref["exact"].tobytes()
    assert _variable_blocks(var) == ref["blocks"]
    out = nmk.decompress(var, base)
    assert out.tobytes() == O.decode(ref, base).tobytes()
    for s, c in ranges:
        part = nmk.decompress(var, base[s:s + c], rng=(s, c))
        assert part.tobytes() == out[s:s + c].tobytes()
    return var


def test_cfg1_full_size():
    base, cur = workloads.cfg1_host(1 << 20, seed=0)
    var = _check_against_oracle(base, cur, 1e-3, 8, ranges=[(0, 10), (123457, 65536), ((1 << 20) - 5, 5)])
    assert var.k == 50


def test_cfg2_reduced_grid():
    base, cur = workloads.cfg2_host(64, seed=0)
    _check_against_oracle(base, cur, 1e-3, 8, block_bytes=1 << 16)


def test_cfg3_transition_reduced():
    snaps = workloads.cfg3_host(shape=(6, 144, 288), steps=3, seed=1)
    _check_against_oracle(snaps[0], snaps[1], 5e-3, 10, block_bytes=1 << 16)


@pytest.mark.parametrize("bits", [8, 10, 12])
@pytest.mark.parametrize("E", [1e-4, 1e-3, 1e-2])
def test_cfg5_sweep_reduced(bits, E):
    base, cur = workloads.cfg5_host(1 << 18, seed=7)
    _check_against_oracle(base, cur, E, bits, block_bytes=1 << 15, ranges=[(1000, 70000), (200000, 60000)])


@pytest.mark.parametrize("bits", [2, 3, 5, 7, 9, 13, 16, 17, 23, 30])
def test_odd_bit_lengths(bits):
    base, cur = workloads.cfg5_host(50_003, seed=bits)
    _check_against_oracle(base, cur, 1e-3, bits, block_bytes=4096, ranges=[(4095, 3), (7, 40_000)])


def test_auto_bits_matches_oracle():
    for seed, spread in ((1, 0.01), (2, 0.3), (3, 3.0)):
        base, cur = workloads.uniform_pair(30_000, seed=seed, dtype=np.float64, spread=spread)
        _check_against_oracle(base, cur, 1e-3, None)


def test_sparse_histogram_planted_outliers():
    base, cur = workloads.outlier_pair(100_000, seed=11)
    var = _check_against_oracle(base, cur, 1e-3, 2)
    assert abs(var.alpha - 0.02) < 1e-3


def test_wild_pairs():
    rng = np.random.default_rng(99)
    for i in range(40):
        dt = np.float32 if i % 2 == 0 else np.float64
        b, c = workloads.wild_pair(rng, dt)
        _check_against_oracle(b, c, 1e-3, None)


# ---------------------------------------------------------------------------
# edge cases
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("n", [1, 2, 7, 8, 9, 2047, 2048, 2049, 4096 * 3 + 1])
def test_small_and_ragged_sizes(n):
    base, cur = workloads.uniform_pair(n, seed=n, dtype=np.float64, spread=0.02)
    _check_against_oracle(base, cur, 1e-3, 8, block_bytes=4096, ranges=[(0, n), (n // 2, n - n // 2)])


def test_all_invalid_degenerate():
    var = _check_against_oracle(np.zeros(5000), np.ones(5000), 1e-3, None)
    assert var.alpha == 1.0 and var.bits == 2 and var.k == 1


def test_constant_pair_single_center():
    rng = np.random.default_rng(5)
    base = rng.uniform(-10, 10, 4000)
    var = _check_against_oracle(base, base.copy(), 1e-3, None)
    assert var.alpha == 0.0 and var.k == 1


def test_nan_payload_and_denormals_bit_exact():
    payload = np.array([0x7FF8000000001234, 0x7FF0000000000001, 0xFFF8000000000042], dtype=np.uint64)
    base = np.ones(64)
    cur = base * 1.0005
    cur[[3, 17, 40]] = payload.view(np.float64)
    base[50] = 5e-310
    cur[51] = 5e-310
    var = _check_against_oracle(base, cur, 1e-3, 4)
    out = nmk.decompress(var, base)
    assert out.view(np.uint64)[[3, 17, 40]].tolist() == payload.tolist()


def test_f32_denormals():
    base = np.full(1000, 1.5, dtype=np.float32)
    cur = (base * np.float32(1.0002)).astype(np.float32)
    base[::7] = np.float32(1e-42)
    cur[::11] = np.float32(1e-42)
    _check_against_oracle(base, cur, 1e-3, 6)


def test_error_bound_holds_everywhere():
    base, cur = workloads.uniform_pair(200_000, seed=13, dtype=np.float32, spread=0.03)
    var = _compress(base, cur, 1e-3, None)
    out = nmk.decompress(var, base)
    idx = nmk.decode_all_indices(var)
    comp = idx != (1 << var.bits) - 1
    b64 = base.astype(np.float64)
    err = np.abs(out.astype(np.float64) - cur.astype(np.float64))
    assert (err[comp] <= 1e-3 * np.abs(b64[comp])).all()
    assert out[~comp].view(np.uint32).tolist() == cur[~comp].view(np.uint32).tolist()


# ---------------------------------------------------------------------------
# codec surface and error behaviour
# ---------------------------------------------------------------------------

def test_pack_unpack_kats():
    assert nmk.pack_block(np.array([0xA, 0x5]), 4) == b"\xa5"
    assert nmk.pack_block(np.array([7, 7, 7]), 3) == b"\xff\x80"
    assert nmk.pack_block(np.arange(256), 8) == bytes(range(256))
    assert list(nmk.unpack_block(b"\xff\x80", 3, 3)) == [7, 7, 7]
    with pytest.raises(nmk.CodecError):
        nmk.pack_block(np.array([8]), 3)
    with pytest.raises(nmk.CodecError):
        nmk.unpack_block(b"\xff", 3, 3)


@pytest.mark.parametrize("bits", range(2, 31))
def test_pack_round_trip_vs_oracle(bits):
    rng = np.random.default_rng(bits)
    idx = rng.integers(0, 1 << bits, 997)
    p = nmk.pack_block(idx, bits)
    assert p == O.pack(idx, bits)
    np.testing.assert_array_equal(nmk.unpack_block(p, bits, 997), idx)


def test_reconstruct_rules():
    f64 = lambda *v: np.array(v, dtype=np.float64)  # noqa: E731
    assert nmk.reconstruct(f64(7.0), f64(0.1), np.array([3]), f64(9.5), bits=2)[0] == 9.5
    assert nmk.reconstruct(f64(4.0), f64(0.0), np.array([0]), f64(), bits=2)[0] == 4.0
    payload = np.array([0x7FF8000000001234], dtype=np.uint64).view(np.float64)
    out = nmk.reconstruct(f64(1.0), f64(0.0), np.array([3]), payload, bits=2)
    assert out.view(np.uint64)[0] == 0x7FF8000000001234
    with pytest.raises(ValueError, match="out of range"):
        nmk.reconstruct(f64(1.0), f64(0.0), np.array([1]), f64(), bits=2)
    with pytest.raises(ValueError, match="exhausted"):
        nmk.reconstruct(f64(1.0, 2.0), f64(0.0), np.array([3, 3]), f64(5.0), bits=2)
    with pytest.raises(ValueError, match="not fully consumed"):
        nmk.reconstruct(f64(1.0), f64(0.0), np.array([0]), f64(5.0), bits=2)


def test_corrupt_block_raises_codec_error():
    base, cur = workloads.uniform_pair(30000, seed=37)
    var = _compress(base, cur, 1e-3, 6, block_bytes=4096)
    broken = container.CompressedVariable(**{**var.__dict__, "index_table": b"\x00" * len(var.index_table)})
    with pytest.raises(nmk.CodecError):
        nmk.decompress(broken, base)


def test_truncated_exact_table_raises():
    base, cur = workloads.outlier_pair(20000, seed=3)
    var = _compress(base, cur, 1e-3, 2)
    short = container.CompressedVariable(**{**var.__dict__,
                                            "incompressible_table": var.incompressible_table[:-5]})
    with pytest.raises(ValueError, match="exhausted"):
        nmk.decompress(short, base)


def test_bad_center_index_raises():
    base, cur = workloads.uniform_pair(5000, seed=4, dtype=np.float64, spread=0.02)
    var = _compress(base, cur, 1e-3, 8)
    fewer = container.CompressedVariable(**{**var.__dict__, "centers": var.centers[:3]})
    with pytest.raises(ValueError, match="out of range"):
        nmk.decompress(fewer, base)


def test_zlib_fault_tags_phase(monkeypatch):
    def boom(packed, level=6):
        raise RuntimeError("injected failure")

    monkeypatch.setattr(codec, "compress_block", boom)
    base, cur = workloads.uniform_pair(5000, seed=29)
    with pytest.raises(nmk.PipelineError) as excinfo:
        nmk.compress_pair(nmk.TemporalPair(base, cur), nmk.PipelineConfig(workers=2))
    assert excinfo.value.phase == "zlib"


def test_workers_do_not_change_output():
    base, cur = workloads.uniform_pair(10007, seed=3)
    outs = []
    for w in (1, 2, 5):
        var, _ = nmk.compress_pair(nmk.TemporalPair(base, cur), nmk.PipelineConfig(workers=w))
        outs.append(container.to_bytes([var]))
    assert outs[0] == outs[1] == outs[2]


def test_timings_cover_phases():
    base, cur = workloads.uniform_pair(5000, seed=23)
    _, t = nmk.compress_pair(nmk.TemporalPair(base, cur), nmk.PipelineConfig(workers=2))
    assert all(getattr(t, p) >= 0 for p in t.PHASES) and t.io == 0.0


def test_range_validation():
    base, cur = workloads.uniform_pair(30000, seed=37)
    var = _compress(base, cur, 1e-3, 6, block_bytes=4096)
    assert nmk.decompress(var, base[:0], rng=(0, 0)).size == 0
    with pytest.raises(ValueError):
        nmk.decompress(var, base[:10], rng=(var.n - 5, 10))
    with pytest.raises(ValueError):
        nmk.decompress(var, base[:-1])


# ---------------------------------------------------------------------------
# device engine: full BASELINE sizes through size-independent properties
# ---------------------------------------------------------------------------

def test_cfg2_full_size_properties():
    """512^3 fp64: decode(encode(x)) within E per compressible element,
    incompressible bit-exact, prefix table = scan of sentinel counts, and the
    model (gmin/gmax, B, centers) equal to the oracle's on the same field."""
    base, cur = workloads.cfg2_device(512, seed=0)
    enc = engine.encode(base, cur, 1e-3, 8)
    assert enc.bits == 8 and enc.k == 255 and enc.nblocks == 128
    res = engine.decode_encoding(enc, base)
    assert not res.bad_index and not res.exhausted
    assert int(res.n_sentinel[0]) == enc.n_inc
    out = res.out
    # codes: unpack the device stream
    codes = torch.empty(enc.n, dtype=torch.int32, device="cuda")
    for b in range(enc.nblocks):
        s, e = b * enc.epb, min((b + 1) * enc.epb, enc.n)
        N.check(N.lib().nmk_unpack(enc.packed.data_ptr() + b * enc.stride, e - s, enc.bits,
                                   codes.data_ptr() + 4 * s, torch.cuda.current_stream().cuda_stream))
    sent = codes == enc.sentinel
    assert int(sent.sum()) == enc.n_inc
    comp = ~sent
    err = (out.double() - cur.double()).abs()
    assert bool((err[comp] <= 1e-3 * base.double().abs()[comp]).all())
    assert torch.equal(out[sent].view(torch.int64), cur[sent].view(torch.int64))
    assert torch.equal(enc.exact.view(torch.int64), cur[sent].view(torch.int64))
    per_block = sent.view(-1)[: enc.nblocks * enc.epb].reshape(enc.nblocks, enc.epb).sum(1)
    pre = torch.zeros_like(per_block)
    pre[1:] = torch.cumsum(per_block, 0)[:-1]
    assert torch.equal(enc.prefix.cpu(), pre.cpu())
    # the model against the oracle on the identical field (host copy)
    hb, hc = base.cpu().numpy(), cur.cpu().numpy()
    r, v = O.ratios_of(hb, hc)
    mm = O.minmax_of(r, v)
    assert (enc.gmin, enc.gmax) == mm
    keys, counts = O.histogram(r[v], mm[0], 2e-3)
    centers = O.quantize(O.top_k(keys, counts, mm[0], 2e-3, 8), hb.dtype)
    assert enc.centers.cpu().numpy().tobytes() == centers.tobytes()


def test_device_partial_segments_batch():
    """1000 random 2^16 segments decoded in one launch == slices of the full decode."""
    base, cur = workloads.cfg5_device(1 << 24, seed=3)
    enc = engine.encode(base, cur, 1e-3, 10)
    full = engine.decode_encoding(enc, base).out
    rng = np.random.default_rng(0)
    starts = rng.integers(0, enc.n - (1 << 16), 1000)
    segs = [(int(s), 1 << 16, i << 16) for i, s in enumerate(starts)]
    idx = torch.from_numpy(np.concatenate([np.arange(s, s + (1 << 16)) for s, _, _ in segs])).cuda()
    base_cat = base[idx]
    res = engine.decode(enc.packed, enc.stride, 0, enc.bits, enc.epb, enc.n, enc.prefix, enc.centers, enc.exact,
                        base_cat, segs)
    assert not res.bad_index and not res.exhausted
    assert torch.equal(res.out.view(torch.int64), full[idx].view(torch.int64))


@pytest.mark.parametrize("bits", [9, 10, 11, 12, 14, 15])
@pytest.mark.parametrize("n", [256 * 37, 256 * 37 + 101, 7])
@pytest.mark.parametrize("frac", [0.0, 0.3, 1.0])
def test_decode_sentinel_counts_vs_oracle(bits, n, frac):
    """K5's per-chunk sentinel counts (the SWAR count for B = 10/12/14, the
    code-extraction count otherwise) through reconstruct: random ids with a
    given sentinel fraction, ragged element counts, all-sentinel streams."""
    rng = np.random.default_rng(bits * 1000 + n)
    k = 37
    sentinel = (1 << bits) - 1
    idx = rng.integers(0, k, n)
    idx[rng.uniform(size=n) < frac] = sentinel
    centers = np.sort(rng.uniform(-0.05, 0.05, k))
    base = rng.lognormal(0.0, 1.0, n)
    exact = rng.normal(size=int((idx == sentinel).sum()))
    got = nmk.reconstruct(base, centers, idx, exact, bits=bits)
    want = O.reconstruct(base, centers, idx, exact, bits)
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("bits", [8, 10, 17])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_bad_index_reports_largest_id(bits, dtype):
    """Ids in [k, 2^B - 1) inside whole chunks (K5's fast path) are reported
    with the largest such id, as the reference's reconstruct does
    (core.py:181-187); the sentinel itself is never a bad id."""
    rng = np.random.default_rng(bits)
    n = 256 * 64
    k = 5
    sentinel = (1 << bits) - 1
    idx = rng.integers(0, k, n)
    idx[rng.uniform(size=n) < 0.2] = sentinel
    bad_pos = rng.choice(n, 7, replace=False)
    bad_ids = rng.integers(k, sentinel, 7)
    idx[bad_pos] = bad_ids
    base = rng.lognormal(0.0, 1.0, n).astype(dtype)
    exact = rng.normal(size=int((idx == sentinel).sum())).astype(dtype)
    with pytest.raises(ValueError, match=f"index {int(bad_ids.max())} out of range for {k} centers"):
        nmk.reconstruct(base, np.linspace(-0.01, 0.01, k), idx, exact, bits=bits)


@pytest.mark.parametrize("zero_frac", [0.0, 0.0020, 0.0030, 0.05])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_decode_ring_regimes(zero_frac, dtype):
    """K5 picks its TMA ring by exact-value density (1 per 400 elements,
    `dec_dense` in k_decode.cu): streams on both sides of the threshold decode
    bit-exactly like the oracle, in full and in partial ranges."""
    rng = np.random.default_rng(1703)
    n = (1 << 20) + 4093
    base = rng.lognormal(0.0, 1.0, n).astype(dtype)
    base[rng.random(n) < zero_frac] = 0
    r = 0.9 * rng.normal(0, 0.002, n) + 0.1 * rng.uniform(-0.05, 0.05, n)
    cur = (base * (1 + r)).astype(dtype)
    _check_against_oracle(base, cur, 1e-3, 8, ranges=[(0, 1000), (12345, 65536), (n - 777, 777)])
