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


@pytest.mark.parametrize("case", ["cfg1", "cfg2", "cfg5_b10", "cfg5_b12_e4", "f32"])
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
    else:
        s = workloads.cfg3_host(shape=(4, 96, 192), steps=2, seed=3)
        b, c = s[0], s[1]; E, bits, bb = 5e-3, 10, 1 << 15
    base = torch.from_numpy(b).cuda()
    cur = torch.from_numpy(c).cuda()
    ref = engine.encode(base, cur, E, bits, bb)
    ref_blocks, ref_exact = _host_blocks(ref), ref.exact.cpu().numpy().copy()
    ref_prefix = ref.prefix.cpu().numpy().copy()
    ref_out = engine.decode_encoding(ref, base).out.cpu().numpy()
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


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("E", [1e-3, 1e-4])
def test_pipeline_keys_exact_at_bin_edges(dtype, E):
    """K1's f32 ratio keys drive K2; ratios planted within 8 ulps of every bin
    edge must still land in the oracle's bins (the exact fallback kicks in)."""
    rng = np.random.default_rng(21)
    n = 200_000
    b = rng.uniform(0.5, 2.0, n)
    c = b * (1.0 + rng.uniform(-0.02, 0.03, n))
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
