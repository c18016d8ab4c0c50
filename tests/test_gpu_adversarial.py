"""Adversarial exactness: change ratios planted within a few ulps of every
decision boundary of the path — histogram bin edges (K2's division-free fast
path), midpoint cuts between centers (K4's grid search), the |r - c| <= E
acceptance edge and the round-trip filter — must give the oracle's bits."""

import numpy as np
import pytest

import nmk_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1703_02438_b200 as nmk  # noqa: E402
from paper_1703_02438_b200 import codec  # noqa: E402


def _plant(rng, targets, n, dtype):
    """Pairs whose ratio lands within ~8 ulps of the given target ratios."""
    t = rng.choice(targets, n)
    t = t + np.spacing(np.abs(t) + 1e-300) * rng.integers(-8, 9, n)
    b = rng.uniform(0.5, 2.0, n) * np.where(rng.uniform(size=n) < 0.3, -1.0, 1.0)
    x = b * (1.0 + t)
    return b.astype(dtype), x.astype(dtype)


def _check(base, cur, E, bits, block_bytes=1 << 16):
    ref = O.encode(base, cur, E, bits, block_bytes, workers=4)
    var, _ = nmk.compress_pair(nmk.TemporalPair(base, cur),
                               nmk.PipelineConfig(tolerance=E, bits=bits, block_bytes=block_bytes))
    assert var.bits == ref["bits"]
    assert var.centers.tobytes() == ref["centers"].astype(base.dtype).tobytes()
    blocks = [codec.decompress_block(codec._block_bytes_of(var, b)) for b in range(var.nblocks)]
    assert blocks == ref["blocks"]
    assert var.incompressible_table.tobytes() == ref["exact"].tobytes()
    assert nmk.decompress(var, base).tobytes() == O.decode(ref, base).tobytes()
    return ref


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("E", [1e-3, 1e-4, 3.3e-3])
def test_bin_edges(dtype, E):
    rng = np.random.default_rng(11)
    n = 300_000
    base = rng.uniform(0.5, 2.0, n)
    cur = base * (1.0 + rng.uniform(-0.02, 0.03, n))
    base, cur = base.astype(dtype), cur.astype(dtype)
    r, v = O.ratios_of(base, cur)
    gmin = float(r[v].min())
    w = 2.0 * E
    edges = gmin + np.arange(1, int(0.04 / w)) * w      # exact-ish bin edges
    pb, px = _plant(rng, edges, n // 2, dtype)
    base = np.concatenate([base, pb])
    cur = np.concatenate([cur, px])
    _check(base, cur, E, None)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_cut_and_tolerance_edges(dtype):
    rng = np.random.default_rng(12)
    E = 1e-3
    n = 200_000
    base = rng.lognormal(0.0, 1.0, n)
    cur = base * (1.0 + np.where(rng.uniform(size=n) < 0.8, rng.normal(0, 0.004, n),
                                 rng.uniform(-0.05, 0.05, n)))
    base, cur = base.astype(dtype), cur.astype(dtype)
    ref = O.encode(base, cur, E, 8)
    c = ref["centers"]
    cuts = 0.5 * (c[:-1] + c[1:])
    targets = np.concatenate([cuts, c + E, c - E, c + E * (1 - 1e-9), c - E * (1 + 1e-9)])
    pb, px = _plant(rng, targets, n, dtype)
    _check(np.concatenate([base, pb]), np.concatenate([cur, px]), E, 8)


def test_extreme_magnitudes_take_the_ieee_path():
    """b near the ends of the exponent range, quotients overflowing or
    subnormal: the fast path must step aside and the IEEE rules apply."""
    rng = np.random.default_rng(13)
    n = 50_000
    mag = 10.0 ** rng.uniform(-300, 300, n)
    base = mag * np.where(rng.uniform(size=n) < 0.5, -1, 1)
    cur = base * (1 + rng.normal(0, 0.003, n))
    cur[::97] = 1e300
    base[::89] = 1e-305
    cur[::101] = 5e-324
    _check(base, cur, 1e-3, None)
