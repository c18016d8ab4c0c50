"""Seeded synthetic temporal fields for the BASELINE.json configurations.

The paper's datasets (FLASH / ASR / CMIP) are not available here; these
generators stand in for them with the shapes, sizes and value distributions
BASELINE.json specifies.  Each config has a host (numpy)
form for parity tests and a device (torch, Philox) form for the large bench
sizes.  They are inputs, not part of the compression path.
"""

from __future__ import annotations

import math

import numpy as np


# ---------------------------------------------------------------------------
# cfg1 / cfg4: lognormal base, 0.9 N(0, 0.002) + 0.1 U(-0.05, 0.05) ratios,
# 0.5 % of the base zeroed AFTER forming x_t (zero base, nonzero current ->
# incompressible; SURVEY.md §8(d) cfg1 note).
# ---------------------------------------------------------------------------

def cfg1_host(n: int = 1 << 20, seed: int = 0):
    rng = np.random.default_rng(seed)
    base = rng.lognormal(0.0, 1.0, n)
    pick = rng.uniform(size=n) < 0.9
    r = np.where(pick, rng.normal(0.0, 0.002, n), rng.uniform(-0.05, 0.05, n))
    cur = base * (1.0 + r)
    zero = rng.uniform(size=n) < 0.005
    base[zero] = 0.0
    return base, cur


def cfg1_device(n: int, seed: int = 0, device="cuda", dtype=None):
    import torch
    dtype = dtype or torch.float64
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    base = torch.empty(n, dtype=torch.float64, device=device)
    base.log_normal_(0.0, 1.0, generator=g)
    u = torch.rand(n, dtype=torch.float64, device=device, generator=g)
    r = torch.randn(n, dtype=torch.float64, device=device, generator=g).mul_(0.002)
    alt = torch.rand(n, dtype=torch.float64, device=device, generator=g).mul_(0.1).sub_(0.05)
    r = torch.where(u < 0.9, r, alt)
    del alt, u
    cur = base * (1.0 + r)
    del r
    zero = torch.rand(n, dtype=torch.float64, device=device, generator=g) < 0.005
    base.masked_fill_(zero, 0.0)
    return base.to(dtype), cur.to(dtype)


def cfg1_device_range(lo: int, hi: int, seed: int = 0, chunk: int = 1 << 26, device="cuda"):
    """Elements [lo, hi) of ONE global config-1 field of any length (config 4
    strong scaling: 4e9 elements), generated chunk by chunk with per-chunk
    seeds, so every rank of every world size sees the same global field."""
    import torch
    n = hi - lo
    base = torch.empty(n, dtype=torch.float64, device=device)
    cur = torch.empty(n, dtype=torch.float64, device=device)
    c0, c1 = lo // chunk, (hi - 1) // chunk if n else lo // chunk - 1
    for c in range(c0, c1 + 1):
        a, b_ = max(lo, c * chunk), min(hi, (c + 1) * chunk)
        cb, cc = cfg1_device(chunk, seed=seed * 1_000_003 + c, device=device)
        base[a - lo:b_ - lo] = cb[a - c * chunk:b_ - c * chunk]
        cur[a - lo:b_ - lo] = cc[a - c * chunk:b_ - c * chunk]
        del cb, cc
    return base, cur


# ---------------------------------------------------------------------------
# cfg2: 3-D smooth field on an N^3 grid in 8^3-cell blocks (row-major block
# order), box-filtered N(0, 0.003) ratio + 2 % Laplace(0, 0.1) outliers.
# ---------------------------------------------------------------------------

def _to_block_order(vol, cell=8):
    """(z, y, x) volume -> (bz, by, bx, cz, cy, cx) flattened."""
    n = vol.shape[0]
    nb = n // cell
    v = vol.reshape(nb, cell, nb, cell, nb, cell)
    return v.transpose(0, 2, 4, 1, 3, 5).reshape(-1)


def cfg2_host(side: int = 64, seed: int = 0):
    rng = np.random.default_rng(seed)
    ax = (np.arange(side) + 0.5) / side
    s = np.sin(2 * np.pi * ax)
    base = 1.0 + 0.5 * s[:, None, None] * s[None, :, None] * s[None, None, :]
    base = base + rng.normal(0.0, 0.01, base.shape)
    noise = rng.normal(0.0, 0.003, base.shape)
    r = noise
    for axis in range(3):            # periodic 5^3 box filter, separable
        acc = np.zeros_like(r)
        for d in range(-2, 3):
            acc += np.roll(r, d, axis=axis)
        r = acc / 5.0
    out = rng.uniform(size=base.shape) < 0.02
    r[out] += rng.laplace(0.0, 0.1, int(out.sum()))
    cur = base * (1.0 + r)
    return _to_block_order(base), _to_block_order(cur)


def cfg2_device(side: int = 512, seed: int = 0, device="cuda"):
    import torch
    import torch.nn.functional as F
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    ax = (torch.arange(side, dtype=torch.float64, device=device) + 0.5) / side
    s = torch.sin(2 * math.pi * ax)
    base = 1.0 + 0.5 * s[:, None, None] * s[None, :, None] * s[None, None, :]
    base = base + torch.randn(base.shape, dtype=torch.float64, device=device, generator=g) * 0.01
    noise = torch.randn(base.shape, dtype=torch.float64, device=device, generator=g) * 0.003
    # periodic 5^3 box filter = separable 1-D circular means
    r = noise
    for dim in range(3):
        acc = torch.zeros_like(r)
        for d in range(-2, 3):
            acc += torch.roll(r, d, dims=dim)
        r = acc / 5.0
    del noise, acc
    out = torch.rand(base.shape, dtype=torch.float64, device=device, generator=g) < 0.02
    u = torch.rand(base.shape, dtype=torch.float64, device=device, generator=g) - 0.5
    lap = -0.1 * torch.sign(u) * torch.log1p(-2.0 * u.abs())
    del u
    r = r + torch.where(out, lap, torch.zeros_like(lap))
    del lap, out
    cur = base * (1.0 + r)
    del r
    nb = side // 8

    def blk(v):
        return v.reshape(nb, 8, nb, 8, nb, 8).permute(0, 2, 4, 1, 3, 5).contiguous().reshape(-1)

    return blk(base), blk(cur)


# ---------------------------------------------------------------------------
# cfg3: fp32 climate-like series on (level, lat, lon), x0 ~ U(200, 320),
# 0.1 % exact zeros at fixed positions, r_t ~ N(0, 0.005) * |sin(lat)|.
# ---------------------------------------------------------------------------

def cfg3_host(shape=(30, 72, 144), steps: int = 16, seed: int = 0):
    rng = np.random.default_rng(seed)
    lev, nlat, nlon = shape
    lat = np.deg2rad(-90.0 + (np.arange(nlat) + 0.5) * 180.0 / nlat)
    env = np.abs(np.sin(lat))[None, :, None]
    x = rng.uniform(200.0, 320.0, shape)
    zero = rng.uniform(size=shape) < 0.001
    x[zero] = 0.0
    snaps = [x.astype(np.float32).reshape(-1)]
    for _ in range(steps - 1):
        r = rng.normal(0.0, 0.005, shape) * env
        nxt = (snaps[-1].astype(np.float64).reshape(shape) * (1.0 + r)).astype(np.float32)
        snaps.append(nxt.reshape(-1))
    return snaps


def cfg3_device_step(prev, t: int, seed: int = 0, shape=(30, 720, 1440)):
    """x_t = f32(f64(x_{t-1}) * (1 + r_t)) on the device."""
    import torch
    lev, nlat, nlon = shape
    g = torch.Generator(device=prev.device)
    g.manual_seed(seed * 1000 + t)
    lat = torch.deg2rad(-90.0 + (torch.arange(nlat, dtype=torch.float64, device=prev.device) + 0.5)
                        * 180.0 / nlat)
    env = torch.sin(lat).abs()[None, :, None]
    r = torch.randn(shape, dtype=torch.float64, device=prev.device, generator=g) * 0.005 * env
    return (prev.double().reshape(shape) * (1.0 + r)).float().reshape(-1)


def cfg3_device_first(seed: int = 0, shape=(30, 720, 1440), device="cuda"):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    x = torch.rand(shape, dtype=torch.float64, device=device, generator=g) * 120.0 + 200.0
    zero = torch.rand(shape, dtype=torch.float64, device=device, generator=g) < 0.001
    x.masked_fill_(zero, 0.0)
    return x.float().reshape(-1)


# ---------------------------------------------------------------------------
# cfg5: lognormal base, bimodal ratio N(-0.02, 0.004) / N(0.03, 0.006) with
# 20 % U(-1, 1) outliers.
# ---------------------------------------------------------------------------

def cfg5_host(n: int = 1 << 16, seed: int = 0):
    rng = np.random.default_rng(seed)
    base = rng.lognormal(0.0, 1.0, n)
    u = rng.uniform(size=n)
    r = np.where(u < 0.4, rng.normal(-0.02, 0.004, n),
                 np.where(u < 0.8, rng.normal(0.03, 0.006, n), rng.uniform(-1.0, 1.0, n)))
    return base, base * (1.0 + r)


def cfg5_device(n: int, seed: int = 0, device="cuda"):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    base = torch.empty(n, dtype=torch.float64, device=device).log_normal_(0.0, 1.0, generator=g)
    u = torch.rand(n, dtype=torch.float64, device=device, generator=g)
    a = torch.randn(n, dtype=torch.float64, device=device, generator=g) * 0.004 - 0.02
    b = torch.randn(n, dtype=torch.float64, device=device, generator=g) * 0.006 + 0.03
    c = torch.rand(n, dtype=torch.float64, device=device, generator=g) * 2.0 - 1.0
    r = torch.where(u < 0.4, a, torch.where(u < 0.8, b, c))
    del a, b, c, u
    return base, base * (1.0 + r)


# ---------------------------------------------------------------------------
# Reference-test style inputs (shapes of pkg/tests generators, own code)
# ---------------------------------------------------------------------------

def uniform_pair(n=5000, seed=0, dtype=np.float32, spread=0.01):
    """U(1,2) base with a U(-spread, spread) relative change."""
    rng = np.random.default_rng(seed)
    base = rng.uniform(1.0, 2.0, n)
    cur = base * (1.0 + rng.uniform(-spread, spread, n))
    return base.astype(dtype), cur.astype(dtype)


def wild_pair(rng: np.random.Generator, dtype, E: float = 1e-3):
    """Random pair with zeros / NaN / +-Inf / denormals and magnitudes
    spanning up to 10^+-30 — the stress shape of the reference's
    acceptance criterion 1."""
    dtype = np.dtype(dtype)
    n = int(10 ** rng.uniform(0, 4.3))
    span = 30.0 if rng.uniform() < 0.3 else 3.0
    mag = 10 ** rng.uniform(-span, span, n)
    base = np.where(rng.uniform(size=n) < 0.5, mag, -mag)
    mode = rng.uniform(size=n)
    cur = base * (1.0 + rng.normal(0.0, 5 * E, n))
    cur = np.where(mode < 0.15, base, cur)
    big = 10 ** rng.uniform(-span, span, n)
    cur = np.where((mode >= 0.15) & (mode < 0.30),
                   np.where(rng.uniform(size=n) < 0.5, big, -big), cur)

    def sprinkle(a):
        spot = rng.uniform(size=n)
        a = np.where(spot < 0.02, 0.0, a)
        a = np.where((spot >= 0.02) & (spot < 0.03), np.nan, a)
        a = np.where((spot >= 0.03) & (spot < 0.04), np.inf, a)
        a = np.where((spot >= 0.04) & (spot < 0.05), -np.inf, a)
        tiny = 1e-42 if dtype.itemsize == 4 else 5e-310
        return np.where((spot >= 0.05) & (spot < 0.06), tiny, a)

    with np.errstate(all="ignore"):
        return sprinkle(base).astype(dtype), sprinkle(cur).astype(dtype)


def outlier_pair(n: int, seed: int = 0, frac: float = 0.02, E: float = 1e-3, dtype="f8"):
    """Tight cluster within E/2 plus far outliers 1e3..1e6 (each in its own
    bin; a 5e8-bin span) — exercises the sparse histogram path."""
    rng = np.random.default_rng(seed)
    d = rng.uniform(-E / 2, E / 2, n)
    k = int(round(n * frac))
    pos = rng.choice(n, size=k, replace=False)
    d[pos] = rng.uniform(1e3, 1e6, k)
    base = rng.uniform(1.0, 2.0, n)
    return base.astype(dtype), (base * (1.0 + d)).astype(dtype)


def drift_series(n: int, steps: int, seed: int = 0, dtype="f4", lo=0.002, hi=0.012):
    """Multiplicative drift chain in [1, 2) growing by U(1+lo, 1+hi) per step."""
    rng = np.random.default_rng(seed)
    dt = np.dtype(dtype)
    out = [rng.uniform(1.0, 2.0, n).astype(dt)]
    for _ in range(steps):
        f = rng.uniform(1.0 + lo, 1.0 + hi, n)
        out.append((out[-1].astype(np.float64) * f).astype(dt))
    return out
