"""Shared pytest configuration: the ``gpu`` marker, golden-fixture loading,
and an import path for the test-only oracle."""

from __future__ import annotations

import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden_names(prefix: str = "") -> list[str]:
    files = sorted(glob.glob(os.path.join(GOLDEN, f"{prefix}*.npz")))
    return [os.path.basename(f)[:-4] for f in files if not os.path.basename(f).startswith("series_")]


def load_golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def golden_blocks(g: dict) -> list[bytes]:
    """Split the concatenated pre-deflate packed stream into per-block bytes."""
    buf = g["packed"].tobytes()
    out, pos = [], 0
    for ln in g["block_lens"]:
        out.append(buf[pos:pos + int(ln)])
        pos += int(ln)
    return out


def golden_bits(g: dict):
    b = int(g["bits_in"])
    return None if b < 0 else b


@pytest.fixture
def gpu_required():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
