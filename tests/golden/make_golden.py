"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package from /root/reference/pkg/src (read-only),
compresses a set of seeded inputs through ``nmk.compress_pair`` /
``nmk.compress_series`` / ``nmk.decompress`` and stores inputs plus every
observable output in ``tests/golden/*.npz``:

* phase-1/2 intermediates from the reference's own functions
  (``core.compute_change_ratios`` -> gmin/gmax, ``binning.build_histogram``),
* the CompressedVariable fields (bits, centers, epb, nblocks, n_inc, prefix,
  incompressible table),
* the pre-deflate packed index blocks (inflated back from the reference's
  index table with ``codec.decompress_block``),
* full and range decodes, and the SHA-256 of the ``.nmk`` file.

Nothing on the GPU box reads /root/reference; the tests use these files.
"""

from __future__ import annotations

import hashlib
import importlib.util
import io
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from nmk import binning, codec, container, core, pipeline  # noqa: E402

_spec = importlib.util.spec_from_file_location(
    "workloads", os.path.join(HERE, "..", "..", "paper_1703_02438_b200", "workloads.py"))
W = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(W)


def run_case(name, base, cur, E=1e-3, bits=None, block_bytes=1 << 20, ranges=()):
    base = np.ascontiguousarray(base)
    cur = np.ascontiguousarray(cur)
    pair = core.TemporalPair(base, cur)
    cfg = pipeline.PipelineConfig(tolerance=E, bits=bits, block_bytes=block_bytes)
    var, _ = pipeline.compress_pair(pair, cfg, name="v")
    rec = {
        "base": base, "cur": cur, "E": np.float64(E),
        "bits_in": np.int64(-1 if bits is None else bits),
        "block_bytes": np.int64(block_bytes),
        "bits": np.int64(var.bits), "centers": var.centers,
        "epb": np.int64(var.elements_per_block), "nblocks": np.int64(var.nblocks),
        "n_inc": np.int64(var.n_incompressible),
        "prefix": var.incompressible_prefix.astype(np.uint64),
        "exact": var.incompressible_table,
    }
    try:
        field = core.compute_change_ratios(pair)
        hist = binning.build_histogram(field, core.Tolerance(E))
        rec.update(gmin=np.float64(field.min_ratio), gmax=np.float64(field.max_ratio),
                   nvalid=np.int64(field.valid.sum()),
                   hist_keys=hist.ordinals, hist_counts=hist.counts)
    except ValueError:  # degenerate: no valid ratio
        rec.update(gmin=np.float64(np.nan), gmax=np.float64(np.nan), nvalid=np.int64(0),
                   hist_keys=np.zeros(0), hist_counts=np.zeros(0, dtype=np.int64))
    blocks = [codec.decompress_block(codec._block_bytes_of(var, b)) for b in range(var.nblocks)]
    rec["block_lens"] = np.array([len(b) for b in blocks], dtype=np.int64)
    rec["packed"] = np.frombuffer(b"".join(blocks), dtype=np.uint8)
    rec["decoded"] = pipeline.decompress(var, base)
    rs, outs = [], []
    for (s, c) in ranges:
        rs.append((s, c))
        outs.append(pipeline.decompress(var, base[s:s + c], rng=(s, c)))
    rec["ranges"] = np.array(rs, dtype=np.int64).reshape(-1, 2)
    rec["range_out"] = np.concatenate(outs) if outs else np.zeros(0, dtype=base.dtype)
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "v.nmk")
        container.write_file(p, [var])
        rec["nmk_sha256"] = np.array(hashlib.sha256(open(p, "rb").read()).hexdigest())
    rec["deflate_level"] = np.int64(cfg.deflate_level)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **rec)
    sent = (1 << var.bits) - 1
    print(f"{name}: n={base.size} {base.dtype} bits={var.bits} k={var.k} epb={var.elements_per_block} "
          f"nblocks={var.nblocks} n_inc={var.n_incompressible} sentinel={sent}")


def series_case(name, snaps, E=1e-3, bits=None, block_bytes=1 << 20):
    cfg = pipeline.PipelineConfig(tolerance=E, bits=bits, block_bytes=block_bytes)
    first, variables = pipeline.compress_series(snaps, cfg, name="s")
    rec = {"E": np.float64(E), "bits_in": np.int64(-1 if bits is None else bits),
           "block_bytes": np.int64(block_bytes), "nsteps": np.int64(len(snaps))}
    for i, s in enumerate(snaps):
        rec[f"snap{i}"] = s
    recon = first
    for i, v in enumerate(variables, start=1):
        recon = pipeline.decompress(v, recon)
        rec[f"recon{i}"] = recon
        rec[f"bits{i}"] = np.int64(v.bits)
        rec[f"centers{i}"] = v.centers
        rec[f"n_inc{i}"] = np.int64(v.n_incompressible)
        rec[f"exact{i}"] = v.incompressible_table
        blocks = [codec.decompress_block(codec._block_bytes_of(v, b)) for b in range(v.nblocks)]
        rec[f"packed{i}"] = np.frombuffer(b"".join(blocks), dtype=np.uint8)
        with tempfile.TemporaryDirectory() as td:
            p = os.path.join(td, "s.nmk")
            container.write_file(p, [v])
            rec[f"sha{i}"] = np.array(hashlib.sha256(open(p, "rb").read()).hexdigest())
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **rec)
    print(f"{name}: {len(snaps)} snapshots of n={snaps[0].size}")


def main():
    b, c = W.cfg1_host(1 << 14, seed=0)
    run_case("cfg1_small", b, c, E=1e-3, bits=8,
             ranges=[(0, 100), (5000, 3000), (16000, 384), (0, 1 << 14), (7, 0)])
    b, c = W.cfg1_host(1 << 15, seed=1)
    run_case("cfg1_blocks", b, c, E=1e-3, bits=8, block_bytes=4096,
             ranges=[(4000, 200), (4095, 2), (0, 1 << 15), (12345, 9000)])
    b, c = W.uniform_pair(20000, seed=3, dtype=np.float32, spread=0.02)
    run_case("f32_b10_blocks", b, c, E=1e-3, bits=10, block_bytes=4096,
             ranges=[(3270, 20), (3276, 3276), (19999, 1), (100, 15000)])
    b, c = W.uniform_pair(5000, seed=0, dtype=np.float32)
    run_case("f32_auto_bits", b, c, E=1e-3, bits=None)
    b, c = W.uniform_pair(20000, seed=71, dtype=np.float64, spread=0.5)
    run_case("f64_auto_bits_smeared", b, c, E=1e-3, bits=None)
    b, c = W.outlier_pair(20000, seed=11)
    run_case("planted_outliers_b2", b, c, E=1e-3, bits=2)
    b = np.array([1.0, 2.0, np.nan, np.inf, 1.0, 0.0], dtype=np.float32)
    c = np.array([1.001, np.nan, 5.0, 2.0, np.inf, 3.0], dtype=np.float32)
    run_case("nonfinite_f32", b, c)
    run_case("degenerate_all_invalid", np.zeros(100), np.ones(100))
    run_case("degenerate_b5", np.zeros(77, dtype=np.float32), np.full(77, 2.0, dtype=np.float32), bits=5)
    rng = np.random.default_rng(20260808)
    for i in range(8):
        dt = np.float32 if i % 2 == 0 else np.float64
        b, c = W.wild_pair(rng, dt)
        run_case(f"wild_{i}_{np.dtype(dt).name}", b, c, E=1e-3, bits=None)
    b, c = W.cfg5_host(1 << 14, seed=5)
    run_case("cfg5_b12_e1e-4", b, c, E=1e-4, bits=12, block_bytes=8192,
             ranges=[(0, 5461), (5460, 2), (10000, 6384)])
    run_case("cfg5_b16_e1e-4", b, c, E=1e-4, bits=16)
    run_case("cfg5_b3_e1e-2", b, c, E=1e-2, bits=3, block_bytes=4096,
             ranges=[(10921, 3), (1, 16000)])
    b, c = W.uniform_pair(1 << 16, seed=9, dtype=np.float32, spread=0.05)
    run_case("f32_edge_rejects", b, c, E=1e-3, bits=8)
    b, c = W.cfg2_host(32, seed=2)
    run_case("cfg2_small", b, c, E=1e-3, bits=8)
    snaps = W.cfg3_host(shape=(3, 24, 48), steps=4, seed=3)
    run_case("cfg3_small_step", snaps[0], snaps[1], E=5e-3, bits=10)
    series_case("series_drift_f32", W.drift_series(3000, 3, seed=47, dtype="f4"), E=1e-3)
    series_case("series_cfg3_b10", snaps, E=5e-3, bits=10)


if __name__ == "__main__":
    main()
