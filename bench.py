#!/usr/bin/env python
"""Benchmark of the NUMARCK per-timestep hot path on B200 (BASELINE.json).

Default workload (BASELINE.json configs[1], "cfg2"): one 512^3 fp64 timestep
(1 GiB) of a smooth 3-D field in 8^3-cell blocks, spatially correlated change
ratio + 2 % Laplace outliers, E = 1e-3, B = 8.  Synthetic, seeded, generated
on the device (the paper's datasets are not available).  One STEP = compress
(K1..K4) + full decompress (K5) of the timestep with inputs resident in HBM;
value = input GB/s = n*L / step time, summed over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--workload cfg2|cfg3|cfg4-weak|cfg4-strong|cfg5] [--bits B --tol E]

Workloads (BASELINE.json configs):
  cfg2         512^3 fp64 per GPU (weak scaling: an N x 512^3 global field)
  cfg3         1440x720x30 fp32 climate series per GPU; a step is one of the
               15 transitions (compress against the previous reconstruction
               + full decompress), cycling through all 15
  cfg4-weak    2^29 fp64 per GPU, config-1 distribution (weak scaling)
  cfg4-strong  4e9 fp64 in total, contiguous shards over the N GPUs (strong)
  cfg5         2^28 fp64 per GPU, bimodal + 20 % outliers, --bits/--tol

--gpus N without WORLD_SIZE re-launches itself under torch.distributed.run
with N ranks (one per GPU, NCCL); with fewer than N visible GPUs it fails.
Under torchrun each rank drives one GPU; times are CUDA events on the
launching stream, max over ranks.  Inputs are >= 124 MB per GPU per snapshot
(2 GiB for cfg2), above the 126 MB L2 once both snapshots are read, so no
flush is needed between steps.

--impl reference times the reference itself (the pure-Python package `nmk`
vendored into oracle/_ref by oracle/make_ref.py, its public compress_pair /
decompress) on the host cores, on a bounded sample of the same field.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compress+decompress GB/s of input (n*L per timestep / (t_compress + t_decompress))"
NOMINAL_HBM_GBS = 8000.0
CFG4_STRONG_N = 4_000_000_000
# kernels per compress + decompress step of the sync-free pipeline:
# k_minmax (the span decision and histogram clear fused in on one rank),
# k_hist_dev, k_select, k_encode_keyed, k_enc_finalize (chunk scan inside) |
# k_dec_count(_wide), k_chunk_scan, k_dec_chunks: 8.  More when a hint from the
# warm-up check is missing: + k_hist_prep with a communicator, + k_encode (the
# snapshot-reading fallback, exits when the keyed kernel did the work), + the
# second k_dec_chunks ring depth (exits at entry).
def gpu_launches_per_step(pipe):
    return 8 + (pipe.comm is not None) + (not pipe.keyed_hint) + (pipe.ring_hint == 0)


WORKLOADS = {
    "cfg2": dict(desc="cfg2: 512^3 fp64 8^3-block field, E=1e-3, B=8, top-k, 1 MiB index blocks",
                 E=1e-3, bits=8, L=8, scaling="weak"),
    "cfg3": dict(desc="cfg3: 1440x720x30 fp32 climate series, 15 transitions against the previous "
                      "reconstruction, E=5e-3, B=10; step = one transition (compress + full decompress)",
                 E=5e-3, bits=10, L=4, scaling="weak"),
    "cfg4-weak": dict(desc="cfg4 weak: 2^29 fp64 per GPU, config-1 distribution, E=1e-3, B=8",
                      E=1e-3, bits=8, L=8, scaling="weak"),
    "cfg4-strong": dict(desc="cfg4 strong: 4e9 fp64 in total over the N GPUs, config-1 distribution, "
                             "E=1e-3, B=8", E=1e-3, bits=8, L=8, scaling="strong"),
    "cfg5": dict(desc="cfg5: 2^28 fp64, bimodal N(-0.02,0.004)/N(0.03,0.006) + 20% U(-1,1)",
                 E=1e-3, bits=8, L=8, scaling="weak"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg2")
    ap.add_argument("--bits", type=int, default=None, help="cfg5: index bits (default 8)")
    ap.add_argument("--tol", type=float, default=None, help="cfg5: error bound E (default 1e-3)")
    ap.add_argument("--side", type=int, default=512, help="cfg2 grid side (testing)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-series-e2e", action="store_true")
    ap.add_argument("--cpu-sample-log2", type=int, default=24)
    ap.add_argument("--force-comm", action="store_true",
                    help="run the multi-GPU code path (NCCL exchanges in the graph) even with one rank (testing)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(args) -> None:
    """--gpus N (N > 1) outside torchrun: re-exec under torch.distributed.run
    with one rank per GPU.  Never silently runs fewer ranks than asked."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    if args.impl == "ours":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} requested but only {have} CUDA device(s) are visible")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, device copy)"
    return 6650.0, "fallback (B200_PROFILING.md, 6.65 TB/s)"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def workload_params(args):
    w = dict(WORKLOADS[args.workload])
    if args.workload == "cfg5":
        w["E"] = args.tol if args.tol is not None else 1e-3
        w["bits"] = args.bits if args.bits is not None else 8
        w["desc"] += f", E={w['E']:g}, B={w['bits']}"
    return w


def shard_of(args, world, rank):
    """(elem0, n_local, n_total) of this rank."""
    from paper_1703_02438_b200 import distributed as D
    if args.workload == "cfg4-strong":
        lo, hi = D.shard_bounds(CFG4_STRONG_N, world, rank, align=256)
        return lo, hi - lo, CFG4_STRONG_N
    n_local = {"cfg2": args.side ** 3, "cfg3": 30 * 720 * 1440, "cfg4-weak": 1 << 29, "cfg5": 1 << 28}[args.workload]
    return rank * n_local, n_local, n_local * world


def make_field(args, world, rank, elem0, n_local):
    """Device snapshots of this rank: a list of (base, cur) pairs (one per
    step kind) -- cfg3's bases are filled in later (the chain)."""
    from paper_1703_02438_b200 import workloads
    if args.workload == "cfg2":
        return [workloads.cfg2_device(args.side, seed=rank)]
    if args.workload == "cfg4-weak":
        return [workloads.cfg1_device(n_local, seed=4 + 1000 * rank)]
    if args.workload == "cfg4-strong":
        return [workloads.cfg1_device_range(elem0, elem0 + n_local, seed=4)]
    if args.workload == "cfg5":
        return [workloads.cfg5_device(n_local, seed=5 + 1000 * rank)]
    x = workloads.cfg3_device_first(seed=rank)
    snaps = [x]
    for t in range(1, 16):
        snaps.append(workloads.cfg3_device_step(snaps[-1], t, seed=rank))
    return snaps


# ---------------------------------------------------------------------------
# reference arm: the reference package itself on the host cores
# ---------------------------------------------------------------------------

def _load_reference():
    ref = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.exists(os.path.join(ref, "nmk", "pipeline.py")):
        return None
    sys.path.insert(0, ref)
    import nmk
    return nmk


class _InflateClock:
    """Wrap the reference's codec.decompress_block to time inflate separately
    (decode hot = decompress wall - inflate)."""

    def __init__(self, nmk):
        self.codec, self.orig, self.t = nmk.codec, nmk.codec.decompress_block, 0.0

        def timed(data, _orig=self.orig):
            t0 = time.perf_counter()
            try:
                return _orig(data)
            finally:
                self.t += time.perf_counter() - t0
        self.codec.decompress_block = timed

    def restore(self):
        self.codec.decompress_block = self.orig


def reference_once(nmk, base, cur, E, bits, workers):
    """One compress_pair + full decompress through the reference's public API.
    Returns (compress_hot_s, zlib_s, decode_hot_s, inflate_s, variable)."""
    pair = nmk.TemporalPair(base, cur)
    cfg = nmk.PipelineConfig(workers=workers, tolerance=E, bits=bits)
    var, tm = nmk.compress_pair(pair, cfg)
    hot = tm.change_ratio + tm.binning + tm.assign_index + tm.index_alignment + tm.bits_packing
    clk = _InflateClock(nmk)
    try:
        t0 = time.perf_counter()
        out = nmk.decompress(var, base)
        wall = time.perf_counter() - t0
    finally:
        clk.restore()
    assert out.shape[0] == base.shape[0]
    return hot, tm.zlib, wall - clk.t, clk.t, var


def reference_sample(args, w):
    """Host arrays the reference arm / cpu_baseline time: the same seeded
    field as the GPU arm (generated with torch on the device when one is
    present, then copied), cut to a bounded sample."""
    sample_n = 1 << args.cpu_sample_log2
    same_field = True
    try:
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device")
        elem0, n_local, _ = shard_of(args, 1, 0)
        # the GPU arm's own field (rank 0), cut to the sample; cfg4-strong's
        # chunk-seeded global field can be generated for its first elements only
        field = make_field(args, 1, 0, elem0, min(n_local, sample_n) if args.workload == "cfg4-strong" else n_local)
        if args.workload == "cfg3":
            b, c = field[0], field[1]          # transition 1 (its base is the raw first snapshot)
        else:
            b, c = field[0]
        n_full = b.numel()
        b, c = b[:sample_n].cpu().numpy(), c[:sample_n].cpu().numpy()
        del field
        torch.cuda.empty_cache()
    except Exception:   # no device: the host recipe (a different draw of the same distribution)
        from paper_1703_02438_b200 import workloads
        same_field = False
        if args.workload == "cfg2":
            b, c = workloads.cfg2_host(256, seed=0)
        elif args.workload == "cfg3":
            s = workloads.cfg3_host((30, 720, 1440), steps=2, seed=0)
            b, c = s[0], s[1]
        elif args.workload == "cfg5":
            b, c = workloads.cfg5_host(sample_n, seed=5)
        else:
            b, c = workloads.cfg1_host(sample_n, seed=4)
        n_full = b.size
        b, c = b[:sample_n], c[:sample_n]
    return np.ascontiguousarray(b), np.ascontiguousarray(c), n_full, same_field


def reference_arm(args, world, rank):
    """--impl reference: the reference package on the host cores."""
    if rank != 0:
        return
    w = workload_params(args)
    nmk = _load_reference()
    if nmk is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not vendored (oracle/make_ref.py)"}))
        return
    cores = os.cpu_count() or 1
    b, c, n_full, same_field = reference_sample(args, w)
    n, L = b.size, b.dtype.itemsize
    times = []
    for i in range(args.warmup + args.steps):
        hot, z, dec, infl, _ = reference_once(nmk, b, c, w["E"], w["bits"], cores)
        if i >= args.warmup:
            times.append((hot, z, dec, infl))
    hot = sum(t[0] for t in times) / len(times)
    dec = sum(t[2] for t in times) / len(times)
    gbs = n * L / (hot + dec) / 1e9
    h1, _, d1, _, _ = reference_once(nmk, b, c, w["E"], w["bits"], 1)
    extra = {}
    if args.workload == "cfg2" and same_field and args.side == 512:
        # one full-size 512^3 run for the record (not the timed steps)
        import torch
        from paper_1703_02438_b200 import workloads
        fb, fc = workloads.cfg2_device(512, seed=0)
        fb, fc = fb.cpu().numpy(), fc.cpu().numpy()
        torch.cuda.empty_cache()
        fh, fz, fd, fi, _ = reference_once(nmk, fb, fc, w["E"], w["bits"], cores)
        extra["full_size_once"] = {"n": fb.size, "compress_hot_s": fh, "zlib_s": fz, "decode_hot_s": fd,
                                   "inflate_s": fi, "gbs": fb.size * 8 / (fh + fd) / 1e9, "workers": cores}
    sample = (f"first {n} elements of the {w['desc'].split(':')[0]} field (full: {n_full}), "
              f"compress_pair + full decompress through the reference's public API, workers={cores}, "
              f"hot phases only (PhaseTimings change_ratio..bits_packing; decompress minus inflate)")
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": (hot + dec) * 1e3, "higher_is_better": True,
        "scaling": w["scaling"], "vs_baseline": None, "dtype": "f64" if L == 8 else "f32",
        "data": "synthetic (seeded, same generator and seed as the GPU arm)" if same_field else
                "synthetic (host recipe; no CUDA device to regenerate the GPU arm's field)",
        "config": {"workload": w["desc"]},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "reference", "sample": sample,
                         "cpu_model": cpu_model(), "workers_1_gbs": n * L / (h1 + d1) / 1e9,
                         "compress_hot_gbs": n * L / hot / 1e9, "decode_hot_gbs": n * L / dec / 1e9,
                         "zlib_s_per_step": sum(t[1] for t in times) / len(times),
                         "inflate_s_per_step": sum(t[3] for t in times) / len(times)},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        **extra,
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(args, w, base_dev, cur_dev):
    """The reference (oracle/_ref; else the oracle port) on a bounded slice of
    this rank's field, on the host cores (rank 0, N = 1)."""
    n = min(1 << args.cpu_sample_log2, base_dev.numel())
    b = base_dev[:n].cpu().numpy()
    c = cur_dev[:n].cpu().numpy()
    cores = os.cpu_count() or 1
    L = b.dtype.itemsize
    nmk = _load_reference()
    if nmk is not None:
        best = None
        for _ in range(2):
            hot, _, dec, _, _ = reference_once(nmk, b, c, w["E"], w["bits"], cores)
            best = hot + dec if best is None else min(best, hot + dec)
        return {"value": n * L / best / 1e9, "unit": "GB/s", "cores": cores, "kind": "reference",
                "cpu_model": cpu_model(),
                "sample": f"first {n} elements of this rank's field, reference compress_pair + decompress "
                          f"(hot phases), workers={cores}, best of 2"}
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import nmk_oracle as O
    best = None
    for _ in range(2):
        t0 = time.perf_counter()
        enc = O.encode(b, c, w["E"], w["bits"], 1 << 20, workers=cores)
        O.decode(enc, b)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return {"value": n * L / best / 1e9, "unit": "GB/s", "cores": cores, "kind": "port", "cpu_model": cpu_model(),
            "sample": f"first {n} elements of this rank's field, numpy oracle port, {cores} workers, best of 2"}


# ---------------------------------------------------------------------------
# roofline arithmetic
# ---------------------------------------------------------------------------

def roofline_report(mean, ms_step, n, L, bits, alpha, nchunks, peak, peak_src, traffic_map):
    """Per kernel: the bytes this design must move (compulsory for its data
    layout), the SURVEY §8(d) three-pass algorithmic bytes for reference, and
    fractions of the measured and the nominal HBM peak.  The step is also
    set against the single-pass compulsory bound of compress + decompress,
    4L + 2B/8 + 2aL bytes per element."""
    Bb = bits / 8.0
    per = {
        # K1 reads both snapshots and writes a 4-byte ratio key per element
        "K1_minmax": (2 * L + 4, 2 * L, "k_minmax"),
        # K2 reads the keys
        "K2_histogram": (4.0, 2 * L, "k_hist_dev"),
        # K4 reads the keys, writes the codes, gathers + writes the exact
        # values, writes a 256-bit sentinel mask and a 4-byte count per chunk
        # (read back once by the finalize kernel, which scans them in place)
        "K4_encode": (4 + Bb + 2 * alpha * L + (32 + 8) * nchunks / n, 2 * L + Bb + alpha * L, "k_encode_keyed"),
        # K5 reads the codes twice (count pass + decode), base, exact; writes out
        "K5_decode": (2 * L + 2 * Bb + alpha * L, 2 * L + Bb + alpha * L, "k_dec_chunks"),
    }
    out = {}
    for ph, (design, survey, kern) in per.items():
        if ph not in mean:
            continue
        sec = mean[ph] / 1e3
        gbs = design * n / sec / 1e9
        out[ph] = {"kernel": kern, "ms": mean[ph], "bytes": design * n, "bytes_per_elem": design,
                   "gbs": gbs, "frac": gbs / peak, "frac_nominal": gbs / NOMINAL_HBM_GBS,
                   "survey_alg_bytes": survey * n, "traffic": traffic_map.get(kern)}
    if "K3_select" in mean:
        out["K3_select"] = {"ms": mean["K3_select"], "note": "single CTA over the histogram (latency-bound)"}
    design_step = sum(v[0] for v in per.values())
    single_pass = 4 * L + 2 * Bb + 2 * alpha * L
    sec = ms_step / 1e3
    out["step"] = {
        "ms": ms_step, "bytes_per_elem": design_step,
        "frac": design_step * n / sec / 1e9 / peak,
        "single_pass_bytes_per_elem": single_pass,
        "single_pass_frac": single_pass * n / sec / 1e9 / peak,
        "single_pass_frac_nominal": single_pass * n / sec / 1e9 / NOMINAL_HBM_GBS,
        "survey_three_pass_bytes_per_elem": 8 * L + 2 * Bb + 2 * alpha * L,
        "note": "graph-replayed step; single pass = compress 2L+B/8+aL + decompress 2L+B/8+aL"}
    out["peak"] = {"gbs": peak, "source": peak_src, "nominal_gbs": NOMINAL_HBM_GBS}
    dom = max((k for k in ("K1_minmax", "K2_histogram", "K4_encode", "K5_decode") if k in out),
              key=lambda k: out[k]["ms"])
    d = out[dom]
    headline = {"bound": "hbm", "kernel": f"{d['kernel']} ({dom.split('_')[0]}, the longest phase)",
                "achieved": d["gbs"], "peak": peak, "unit": "GB/s", "frac": d["frac"],
                "frac_nominal": d["frac_nominal"], "traffic": d["traffic"],
                "bytes_per_launch": d["bytes"],
                "bytes_basis": "compulsory bytes of this kernel in this design (DESIGN.md §3)",
                "survey_alg_bytes_per_launch": d["survey_alg_bytes"],
                "survey_alg_frac": d["survey_alg_bytes"] / (d["ms"] / 1e3) / 1e9 / peak,
                "peak_source": peak_src}
    return headline, out


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def main():
    args = parse()
    self_launch(args)
    world, rank, local = dist_env()
    if args.impl == "reference":
        if world > 1 and world != args.gpus:
            sys.exit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
        reference_arm(args, max(world, args.gpus), rank)
        return
    if world != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}: refusing to report a different N")
    import torch
    import torch.distributed as dist
    from paper_1703_02438_b200 import distributed as D, engine, pipeline

    if torch.cuda.device_count() < 1:
        sys.exit("bench.py: no CUDA device")
    torch.cuda.set_device(local)
    comm = None
    if world > 1 or args.force_comm:
        if not dist.is_initialized():
            if world == 1 and "MASTER_ADDR" not in os.environ:
                os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0", WORLD_SIZE="1")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = D.ProcessGroupComm()
    w = workload_params(args)
    E, bits, L = w["E"], w["bits"], w["L"]
    elem0, n_local, n_total = shard_of(args, world, rank)
    field = make_field(args, world, rank, elem0, n_local)
    dtype = field[0][0].dtype if args.workload != "cfg3" else field[0].dtype
    pipe = engine.DevicePipeline(n_local, dtype, E, bits, 1 << 20, elem0=elem0, n_total=n_total, comm=comm)
    out = torch.empty(n_local, dtype=dtype, device="cuda")
    if args.workload == "cfg3":
        # the chain: the base of transition t is the reconstruction of t-1 (untimed set-up)
        snaps = field
        bases = [snaps[0].clone()]
        for t in range(1, 16):
            nxt = torch.empty_like(snaps[0])
            pipe.encode(bases[-1], snaps[t], recon=nxt)
            bases.append(nxt)
        pairs = [(bases[t - 1], snaps[t]) for t in range(1, 16)]
        del bases[-1]
    else:
        pairs = field
    torch.cuda.synchronize()
    # warm-up, and the span of the exchanged histogram sized from it
    for i in range(max(args.warmup, 1)):
        b, c = pairs[i % len(pairs)]
        pipe.step(b, c, out)
    chk = pipe.check()
    assert chk["status"] == 0 and not chk["bad_index"] and not chk["exhausted"], chk
    assert chk["n_sentinel"] == chk["n_inc"] and chk["tripwire"] == 0, chk
    if comm is not None:
        spans = [chk["nbins"]]
        for b, c in pairs[1:]:
            pipe.step(b, c, out)
            spans.append(pipe.check()["nbins"])
        pipe.fit_comm_bins(max(spans))
    graphs = []
    launches_per_step = gpu_launches_per_step(pipe)   # the hints the captures below are made with
    try:
        for b, c in pairs:
            graphs.append(pipe.capture(b, c, out))
    except Exception as exc:   # pragma: no cover - capture unsupported: eager launches
        print(f"graph capture failed ({exc}); timing eager launches", file=sys.stderr)
        graphs = []

    def step(i):
        if graphs:
            graphs[i % len(graphs)].replay()
        else:
            b, c = pairs[i % len(pairs)]
            pipe.step(b, c, out)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    if comm:
        dist.barrier()
    stream = torch.cuda.current_stream()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.1)
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if comm:
        dist.barrier()
    t_start.record(stream)
    for i in range(args.steps):
        step(i)
    t_end.record(stream)
    torch.cuda.synchronize()
    if comm:
        dist.barrier()
    clk = clocks.stop()
    elapsed_ms = t_start.elapsed_time(t_end)
    if comm:
        t = torch.tensor([elapsed_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    ms_step = elapsed_ms / args.steps
    value = n_total * L / (ms_step / 1e3) / 1e9

    # correctness guard on the timed buffers (outside the timed region)
    chk = pipe.check()
    assert chk["status"] == 0 and not chk["bad_index"] and not chk["exhausted"], chk
    assert chk["n_sentinel"] == chk["n_inc"], chk

    # per-phase device times: an instrumented eager pass over the same steps
    phases, alphas = {}, []
    for i in range(max(args.steps, 3)):
        b, c = pairs[i % len(pairs)]
        evs = [("start", torch.cuda.Event(enable_timing=True))]
        evs[0][1].record(stream)

        def mark(name, evs=evs):
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            evs.append((name, e))

        pipe.step(b, c, out, mark=mark)
        torch.cuda.synchronize()
        alphas.append(pipe.check()["n_inc"] / n_local)
        for (_, e0), (nm, e1) in zip(evs[:-1], evs[1:]):
            phases.setdefault(nm, []).append(e0.elapsed_time(e1))
    mean = {k: sum(v) / len(v) for k, v in phases.items()}
    alpha = sum(alphas) / len(alphas)
    peak, peak_src = peaks()
    traffic_map = {}
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if args.workload == "cfg2" and args.side == 512 and os.path.exists(tp):
        with open(tp) as f:
            traffic_map = json.load(f).get("dram_bytes_per_launch", {})
    nchunks = -(-n_local // 256)
    roofline, roof_all = roofline_report(mean, ms_step, n_local, L, bits, alpha, nchunks, peak, peak_src,
                                         traffic_map)
    roof_all["timing"] = (f"phase times: CUDA events between phases on the launch stream, mean of "
                          f"{max(args.steps, 3)} eager steps after the timed graph replays")
    compress_ms = sum(mean[k] for k in ("K1_minmax", "K2_histogram", "K3_select", "K4_encode"))

    e2e = None
    if not args.no_e2e and args.workload != "cfg4-strong":
        cfg = pipeline.PipelineConfig(tolerance=E, bits=bits, block_bytes=1 << 20)
        e2e = e2e_series(args, cfg, pairs, n_local, L, comm, world) if args.workload == "cfg3" else \
            e2e_pairs(args, cfg, pairs[0], n_local, L, elem0, n_total, comm, chk)
    elif args.workload == "cfg4-strong":
        e2e = {"value": None, "unit": "GB/s", "h2d_bytes_per_step": None, "d2h_bytes_per_step": None,
               "skipped": "4e9-element host staging (64 GB pinned per pair) not attempted; see cfg2/cfg4-weak e2e"}
    series = None
    if (rank == 0 and world == 1 and args.workload == "cfg2" and not args.no_series_e2e and not args.no_e2e):
        series = series_e2e_cfg3(pipeline)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, w, pairs[0][0], pairs[0][1])

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": w["scaling"],
            "vs_baseline": None, "dtype": "f64" if L == 8 else "f32",
            "data": "synthetic (seeded BASELINE recipe, generated on device)",
            "config": {"workload": w["desc"], "n_per_gpu": n_local, "n_total": n_total,
                       "parallelism": f"dp{world} (contiguous element shards)",
                       "l2": f"inputs {2 * n_local * L / 2**20:.0f} MiB per GPU per step > 126 MB L2 (no flush needed)",
                       "k": chk["k"], "alpha": alpha, "hist_form": "dense",
                       "hist_allreduce_bins": pipe.cap_bins + 1 if comm else None,
                       "execution": "sync-free device pipeline" + (" replayed as CUDA graphs" if graphs else "")},
            "compress": {"ms": compress_ms, "gbs_per_gpu": n_local * L / (compress_ms / 1e3) / 1e9},
            "decompress": {"ms": mean["K5_decode"], "gbs_per_gpu": n_local * L / (mean["K5_decode"] / 1e3) / 1e9},
            "phase_ms": mean,
            "roofline": roofline,
            "roofline_all": roof_all,
            "e2e": e2e,
            "series_e2e": series,
            "gpu_launches": launches_per_step * args.steps,
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if comm:
        dist.barrier()
        dist.destroy_process_group()


def e2e_pairs(args, cfg, pair, n_local, L, elem0, n_total, comm, chk):
    """Same metric end to end through the host-buffer API: pinned host
    snapshot pair in, compressed stream + reconstruction out, H2D / kernels /
    D2H of consecutive steps overlapped (pipeline.StreamCompressor)."""
    import torch
    import torch.distributed as dist
    from paper_1703_02438_b200 import pipeline
    base, cur = pair
    hb = torch.empty(n_local, dtype=base.dtype, pin_memory=True)
    hc = torch.empty(n_local, dtype=base.dtype, pin_memory=True)
    hb.copy_(base)
    hc.copy_(cur)
    depth = 3
    sc = pipeline.StreamCompressor(n_local, np.float64 if L == 8 else np.float32, cfg, depth=depth, elem0=elem0,
                                   n_total=n_total, comm=comm)
    for _ in range(2):
        sc.result(sc.submit(hb, hc))
    if comm:
        dist.barrier()
    reps = max(args.steps, 8)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pending, d2h_total = [], 0
    for i in range(reps + depth):
        if len(pending) == depth or (i >= reps and pending):
            h, rec = sc.result(pending.pop(0))
            d2h_total += sc.last_d2h_bytes
        if i < reps:
            pending.append(sc.submit(hb, hc))
    dt = (time.perf_counter() - t0) / reps
    assert h.n_inc == chk["n_inc"] and rec.shape[0] == n_local
    if comm:
        t = torch.tensor([dt], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    del sc
    torch.cuda.empty_cache()
    return {"value": n_total * L / dt / 1e9, "unit": "GB/s",
            "h2d_bytes_per_step": int(2 * n_local * L), "d2h_bytes_per_step": int(d2h_total // reps),
            "path": "pipeline.StreamCompressor: pinned host pair -> compress + full decompress -> host "
                    "(packed stream, exact values, prefix, centers, reconstruction); zlib excluded; "
                    "copies of consecutive steps overlapped on separate streams",
            "wall_clock": "perf_counter over all steps incl. every H2D/D2H"}


def _series_run(pipeline, cfg, snaps_h, n, dtype, reps):
    """compress_series from host snapshots where only x_t crosses PCIe
    (pipeline.SeriesStreamCompressor); returns (s per step, d2h bytes/step)."""
    import torch
    sc = pipeline.SeriesStreamCompressor(n, dtype, cfg, depth=2)
    sc.start(snaps_h[0])
    for t in range(1, len(snaps_h)):
        sc.result(sc.submit(snaps_h[t]))
    sc.start(snaps_h[0])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pending, d2h, done = [], 0, 0
    i = 0
    while done < reps:
        if i < reps:
            t = 1 + i % (len(snaps_h) - 1)
            if t == 1 and i > 0:           # restart the chain: drain first
                while pending:
                    sc.result(pending.pop(0))
                    d2h += sc.last_d2h_bytes
                    done += 1
                sc.start(snaps_h[0])
            pending.append(sc.submit(snaps_h[t]))
            i += 1
        if len(pending) == 2 or (i >= reps and pending):
            sc.result(pending.pop(0))
            d2h += sc.last_d2h_bytes
            done += 1
    dt = (time.perf_counter() - t0) / reps
    return dt, d2h / reps, sc.h2d_bytes()


def e2e_series(args, cfg, pairs, n_local, L, comm, world):
    """cfg3's e2e: only x_t crosses PCIe; the base stays resident."""
    import torch
    from paper_1703_02438_b200 import pipeline
    snaps_h = [pairs[0][0].cpu().pin_memory()] + [c.cpu().pin_memory() for _, c in pairs]
    dt, d2h, h2d = _series_run(pipeline, cfg, snaps_h, n_local, np.float32, max(args.steps, 15))
    torch.cuda.empty_cache()
    return {"value": n_local * L * world / dt / 1e9, "unit": "GB/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h),
            "path": "pipeline.SeriesStreamCompressor: pinned host x_t -> compress against the resident "
                    "reconstruction (K4's fused recon) -> packed stream, exact values, prefix, centers to host; "
                    "zlib excluded", "wall_clock": "perf_counter over all steps incl. every H2D/D2H"}


def series_e2e_cfg3(pipeline):
    """The default run's series-mode e2e line: cfg3 (1440x720x30 fp32, 15
    transitions) through SeriesStreamCompressor; only x_t crosses PCIe."""
    import torch
    from paper_1703_02438_b200 import workloads
    x = workloads.cfg3_device_first(seed=0)
    snaps = [x.cpu().pin_memory()]
    for t in range(1, 16):
        x = workloads.cfg3_device_step(x, t, seed=0)
        snaps.append(x.cpu().pin_memory())
    n = x.numel()
    del x
    torch.cuda.empty_cache()
    cfg = pipeline.PipelineConfig(tolerance=5e-3, bits=10, block_bytes=1 << 20)
    dt, d2h, h2d = _series_run(pipeline, cfg, snaps, n, np.float32, 30)
    return {"workload": WORKLOADS["cfg3"]["desc"].split("; step")[0], "metric": "compress GB/s of input per "
            "transition, host x_t in -> compressed stream out", "value": n * 4 / dt / 1e9, "unit": "GB/s",
            "ms_per_step": dt * 1e3, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "path": "pipeline.SeriesStreamCompressor (compress_series without the per-step decode; the "
                    "reconstruction stays in HBM)"}


if __name__ == "__main__":
    main()
