#!/usr/bin/env python
"""Benchmark of the NUMARCK per-timestep hot path on B200 (BASELINE.json).

Workload (BASELINE.json configs[1], "cfg2"): one 512^3 fp64 timestep (1 GiB)
of a smooth 3-D field in 8^3-cell blocks, spatially correlated change ratio
+ 2 % Laplace outliers, E = 1e-3, B = 8.  Synthetic, seeded, generated on the
device.  One STEP = compress (K1..K4) + full decompress (K5) of the timestep
with inputs resident in HBM; value = input GB/s = n*L / step time, summed
over ranks (weak scaling: every rank owns its own 512^3 shard of an N x
512^3 global field and the three collectives run between the phases).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Under torchrun (N > 1) each rank drives one GPU over NCCL; times are CUDA
events on the launching stream, max over ranks.  Inputs (2 GiB / rank) are
larger than the 126 MB L2, so no flush is needed between steps.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

E = 1e-3
BITS = 8
SIDE = 512
METRIC = "compress+decompress GB/s of input (n*L per timestep / (t_compress + t_decompress))"
CONFIG_NAME = "cfg2: 512^3 fp64 8^3-block field, E=1e-3, B=8, top-k, 1 MiB index blocks"
# k_minmax, k_hist_prep, k_hist_dev, k_select, k_encode_keyed, k_encode (exits when the
# keyed kernel did the work), k_chunk_scan, k_enc_finalize, k_dec_count_wide, k_chunk_scan,
# k_dec_chunks x 2 (six- and five-stage rings; the one whose exact-value regime does not match
# exits at entry)
GPU_LAUNCHES_PER_STEP = 12   # K1, prep, K2, K3, K4 keyed + fallback, scan, finalize | count, scan, K5 x 2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--side", type=int, default=SIDE)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample-log2", type=int, default=24)
    ap.add_argument("--force-comm", action="store_true",
                    help="run the multi-GPU code path (NCCL exchanges, no graph) even with one rank (testing)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md, 6.65 TB/s)"


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
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
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


def reference_arm(args, world, rank):
    """--impl reference: the reference's CPU algorithm (oracle port, numpy,
    threaded over all host cores) on a bounded sample of the same workload."""
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import nmk_oracle as O
    from paper_1703_02438_b200 import workloads
    side = 256
    base, cur = workloads.cfg2_host(side, seed=0)
    n = base.size
    cores = os.cpu_count() or 1
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        enc = O.encode(base, cur, E, BITS, 1 << 20, workers=cores)
        out = O.decode(enc, base)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    assert out.shape[0] == n
    t = sum(times) / len(times)
    gbs = n * 8 / t / 1e9
    sample = f"cfg2 recipe at {side}^3 fp64 ({n} elements) per step, compress+full decompress, workers={cores}"
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded cfg2 recipe)",
        "config": {"workload": CONFIG_NAME, "n_per_step": n, "sample": f"{side}^3"},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(base_dev, cur_dev, log2n: int):
    """Oracle port on a bounded slice of this rank's field (host cores)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import nmk_oracle as O
    n = min(1 << log2n, base_dev.numel())
    b = base_dev[:n].cpu().numpy()
    c = cur_dev[:n].cpu().numpy()
    cores = os.cpu_count() or 1
    O.encode(b[: 1 << 16], c[: 1 << 16], E, BITS, workers=cores)  # warm the pool/imports
    best = None
    for _ in range(2):
        t0 = time.perf_counter()
        enc = O.encode(b, c, E, BITS, 1 << 20, workers=cores)
        O.decode(enc, b)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return {"value": n * 8 / best / 1e9, "unit": "GB/s", "cores": cores, "kind": "port",
            "sample": f"first {n} elements of the 512^3 cfg2 field, compress+full decompress, "
                      f"numpy oracle with {cores} worker threads, best of 2"}


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        reference_arm(args, world, rank)
        return
    import torch
    import torch.distributed as dist
    from paper_1703_02438_b200 import distributed as D, engine, pipeline, workloads

    torch.cuda.set_device(local)
    comm = None
    if world > 1 or args.force_comm:
        if not dist.is_initialized():
            if world == 1 and "MASTER_ADDR" not in os.environ:
                os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29500 + os.getpid() % 1000),
                                  RANK="0", WORLD_SIZE="1")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = D.ProcessGroupComm()
    n_local = args.side ** 3
    n_total = n_local * world
    elem0 = rank * n_local
    base, cur = workloads.cfg2_device(args.side, seed=rank)
    out = torch.empty_like(base)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    # sync-free compress + decompress of this rank's shard (engine.DevicePipeline)
    pipe = engine.DevicePipeline(n_local, base.dtype, E, BITS, 1 << 20, elem0=elem0, n_total=n_total, comm=comm)
    for _ in range(args.warmup):
        pipe.step(base, cur, out)
    chk = pipe.check()
    assert chk["status"] == 0 and not chk["bad_index"] and not chk["exhausted"], chk
    assert chk["n_sentinel"] == chk["n_inc"] and chk["tripwire"] == 0, chk
    # one CUDA graph per step, the NCCL exchanges captured with the kernels
    try:
        graph = pipe.capture(base, cur, out)
    except Exception as exc:   # pragma: no cover - capture unsupported: eager launches
        print(f"graph capture failed ({exc}); timing eager launches", file=sys.stderr)
        graph = None
    use_graph = graph is not None

    def step():
        if graph is not None:
            graph.replay()
        else:
            pipe.step(base, cur, out)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if comm:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if comm:
        dist.barrier()
    t_start.record(stream)
    for _ in range(args.steps):
        step()
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
    L = 8
    value = n_total * L / (ms_step / 1e3) / 1e9

    # correctness guard on the timed buffers (outside the timed region)
    chk = pipe.check()
    assert chk["status"] == 0 and not chk["bad_index"] and not chk["exhausted"], chk
    assert chk["n_sentinel"] == chk["n_inc"], chk

    # per-phase device times: a separate instrumented pass (events between phases)
    phases = {}
    for _ in range(max(args.steps, 3)):
        evs = [("start", torch.cuda.Event(enable_timing=True))]
        evs[0][1].record(stream)

        def mark(name, evs=evs):
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            evs.append((name, e))

        pipe.step(base, cur, out, mark=mark)
        torch.cuda.synchronize()
        for (_, e0), (nm, e1) in zip(evs[:-1], evs[1:]):
            phases.setdefault(nm, []).append(e0.elapsed_time(e1))
    mean = {k: sum(v) / len(v) for k, v in phases.items()}

    # roofline arithmetic per phase.  alg = SURVEY.md 8(d) algorithmic bytes
    # (the reference's three-pass schedule); moved = what this design reads
    # and writes: K1 also writes 4-byte ratio keys, so K2 and K4 read 4 B per
    # element instead of 2L (K4: + packed codes, the incompressible values
    # gathered and written, chunk counts/offsets); K5 adds the B/8
    # sentinel-count pass.
    n_inc, nb_local = chk["n_inc"], pipe.prefix.numel()
    pk = n_local * BITS / 8
    nchunks = -(-n_local // 256)
    rf = {
        "K1_minmax": (2 * L * n_local, 2 * L * n_local + 4 * n_local, "k_minmax"),
        "K2_histogram": (2 * L * n_local, 4 * n_local, "k_hist_dev"),
        "K4_encode": (2 * L * n_local + pk + n_inc * L + 8 * nb_local,
                      4 * n_local + pk + 2 * n_inc * L + 16 * nchunks + 8 * nb_local, "k_encode_keyed"),
        "K5_decode": (2 * L * n_local + pk + n_inc * L, 2 * L * n_local + 2 * pk + n_inc * L, "k_dec_chunks"),
    }
    peak, peak_src = peaks()
    traffic_map = {}
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic_map = json.load(f).get("dram_bytes_per_launch", {})
    roof_all = {}
    for ph, (alg, moved, kern) in rf.items():
        sec = mean[ph] / 1e3
        roof_all[ph] = {"kernel": kern, "ms": mean[ph], "alg_bytes": alg, "moved_bytes": moved,
                        "gbs": alg / sec / 1e9, "frac": alg / sec / 1e9 / peak,
                        "moved_gbs": moved / sec / 1e9, "moved_frac": moved / sec / 1e9 / peak}
    roof_all["K3_select"] = {"ms": mean["K3_select"], "note": "single CTA over the histogram (latency-bound)"}
    roof_all["K4_encode"]["note"] = "includes the chunk-count scan and the finalize pass"
    roof_all["K5_decode"]["note"] = "includes the sentinel-count pass (+B/8 bytes/element) and its scan"
    step_alg = sum(v[0] for v in rf.values())
    step_moved = sum(v[1] for v in rf.values())
    roof_all["step"] = {"alg_bytes": step_alg, "moved_bytes": step_moved, "ms": ms_step,
                        "frac": step_alg / (ms_step / 1e3) / 1e9 / peak,
                        "moved_frac": step_moved / (ms_step / 1e3) / 1e9 / peak,
                        "note": "graph-replayed step; alg = SURVEY 8(d) compress 6L+B/8+aL + decompress 2L+B/8+aL"}
    roof_all["timing"] = (f"phase times: CUDA events between phases on the launch stream, mean of "
                          f"{max(args.steps, 3)} eager steps after the timed steps")
    dom = max(("K1_minmax", "K2_histogram", "K4_encode", "K5_decode"), key=lambda k: mean[k])
    d = roof_all[dom]
    roofline = {"bound": "hbm", "kernel": f"{d['kernel']} ({dom.split('_')[0]}, the longest phase)",
                "achieved": d["gbs"], "peak": peak, "unit": "GB/s", "frac": d["frac"],
                "traffic": traffic_map.get(d["kernel"]), "alg_bytes_per_launch": d["alg_bytes"],
                "moved_bytes_per_launch": d["moved_bytes"], "moved_frac": d["moved_frac"], "peak_source": peak_src}
    compress_ms = mean["K1_minmax"] + mean["K2_histogram"] + mean["K3_select"] + mean["K4_encode"]

    e2e = None
    if not args.no_e2e:
        # end to end through the public host-buffer API: pinned host snapshots
        # in, compressed stream + reconstruction out, H2D / kernels / D2H of
        # consecutive steps overlapped (pipeline.StreamCompressor)
        cfg = pipeline.PipelineConfig(tolerance=E, bits=BITS, block_bytes=1 << 20)
        hb = torch.empty(n_local, dtype=torch.float64, pin_memory=True)
        hc = torch.empty(n_local, dtype=torch.float64, pin_memory=True)
        hb.copy_(base)
        hc.copy_(cur)
        depth = 3
        sc = pipeline.StreamCompressor(n_local, np.float64, cfg, depth=depth, elem0=elem0, n_total=n_total,
                                       comm=comm)
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
        e2e = {"value": n_total * L / dt / 1e9, "unit": "GB/s", "h2d_bytes_per_step": int(sc.h2d_bytes()),
               "d2h_bytes_per_step": int(d2h_total // reps),
               "path": "pipeline.StreamCompressor: pinned host pair -> compress + full decompress -> host "
                       "(packed stream, exact values, prefix, centers, reconstruction); zlib excluded; "
                       "copies of consecutive steps overlapped on separate streams",
               "wall_clock": "perf_counter over all steps incl. every H2D/D2H"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(base, cur, args.cpu_sample_log2)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded cfg2 recipe, generated on device)",
            "config": {"workload": CONFIG_NAME, "n_per_gpu": n_local, "n_total": n_total,
                       "parallelism": f"dp{world} (contiguous element shards)",
                       "l2": "inputs 2 GiB/GPU > 126 MB L2 (no flush needed)",
                       "k": chk["k"], "alpha": n_inc / n_local, "hist_form": "dense",
                       "execution": "sync-free device pipeline" + (" replayed as one CUDA graph" if use_graph else "")},
            "compress": {"ms": compress_ms, "gbs_per_gpu": n_local * L / (compress_ms / 1e3) / 1e9},
            "decompress": {"ms": mean["K5_decode"], "gbs_per_gpu": n_local * L / (mean["K5_decode"] / 1e3) / 1e9},
            "phase_ms": mean,
            "roofline": roofline,
            "roofline_all": roof_all,
            "e2e": e2e,
            "gpu_launches": GPU_LAUNCHES_PER_STEP * args.steps,
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if comm:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
