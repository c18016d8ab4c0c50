"""Device throughput of every BASELINE config on one B200.

One JSON line per workload, CUDA events on the launch stream, inputs
resident in HBM (generated on the device, seeded):

* cfg1  2^20 fp64, E=1e-3, B=8 (L2-resident: a latency config);
* cfg2  512^3 fp64 (bench.py's workload; --only cfg2 for A/B runs);
* cfg4  weak share 2^29 fp64 per GPU, and the per-GPU shares of the strong
        4e9-element run at 8 / 4 / 2 GPUs (5e8, 1e9, 2e9 elements), E=1e-3, B=8;
* cfg5  2^28 fp64, B in {8, 10, 12} x E in {1e-4, 1e-3, 1e-2}: compress,
        full decompress, then 1000 random 2^16-element segments in one
        batched partial-decode launch.

(cfg3's fp32 series is tools/series_bench.py.)

A step is compress (K1..K4) + full decompress (K5) through the sync-free
DevicePipeline replayed as a CUDA graph; GB/s = n * L / time.  When a config
needs the general path (span too wide for the dense histogram) it is timed
through engine.encode / decode_encoding instead and the line says so.

    python tools/config_bench.py [--only cfg5] > profiles/r1_configs.jsonl
"""
import argparse
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1703_02438_b200 import engine, workloads  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def time_graph(g, reps):
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def phases(pipe, base, cur, out, reps=5):
    acc = {}
    for _ in range(reps):
        marks = [("start", ev())]
        marks[0][1].record()

        def mark(name):
            e = ev()
            e.record()
            marks.append((name, e))
        pipe.step(base, cur, out, mark)
        torch.cuda.synchronize()
        for (_, ea), (nb, eb) in zip(marks[:-1], marks[1:]):
            acc.setdefault(nb, []).append(ea.elapsed_time(eb))
    ph = {k: sum(v) / len(v) for k, v in acc.items()}
    comp = sum(v for k, v in ph.items() if k != "K5_decode")
    return ph, comp, ph.get("K5_decode", 0.0)


def run_pair(name, base, cur, E, bits, reps=10, segments=0, seed=0):
    n, L = base.numel(), base.element_size()
    out = torch.empty_like(base)
    pipe = engine.DevicePipeline(n, base.dtype, E, bits)
    pipe.step(base, cur, out)
    chk = pipe.check()
    line = {"workload": name, "n": n, "L": L, "E": E, "bits": bits}
    if chk["status"] == 0:
        g = pipe.capture(base, cur, out)
        ms = time_graph(g, reps)
        ph, comp, dec = phases(pipe, base, cur, out)
        chk = pipe.check()
        line.update(path="sync-free graph", step_ms=ms, gbs=n * L / ms / 1e6, compress_ms=comp,
                    compress_gbs=n * L / comp / 1e6, decompress_ms=dec, decompress_gbs=n * L / dec / 1e6,
                    phase_ms=ph, k=chk["k"], alpha=chk["n_inc"] / n, nbins=chk["nbins"])
        del g
        enc = pipe.encoding()
    else:   # general path (sparse histogram): host-synchronising encode
        a, b, c = ev(), ev(), ev()
        times = []
        for i in range(reps // 2 + 2):
            a.record()
            enc = engine.encode(base, cur, E, bits)
            b.record()
            res = engine.decode_encoding(enc, base, out, check=False)
            c.record()
            torch.cuda.synchronize()
            if i >= 2:
                times.append((a.elapsed_time(b), b.elapsed_time(c)))
        comp = float(np.median([t[0] for t in times]))
        dec = float(np.median([t[1] for t in times]))
        line.update(path=f"general (status {chk['status']}: {enc.hist_form} histogram)", step_ms=comp + dec,
                    gbs=n * L / (comp + dec) / 1e6, compress_ms=comp, compress_gbs=n * L / comp / 1e6,
                    decompress_ms=dec, decompress_gbs=n * L / dec / 1e6, k=enc.k, alpha=enc.n_inc / n)
    if segments:
        seg_len = 1 << 16
        rng = np.random.default_rng(seed)
        starts = rng.integers(0, n - seg_len, segments)
        segs = [(int(s), seg_len, i * seg_len) for i, s in enumerate(starts)]
        idx = torch.from_numpy(np.concatenate([np.arange(s, s + seg_len) for s, _, _ in segs])).cuda()
        pbase = base[idx]
        pout = torch.empty_like(pbase)
        args = (enc.packed, enc.stride, enc.b0, enc.bits, enc.epb, enc.n, enc.prefix, enc.centers, enc.exact, pbase,
                segs, pout)
        for _ in range(2):
            engine.decode(*args, check=False)
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record()
        for _ in range(reps):
            engine.decode(*args, check=False)
        b.record()
        torch.cuda.synchronize()
        pms = a.elapsed_time(b) / reps
        res = engine.decode(*args)
        assert not res.bad_index and not res.exhausted
        line.update(partial_segments=segments, partial_segment_len=seg_len, partial_ms=pms,
                    partial_gbs=segments * seg_len * L / pms / 1e6,
                    partial_note="one batched K5 launch over all segments (host ctypes set-up included)")
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--lib", default=None, help="alternative libnmkgpu.so (A/B)")
    args = ap.parse_args()
    if args.lib:
        from paper_1703_02438_b200 import _native as N
        N._lib = N.load(args.lib)
    want = lambda k: not args.only or args.only in k  # noqa: E731
    lines = []
    if want("cfg1"):
        base, cur = workloads.cfg1_device(1 << 20, seed=0)
        lines.append(run_pair("cfg1: 2^20 fp64 (L2-resident)", base, cur, 1e-3, 8, reps=50))
        del base, cur
    if want("cfg2"):
        base, cur = workloads.cfg2_device(512, seed=0)
        lines.append(run_pair("cfg2: 512^3 fp64 8^3-block field", base, cur, 1e-3, 8, reps=20))
        del base, cur
    if want("cfg4"):
        for n, label in [(1 << 29, "cfg4 weak: 2^29 fp64 per GPU"),
                         (500_000_000, "cfg4 strong, per-GPU share at 8 GPUs (4e9/8)"),
                         (1_000_000_000, "cfg4 strong, per-GPU share at 4 GPUs (4e9/4)"),
                         (2_000_000_000, "cfg4 strong, per-GPU share at 2 GPUs (4e9/2)")]:
            try:
                base, cur = workloads.cfg1_device(n, seed=4)
                torch.cuda.empty_cache()
                lines.append(run_pair(label, base, cur, 1e-3, 8, reps=5))
            except torch.OutOfMemoryError as e:
                lines.append({"workload": label, "n": n, "skipped": f"out of memory: {str(e)[:80]}"})
            base = cur = None
            torch.cuda.empty_cache()
    if want("cfg5"):
        base, cur = workloads.cfg5_device(1 << 28, seed=5)
        for bits in (8, 10, 12):
            for E in (1e-4, 1e-3, 1e-2):
                lines.append(run_pair(f"cfg5: 2^28 fp64 B={bits} E={E:g}", base, cur, E, bits, reps=6,
                                      segments=1000, seed=bits))
                torch.cuda.empty_cache()
    for ln in lines:
        print(json.dumps(ln), flush=True)


if __name__ == "__main__":
    main()
