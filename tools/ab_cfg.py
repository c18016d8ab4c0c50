"""A/B of library variants on several BASELINE workloads (device step time
and per-phase times from tools/config_bench.run_pair).
    python tools/ab_cfg.py [variant.so ...]   (the in-tree library first)"""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from paper_1703_02438_b200 import _native as N, workloads  # noqa: E402
from config_bench import run_pair  # noqa: E402

paths = [None] + sys.argv[1:]
libs = {p: (N.load(p) if p else N.load()) for p in paths}
def cfg3_pair():
    x0 = workloads.cfg3_device_first(seed=0)
    return x0, workloads.cfg3_device_step(x0, 1, seed=0)


cases = [("cfg3", cfg3_pair, 5e-3, 10),
         ("cfg2", lambda: workloads.cfg2_device(512, seed=0), 1e-3, 8),
         ("cfg4w", lambda: workloads.cfg1_device(1 << 29, seed=4), 1e-3, 8),
         ("cfg5 B8 E1e-3", lambda: workloads.cfg5_device(1 << 28, seed=5), 1e-3, 8),
         ("cfg5 B8 E1e-4", lambda: workloads.cfg5_device(1 << 28, seed=5), 1e-4, 8),
         ("cfg5 B8 E1e-2", lambda: workloads.cfg5_device(1 << 28, seed=5), 1e-2, 8),
         ("cfg5 B12 E1e-4", lambda: workloads.cfg5_device(1 << 28, seed=5), 1e-4, 12)]
only = os.environ.get("AB_CASES")   # comma-separated case names to run (default: all)
if only:
    cases = [c for c in cases if c[0] in only.split(",")]
for name, gen, E, bits in cases:
    base, cur = gen()
    for rnd in range(2):
        for p in paths:
            N._lib = libs[p]
            ln = run_pair(name, base, cur, E, bits, reps=10)
            ph = {k[:2]: round(v, 4) for k, v in ln.get("phase_ms", {}).items()}
            print(f"{name:16s} {str(p):22s} step {ln['step_ms']:.4f} ms {ln['gbs']:7.1f} GB/s {ph}", flush=True)
    del base, cur
    torch.cuda.empty_cache()
