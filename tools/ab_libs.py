"""A/B timing of the sync-free step on the cfg2 512^3 field for the in-tree
library and each variant .so on the command line.  Variants are interleaved
over several rounds (drift cancels); per round: graph-replay step time and
the per-phase times of an event-instrumented pass (CUDA events, means over
20 steps after 3 warm-ups).  Prints the median over rounds."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_1703_02438_b200 import _native as N, engine, workloads  # noqa: E402

ROUNDS = 5
base, cur = workloads.cfg2_device(512, seed=0)
out = torch.empty_like(base)
paths = [None] + sys.argv[1:]
libs = {}
for p in paths:
    N._lib = None
    libs[p] = N.load(p) if p else N.load()


def measure(p, reps=20):
    N._lib = libs[p]
    pipe = engine.DevicePipeline(base.numel(), base.dtype, 1e-3, 8)
    pipe.step(base, cur, out)
    g = pipe.capture(base, cur, out)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    step = e0.elapsed_time(e1) / reps
    ph = {}
    for _ in range(reps):
        evs = [("start", torch.cuda.Event(enable_timing=True))]
        evs[0][1].record()

        def mark(name):
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            evs.append((name, ev))
        pipe.step(base, cur, out, mark)
        torch.cuda.synchronize()
        for (a, ea), (b, eb) in zip(evs[:-1], evs[1:]):
            ph.setdefault(b, []).append(ea.elapsed_time(eb))
    del g, pipe
    return step, {k: sum(v) / len(v) for k, v in ph.items()}


res = {p: [] for p in paths}
for r in range(ROUNDS):
    for p in paths:
        res[p].append(measure(p))
for p in paths:
    steps = [s for s, _ in res[p]]
    keys = res[p][0][1].keys()
    med = {k: statistics.median(ph[k] for _, ph in res[p]) for k in keys}
    print(f"{p or 'in-tree':26s} step {statistics.median(steps):.4f} ms [{min(steps):.4f}..{max(steps):.4f}]  " +
          " ".join(f"{k.split('_')[0]}={v:.4f}" for k, v in med.items()))
