"""Per-step time of the sync-free step when S steps share one CUDA graph (gap between graph launches)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1703_02438_b200 import engine, workloads  # noqa: E402

for name in ("cfg3", "cfg2"):
    if name == "cfg3":
        base = workloads.cfg3_device_first(seed=0)
        cur = workloads.cfg3_device_step(base, 1, seed=0)
        E, B = 5e-3, 10
    else:
        base, cur = workloads.cfg2_device(512, seed=0)
        E, B = 1e-3, 8
    out = torch.empty_like(base)
    pipe = engine.DevicePipeline(base.numel(), base.dtype, E, B)
    for _ in range(3):
        pipe.step(base, cur, out)
    pipe.check()
    for S in (1, 2, 5, 15):
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            pipe.step(base, cur, out)
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(S):
                pipe.step(base, cur, out)
        reps = 60 // S
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            g.replay()
        z.record()
        torch.cuda.synchronize()
        print(f"{name}: {S:2d} steps per graph: {a.elapsed_time(z) / (reps * S):.4f} ms per step", flush=True)
    del base, cur, out, pipe
    torch.cuda.empty_cache()
