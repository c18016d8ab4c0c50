"""One sync-free compress + decompress step on a named workload (for ncu).
    python tools/one_step.py cfg4w|cfg5|cfg2|cfg3 [n_log2] [E] [B]
The first step launches every kernel (10); the second one runs with the
check() hints (8 launches): ncu -s 10 -c 8 captures it."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1703_02438_b200 import engine, workloads  # noqa: E402

name = sys.argv[1]
lg = int(sys.argv[2]) if len(sys.argv) > 2 else 27
E = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-3
B = int(sys.argv[4]) if len(sys.argv) > 4 else 8
if name == "cfg4w":
    base, cur = workloads.cfg1_device(1 << lg, seed=4)
elif name == "cfg5":
    base, cur = workloads.cfg5_device(1 << lg, seed=5)
elif name == "cfg3":
    base = workloads.cfg3_device_first(seed=0)
    cur = workloads.cfg3_device_step(base, 1, seed=0)
    E = float(sys.argv[3]) if len(sys.argv) > 3 else 5e-3
    B = int(sys.argv[4]) if len(sys.argv) > 4 else 10
else:
    base, cur = workloads.cfg2_device(512, seed=0)
out = torch.empty_like(base)
pipe = engine.DevicePipeline(base.numel(), base.dtype, E, B)
for _ in range(2):
    pipe.step(base, cur, out)
    torch.cuda.synchronize()
    print(pipe.check())   # also sets the span hint the next step's K2 launch uses
