import sys, torch
sys.path.insert(0, ".")
from paper_1703_02438_b200 import engine, workloads
x0 = workloads.cfg3_device_first(seed=0); x1 = workloads.cfg3_device_step(x0, 1, seed=0)
pipe = engine.DevicePipeline(x0.numel(), x0.dtype, 5e-3, 10)
out = torch.empty_like(x0)
for _ in range(2): pipe.step(x0, x1, out)
torch.cuda.synchronize(); print(pipe.check())
