import sys, torch
sys.path.insert(0, "/root/repo")
from paper_1703_02438_b200 import engine, workloads
base, cur = workloads.cfg2_device(128, seed=0)
pipe = engine.DevicePipeline(base.numel(), base.dtype, 1e-3, 8)
out = torch.empty_like(base)
pipe.step(base, cur, out)
torch.cuda.synchronize()
print("n", base.numel())
