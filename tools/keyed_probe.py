"""Diagnostic: how many cfg2 elements K4's keyed mode sends down the slow
path, emulating classify_key from K1's keys on the device (torch f32)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1703_02438_b200 import engine, workloads, _native as N

side = int(sys.argv[1]) if len(sys.argv) > 1 else 512
base, cur = workloads.cfg2_device(side, seed=0)
E = 1e-3
pipe = engine.DevicePipeline(base.numel(), base.dtype, E, 8)
out = torch.empty_like(base)
pipe.step(base, cur, out)
torch.cuda.synchronize()
c = pipe.check()
print(c)
keys = pipe.keys[: base.numel()]
print("nan keys", int(torch.isnan(keys).sum()), "inf keys", int(torch.isinf(keys).sum()))
gmin, gmax = c["gmin"], c["gmax"]
w = 2 * E
iw = 1.0 / w
iw32 = torch.tensor(iw, dtype=torch.float32, device="cuda")
c32 = torch.tensor(-gmin * iw - 0.5, dtype=torch.float32, device="cuda")
th = (keys.double() * iw32.double() + c32.double()).float()
m = th + 12582912.0
d = (th - (m - 12582912.0)).abs()
for t in (0.4999, 0.499, 0.49, 0.45):
    print(t, float((d >= t).float().mean()))
r = (cur - base) / base
rk = r.float()
print("keys == RN32(r):", float((rk == keys).float().mean()))
bad = (rk != keys)
print("first mismatches", r[bad][:5].tolist(), keys[bad][:5].tolist())
