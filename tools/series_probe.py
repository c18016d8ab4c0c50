import sys, time, numpy as np, torch
sys.path.insert(0, ".")
from paper_1703_02438_b200 import pipeline, workloads
x = workloads.cfg3_device_first(seed=0)
snaps = [x.cpu().pin_memory()]
for t in range(1, 16):
    x = workloads.cfg3_device_step(x, t, seed=0); snaps.append(x.cpu().pin_memory())
n = x.numel(); d = torch.empty_like(x)
# raw H2D rate
torch.cuda.synchronize(); t0 = time.perf_counter()
for i in range(20): d.copy_(snaps[i % 16], non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 20
print(f"H2D {n*4/1e6:.1f} MB: {dt*1e3:.3f} ms  {n*4/dt/1e9:.1f} GB/s")
cfg = pipeline.PipelineConfig(tolerance=5e-3, bits=10, block_bytes=1 << 20)
for depth in (2, 3, 4):
    sc = pipeline.SeriesStreamCompressor(n, np.float32, cfg, depth=depth)
    sc.start(snaps[0])
    for t in range(1, 16): sc.result(sc.submit(snaps[t]))
    sc.start(snaps[0]); torch.cuda.synchronize()
    t0 = time.perf_counter(); pend = []; ts = []
    for t in range(1, 16):
        a = time.perf_counter(); pend.append(sc.submit(snaps[t])); b = time.perf_counter()
        if len(pend) == depth: sc.result(pend.pop(0))
        c = time.perf_counter(); ts.append((b - a, c - b))
    while pend: sc.result(pend.pop(0))
    dt = (time.perf_counter() - t0) / 15
    print(f"depth {depth}: {dt*1e3:.3f} ms/step {n*4/dt/1e9:.1f} GB/s; submit {np.mean([x[0] for x in ts])*1e3:.3f} ms result {np.mean([x[1] for x in ts])*1e3:.3f} ms")
