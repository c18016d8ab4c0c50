"""A/B timing of the decode entry points on the cfg2 field (CUDA events)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1703_02438_b200 import engine, workloads  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


base, cur = workloads.cfg2_device(512, seed=0)
out = torch.empty_like(base)
pipe = engine.DevicePipeline(base.numel(), base.dtype, 1e-3, 8)
pipe.step(base, cur, out)
enc = pipe.encoding()
print("dev decode      ms", timeit(lambda: pipe.decode(base, out)))
print("host-k decode   ms", timeit(lambda: engine.decode(enc.packed, enc.stride, 0, 8, enc.epb, enc.n, enc.prefix,
                                                          enc.centers, enc.exact, base, [(0, enc.n, 0)], out,
                                                          check=False)))
print("encode (dev)    ms", timeit(lambda: pipe.encode(base, cur)))
g = pipe.capture(base, cur, out)
print("graph step      ms", timeit(lambda: g.replay()))

if len(sys.argv) > 1:
    from paper_1703_02438_b200 import _native as N
    for path in sys.argv[1:]:
        N._lib = None
        N._lib = N.load(path)
        p2 = engine.DevicePipeline(base.numel(), base.dtype, 1e-3, 8)
        p2.step(base, cur, out)
        print(path, "dev decode ms", timeit(lambda: p2.decode(base, out)))
