"""cProfile of single partial_decode calls on cfg5 (2^28, B=8, E=1e-4)."""
import cProfile
import pstats
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1703_02438_b200 as nmk  # noqa: E402
from paper_1703_02438_b200 import codec, workloads  # noqa: E402

n5 = 1 << 26
b5, c5 = workloads.cfg5_device(n5, seed=5)
b5h, c5h = b5.cpu().numpy(), c5.cpu().numpy()
cfg5 = nmk.PipelineConfig(tolerance=1e-4, bits=8, workers=16)
v5, _ = nmk.compress_pair(nmk.TemporalPair(b5h, c5h), cfg5)
rng = np.random.default_rng(0)
starts = rng.integers(0, n5 - (1 << 16), 20)
for s in starts[:3]:
    codec.partial_decode(v5, int(s), 1 << 16, b5h[s:s + (1 << 16)])
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for s in starts:
    codec.partial_decode(v5, int(s), 1 << 16, b5h[s:s + (1 << 16)])
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
