"""A/B of library variants: kernel time of inflating one cfg5 index block (noisy, ratio 1.2).
    python tools/partial_ab.py variants/a.so ..."""
import sys
import zlib

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1703_02438_b200 import _native as N, codec, engine, workloads  # noqa: E402

b, c = workloads.cfg5_device(1 << 22, seed=5)
enc = engine.encode(b, c, 1e-4, 8)
lens = enc.block_lengths()
packed = enc.packed.cpu().numpy()
blobs = []
for i, ln in enumerate(lens):
    co = zlib.compressobj(6, zlib.DEFLATED, -15)
    blobs.append(co.compress(packed[i * enc.stride: i * enc.stride + int(ln)].tobytes()) + co.flush())
for path in [None] + sys.argv[1:]:
    N._lib = N.load(path) if path else N.load()
    codec.gpu_inflate_blocks(blobs[:1], enc.stride)
    torch.cuda.synchronize()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        out, produced = codec.gpu_inflate_blocks(blobs[:1], enc.stride)
    z.record()
    torch.cuda.synchronize()
    assert out[: int(lens[0])].cpu().numpy().tobytes() == packed[: int(lens[0])].tobytes()
    print(f"{path or 'in-tree'}: one block, {len(blobs[0])} -> {int(lens[0])} bytes: {a.elapsed_time(z) / 3:.2f} ms per call")
