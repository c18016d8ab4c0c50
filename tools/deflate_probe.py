"""GPU DEFLATE stage vs host zlib on the cfg2 512^3 index stream: time and
compressed size (CUDA events for the GPU stage incl. the D2H of its output;
wall clock for zlib over all host cores)."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import torch

sys.path.insert(0, ".")
from paper_1703_02438_b200 import codec, engine, workloads  # noqa: E402

base, cur = workloads.cfg2_device(512, seed=0)
enc = engine.encode(base, cur, 1e-3, 8)
lens = enc.block_lengths()
raw_total = int(sum(lens))
for seg in (4096, 8192, 16384, 32768):
    codec.gpu_deflate_blocks(enc.packed, enc.stride, lens, seg)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = codec.gpu_deflate_blocks(enc.packed, enc.stride, lens, seg)
    dt = time.perf_counter() - t0
    tot = sum(len(o) for o in out)
    print(f"gpu deflate seg={seg:6d}: {dt*1e3:8.2f} ms  {tot/1e6:8.3f} MB  ratio {raw_total/tot:7.2f}  "
          f"{raw_total/dt/1e9:6.2f} GB/s of packed input")
packed = enc.packed.cpu().numpy()
blocks = [packed[b * enc.stride: b * enc.stride + int(n)].tobytes() for b, n in enumerate(lens)]
w = os.cpu_count()
t0 = time.perf_counter()
with ThreadPoolExecutor(max_workers=w) as ex:
    z = list(ex.map(codec.compress_block, blocks))
dt = time.perf_counter() - t0
tot = sum(len(o) for o in z)
print(f"host zlib level 6 ({w} threads): {dt*1e3:8.2f} ms  {tot/1e6:8.3f} MB  ratio {raw_total/tot:7.2f}  "
      f"{raw_total/dt/1e9:6.2f} GB/s")
