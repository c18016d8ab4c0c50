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

wl = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
if wl == "cfg3":
    base = workloads.cfg3_device_first(seed=0)
    cur = workloads.cfg3_device_step(base, 1, seed=0)
    enc = engine.encode(base, cur, 5e-3, 10)
elif wl == "cfg5":
    base, cur = workloads.cfg5_device(1 << 26, seed=5)
    enc = engine.encode(base, cur, 1e-4, 12)
else:
    base, cur = workloads.cfg2_device(512, seed=0)
    enc = engine.encode(base, cur, 1e-3, 8)
print("workload", wl)
lens = enc.block_lengths()
raw_total = int(sum(lens))
from paper_1703_02438_b200 import _native as N  # noqa: E402


def kernel_ms(seg, reps=3):
    """nmk_deflate alone (segments + scan + gather), CUDA events"""
    lib = N.lib()
    nb, bl, ll = len(lens), int(lens[0]), int(lens[-1])
    wsb = lib.nmk_deflate_ws_bytes(nb, bl, seg)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    out = torch.empty(lib.nmk_deflate_bound(nb, bl, seg), dtype=torch.uint8, device="cuda")
    off = torch.empty(nb + 1, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        N.check(lib.nmk_deflate(enc.packed.data_ptr(), enc.stride, nb, bl, ll, seg, out.data_ptr(), off.data_ptr(),
                                ws.data_ptr(), wsb, st))
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for seg in (4096, 8192, 16384, 32768, 65520):
    codec.gpu_deflate_blocks(enc.packed, enc.stride, lens, seg)
    print(f"gpu deflate seg={seg:6d}: kernels {kernel_ms(seg):8.2f} ms")
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
