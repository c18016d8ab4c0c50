"""Kernel time of the GPU inflate on cfg2's 128 index blocks (zlib level 6 and
GPU-deflate streams), device buffers prepared beforehand.
    python tools/inflate_probe.py"""
import sys
import zlib

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1703_02438_b200 import _native as N, codec, engine, workloads  # noqa: E402

b, c = workloads.cfg2_device(512, seed=0)
enc = engine.encode(b, c, 1e-3, 8)
lens = enc.block_lengths()
packed = enc.packed.cpu().numpy()
host_blobs = [zlib.compressobj(6, zlib.DEFLATED, -15).compress(packed[i * enc.stride: i * enc.stride + int(ln)].tobytes())
              for i, ln in enumerate(lens)]
host_blobs = [hb + zlib.compressobj(6, zlib.DEFLATED, -15).flush() if False else hb for hb in host_blobs]
host_blobs = []
for i, ln in enumerate(lens):
    co = zlib.compressobj(6, zlib.DEFLATED, -15)
    host_blobs.append(co.compress(packed[i * enc.stride: i * enc.stride + int(ln)].tobytes()) + co.flush())
gpu_blobs = codec.gpu_deflate_blocks(enc.packed, enc.stride, lens)
for name, blobs in (("zlib6", host_blobs), ("gpu_deflate", gpu_blobs)):
    off = np.zeros(len(blobs) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(x) for x in blobs])
    d_comp = torch.from_numpy(np.frombuffer(b"".join(blobs) + bytes(16), dtype=np.uint8).copy()).cuda()
    d_off = torch.from_numpy(off).cuda()
    out = torch.empty(len(blobs) * enc.stride, dtype=torch.uint8, device="cuda")
    st = torch.empty(len(blobs), dtype=torch.int32, device="cuda")
    pr = torch.empty(len(blobs), dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    run = lambda: N.check(N.lib().nmk_inflate(d_comp.data_ptr(), d_off.data_ptr(), len(blobs), out.data_ptr(),  # noqa
                                               enc.stride, None, st.data_ptr(), pr.data_ptr(), s))
    run()
    torch.cuda.synchronize()
    a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        run()
    z.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(z) / 3
    assert int(st.abs().sum()) == 0 and np.array_equal(pr.cpu().numpy(), lens)
    assert torch.equal(out.view(len(blobs), enc.stride)[:, : int(lens[0])], enc.packed.view(-1, enc.stride)[:, : int(lens[0])])
    print(f"{name}: {len(blobs)} streams, {off[-1] / 1e6:.1f} MB -> {lens.sum() / 1e6:.1f} MB, kernel {ms:.2f} ms, "
          f"{lens.sum() / ms / 1e6:.2f} GB/s")
