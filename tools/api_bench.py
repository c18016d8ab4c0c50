"""Throughput of the reference-facing public API on one B200 (host buffers in,
host objects out), next to the lossless stage timed on its own.

    python tools/api_bench.py > profiles/r2_api.json

* compress_pair on cfg2 (512^3 fp64, E=1e-3, B=8): wall time, split into
  PhaseTimings' hot phases and the host zlib (DEFLATE) column;
* decompress (full) of the same variable: wall time; inflate runs on the
  GPU (k_inflate.cu), timed separately on the same streams;
* GPU inflate of the 128 index blocks alone, zlib's streams and the GPU
  deflate stage's streams (GB/s of inflated bytes), GPU deflate alone;
* cfg5 (2^28, B=8, E=1e-3): 1000 random 2^16-element segments through
  codec.partial_decode_many (one batched K5 launch) and through
  partial_decode one call at a time;
* compress_series on cfg3's 16 snapshots (1440x720x30 fp32, E=5e-3, B=10).
GB/s = n * L of the timestep / wall time.
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1703_02438_b200 as nmk  # noqa: E402
from paper_1703_02438_b200 import codec, engine, workloads  # noqa: E402


def wall(fn, reps=3):
    best, out = None, None
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best, out


def ev_time(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3


res = {}
# ---- cfg2 through compress_pair / decompress --------------------------------
b_d, c_d = workloads.cfg2_device(512, seed=0)
base, cur = b_d.cpu().numpy(), c_d.cpu().numpy()
n, L = base.size, 8
cfg = nmk.PipelineConfig(tolerance=1e-3, bits=8, workers=16)
pair = nmk.TemporalPair(base, cur)
nmk.compress_pair(pair, cfg)
t_c, (var, tm) = wall(lambda: nmk.compress_pair(pair, cfg))
hot = tm.change_ratio + tm.binning + tm.assign_index + tm.index_alignment + tm.bits_packing
t_d, out = wall(lambda: nmk.decompress(var, base))
res["cfg2_compress_pair"] = {"wall_s": t_c, "gbs_wall": n * L / t_c / 1e9, "hot_s": hot,
                             "gbs_hot": n * L / hot / 1e9, "zlib_s_host_16_threads": tm.zlib,
                             "phases": {p: getattr(tm, p) for p in tm.PHASES}}
res["cfg2_decompress"] = {"wall_s": t_d, "gbs_wall": n * L / t_d / 1e9,
                          "note": "GPU inflate + K5 + H2D of compressed bytes, base and exact values + D2H"}
# the whole compressor on the GPU: PipelineConfig(deflate="gpu") (valid DEFLATE, not zlib's bytes)
cfg_g = nmk.PipelineConfig(tolerance=1e-3, bits=8, workers=16, deflate="gpu")
nmk.compress_pair(pair, cfg_g)
t_cg, (var_g, tm_g) = wall(lambda: nmk.compress_pair(pair, cfg_g))
t_dg, out_g = wall(lambda: nmk.decompress(var_g, base))
assert out_g.tobytes() == out.tobytes()
res["cfg2_compress_pair_gpu_deflate"] = {"wall_s": t_cg, "gbs_wall": n * L / t_cg / 1e9, "lossless_s": tm_g.zlib,
                                         "index_table_bytes": len(var_g.index_table),
                                         "index_table_bytes_zlib": len(var.index_table),
                                         "decompress_wall_s": t_dg}
# ---- lossless stage alone ----------------------------------------------------
blobs = [codec._block_bytes_of(var, b) for b in range(var.nblocks)]
stride = engine.block_stride(var.elements_per_block, var.bits)
raw = sum(codec.packed_size(min((b + 1) * var.elements_per_block, n) - b * var.elements_per_block, 8)
          for b in range(var.nblocks))
t_inf = ev_time(lambda: codec.gpu_inflate_blocks(blobs, stride))
enc = engine.encode(b_d, c_d, 1e-3, 8)
gblobs = codec.gpu_deflate_blocks(enc.packed, enc.stride, enc.block_lengths())
t_inf_g = ev_time(lambda: codec.gpu_inflate_blocks(gblobs, stride))
t_def_g = ev_time(lambda: codec.gpu_deflate_blocks(enc.packed, enc.stride, enc.block_lengths()), reps=2)
t0 = time.perf_counter()
for blob in blobs:
    codec.decompress_block(blob)
t_inf_host = time.perf_counter() - t0
res["cfg2_lossless"] = {
    "packed_bytes": raw, "zlib_level6_bytes": sum(map(len, blobs)), "gpu_deflate_bytes": sum(map(len, gblobs)),
    "gpu_inflate_zlib_streams_s": t_inf, "gpu_inflate_zlib_streams_gbs": raw / t_inf / 1e9,
    "gpu_inflate_gpu_streams_s": t_inf_g, "gpu_inflate_gpu_streams_gbs": raw / t_inf_g / 1e9,
    "gpu_deflate_s": t_def_g, "gpu_deflate_gbs": raw / t_def_g / 1e9,
    "host_zlib_inflate_1_thread_s": t_inf_host,
    "timing": "gpu: CUDA events around the call incl. its H2D of compressed bytes; host: perf_counter"}
del b_d, c_d, enc
torch.cuda.empty_cache()
# ---- cfg5 partial decodes ----------------------------------------------------
b5, c5 = workloads.cfg5_device(1 << 28, seed=5)
base5, cur5 = b5.cpu().numpy(), c5.cpu().numpy()
del b5, c5
torch.cuda.empty_cache()
v5, _ = nmk.compress_pair(nmk.TemporalPair(base5, cur5), nmk.PipelineConfig(tolerance=1e-3, bits=8, workers=16))
rng = np.random.default_rng(0)
starts = rng.integers(0, base5.size - (1 << 16), 1000)
ranges = [(int(s), 1 << 16) for s in starts]
bases = [base5[s:s + c] for s, c in ranges]
codec.partial_decode_many(v5, ranges[:4], bases[:4])
t_many, outs = wall(lambda: codec.partial_decode_many(v5, ranges, bases), reps=2)
t_one, _ = wall(lambda: [codec.partial_decode(v5, s, c, bb) for (s, c), bb in zip(ranges[:50], bases[:50])], reps=1)
full = nmk.decompress(v5, base5)
assert all(np.array_equal(o.view(np.uint64), full[s:s + c].view(np.uint64)) for o, (s, c) in zip(outs, ranges))
res["cfg5_partial_1000x2^16"] = {"batched_s": t_many, "segments_per_s_batched": 1000 / t_many,
                                 "one_call_per_segment_s_per_segment": t_one / 50,
                                 "segments_per_s_one_call": 50 / t_one,
                                 "note": "inflate included (GPU); equal to slices of the full decompress"}
del v5, full, outs
# ---- cfg3 compress_series ----------------------------------------------------
x = workloads.cfg3_device_first(seed=0)
snaps = [x.cpu().numpy()]
for t in range(1, 16):
    x = workloads.cfg3_device_step(x, t, seed=0)
    snaps.append(x.cpu().numpy())
cfg3 = nmk.PipelineConfig(tolerance=5e-3, bits=10, workers=16)
nmk.compress_series(snaps[:3], cfg3)
t_s, (first, variables) = wall(lambda: nmk.compress_series(snaps, cfg3), reps=1)
res["cfg3_compress_series"] = {"wall_s": t_s, "transitions": 15, "s_per_transition": t_s / 15,
                               "gbs_wall": 15 * snaps[0].size * 4 / t_s / 1e9,
                               "note": "includes host zlib of every block (reference-identical .nmk bytes)"}
cfg3g = nmk.PipelineConfig(tolerance=5e-3, bits=10, workers=16, deflate="gpu")
nmk.compress_series(snaps[:3], cfg3g)
t_sg, (first_g, variables_g) = wall(lambda: nmk.compress_series(snaps, cfg3g), reps=1)
res["cfg3_compress_series_gpu_deflate"] = {"wall_s": t_sg, "s_per_transition": t_sg / 15,
                                           "gbs_wall": 15 * snaps[0].nbytes / t_sg / 1e9,
                                           "index_bytes": sum(len(v.index_table) for v in variables_g),
                                           "index_bytes_zlib": sum(len(v.index_table) for v in variables)}
res["host"] = {"cpu_count": __import__("os").cpu_count()}
print(json.dumps(res, indent=1))
