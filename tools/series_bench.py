"""BASELINE config 3: the fp32 climate-like series (1440 x 720 x 30, 16 steps,
E = 5e-3, B = 10), each transition compressed against the previous
reconstruction.  Reports per-step device throughput of the sync-free chain
(K1..K4 with K4's fused reconstruction = compress_series' inner loop) and of
compress + full decompress per transition, CUDA events, GB/s of input."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1703_02438_b200 import engine, workloads  # noqa: E402

E, BITS = 5e-3, 10
x = workloads.cfg3_device_first(seed=0)
n = x.numel()
steps = [x]
for t in range(1, 16):
    steps.append(workloads.cfg3_device_step(steps[-1], t, seed=0))
pipe = engine.DevicePipeline(n, torch.float32, E, BITS)
recon = [torch.empty_like(x) for _ in range(2)]
out = torch.empty_like(x)


def chain(decode: bool):
    recon[0].copy_(steps[0])
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(16)]
    ev[0].record()
    for t in range(1, 16):
        a, b = recon[(t - 1) % 2], recon[t % 2]
        pipe.encode(a, steps[t], recon=b)
        if decode:
            pipe.decode(a, out)
        ev[t].record()
    torch.cuda.synchronize()
    return [ev[t - 1].elapsed_time(ev[t]) for t in range(1, 16)]


for _ in range(2):
    chain(False)
    chain(True)
enc_ms = chain(False)
full_ms = chain(True)
chk = pipe.check()
assert chk["status"] == 0 and not chk["exhausted"] and not chk["bad_index"]
L = 4
res = {
    "workload": "cfg3: 1440x720x30 fp32, 16 steps (15 transitions), E=5e-3, B=10",
    "n": n, "k_last": chk["k"], "alpha_last": chk["n_inc"] / n,
    "compress_chain_ms_per_step": sum(enc_ms) / len(enc_ms),
    "compress_chain_gbs": n * L / (sum(enc_ms) / len(enc_ms) / 1e3) / 1e9,
    "compress_plus_decompress_ms_per_step": sum(full_ms) / len(full_ms),
    "compress_plus_decompress_gbs": n * L / (sum(full_ms) / len(full_ms) / 1e3) / 1e9,
}
print(json.dumps(res))

# per-phase split of one transition (events between phases)
ph = {}
for _ in range(5):
    evs = [("start", torch.cuda.Event(enable_timing=True))]
    evs[0][1].record()

    def mark(name, evs=evs):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        evs.append((name, e))
    pipe.step(recon[0], steps[1], out, mark=mark)
    torch.cuda.synchronize()
    for (_, e0), (nm, e1) in zip(evs[:-1], evs[1:]):
        ph.setdefault(nm, []).append(e0.elapsed_time(e1))
print(json.dumps({k: round(sum(v) / len(v), 4) for k, v in ph.items()}))
