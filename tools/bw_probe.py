import torch
x = torch.empty(2**28, dtype=torch.float64, device="cuda").uniform_()
y = torch.empty_like(x)
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
ms = t(lambda: x.sum()); print("read-only sum 2 GiB: %.3f ms  %.0f GB/s" % (ms, x.numel()*8/ms/1e6))
ms = t(lambda: y.copy_(x)); print("copy 2 GiB: %.3f ms  %.0f GB/s (r+w)" % (ms, 2*x.numel()*8/ms/1e6))
h = x[: 2**27]
ms = t(lambda: h.sum()); print("read-only sum 1 GiB: %.3f ms  %.0f GB/s" % (ms, h.numel()*8/ms/1e6))
