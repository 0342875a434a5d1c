"""Practical HBM floor for an 80-90 MB single-pass read on this GPU: torch
reductions / copies timed with CUDA events, cold (L2 flushed) and warm."""
import json
import torch

def timeit(fn, flush, reps=20):
    l2 = torch.zeros(64 * 1024 * 1024, device="cuda")
    ts = []
    for _ in range(reps):
        if flush:
            l2.add_(1)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]

out = {}
for n in (10_000_000, 100_000_000):
    x = torch.rand(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for nm, fn in (("sum", lambda: x.sum()), ("copy", lambda: y.copy_(x))):
        for fl in (True, False):
            us = timeit(fn, fl)
            byts = 8 * n * (2 if nm == "copy" else 1)
            out[f"{nm}_{n}_{'cold' if fl else 'warm'}"] = (round(us, 1), round(byts / us / 1e3, 1))
print(json.dumps(out))
