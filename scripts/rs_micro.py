"""Microbenchmark of the risk-suffix cycle's fused risk scan (scx_risk_prefix)
and of one risk-suffix coordinate evaluation.

python scripts/rs_micro.py [--n 1e7] [--k 1000] [--p 64] [--reps 8]
Prints per-launch device time (library CUDA events, L2 flushed before each
launch) and GB/s on the algorithmic bytes N*(8 + code bytes + 16).
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=float, default=1e7)
    ap.add_argument("--k", type=int, default=1000)
    ap.add_argument("--p", type=int, default=64)
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--reps", type=int, default=8)
    args = ap.parse_args()
    import torch
    import paper_2310_16238_b200 as sx
    from paper_2310_16238_b200 import _capi, synthetic

    lib = _capi.load()
    l2 = torch.zeros(64 * 1024 * 1024, device="cuda")
    n = int(args.n)
    syn = synthetic.generate(n, args.p, args.k, args.density, seed=3, device="cuda")
    d = syn.sorted_design()
    dd = sx.upload(d)
    info = dd.info()
    h = dd.handle
    assert dd.set_fit_path(0)
    rng = np.random.default_rng(1)
    st = sx.make_state(dd, rng.normal(0, 0.05, args.p))
    byts = n * (8 + info["code_bytes"] + 16)
    out = {"n": n, "k": info["n_strata"], "code_bytes": info["code_bytes"]}
    tot = C.c_double()
    nl = C.c_int64()
    for mode in ("cold", "warm"):
        lib.scx_timing_enable(h, 1)
        lib.scx_timing_reset(h)
        for _ in range(args.reps):
            if mode == "cold":
                l2.add_(1.0)
                torch.cuda.synchronize()
            assert lib.scx_risk_prefix(h) == 0
        lib.scx_timing_get(h, 3, C.byref(tot), C.byref(nl))
        ms = tot.value / max(1, nl.value)
        out[f"prefix_{mode}_us"] = ms * 1e3
        out[f"prefix_{mode}_gbs"] = byts / (ms * 1e-3) / 1e9
    # back-to-back scans inside one launch (the fit's regime: no launch, no
    # pipeline fill per scan); L2 flushed before the launch
    for reps in (1, 2, 8, 32):
        lib.scx_timing_reset(h)
        for _ in range(3):
            l2.add_(1.0)
            torch.cuda.synchronize()
            assert lib.scx_risk_prefix_n(h, reps) == 0
        lib.scx_timing_get(h, 3, C.byref(tot), C.byref(nl))
        ms = tot.value / max(1, nl.value) / reps
        out[f"prefix_x{reps}_us"] = ms * 1e3
        out[f"prefix_x{reps}_gbs"] = byts / (ms * 1e-3) / 1e9
    lib.scx_timing_reset(h)
    for j in range(min(args.p, 16)):
        sx.risk_suffix_gradient_hessian(dd, st, j)
    lib.scx_timing_get(h, 3, C.byref(tot), C.byref(nl))
    out["eval_incl_prefix_us"] = tot.value / max(1, nl.value) * 1e3
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
