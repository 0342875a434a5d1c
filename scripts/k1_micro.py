"""Microbenchmark of the fused scan+reduce kernel (K1) alone.

python scripts/k1_micro.py [--n 1e7] [--k 1000] [--p 64]
Prints per-launch device time (library CUDA events) cold (L2 flushed before
each launch) and warm (back-to-back), and the effective GB/s on the
algorithmic bytes N*(8 + code bytes) + 4*nnz_j.
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
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    import torch
    import paper_2310_16238_b200 as sx
    from paper_2310_16238_b200 import _capi, synthetic

    lib = _capi.load()
    n = int(args.n)
    syn = synthetic.generate(n, args.p, args.k, args.density, seed=3)
    d = syn.sorted_design()
    dd = sx.upload(d)
    info = dd.info()
    h = dd.handle
    rng = np.random.default_rng(1)
    beta = rng.normal(0, 0.05, args.p)
    st = sx.make_state(dd, beta)
    l2 = torch.zeros(64 * 1024 * 1024, device="cuda")
    out = {"n": n, "k": args.k, "code_bytes": info["code_bytes"], "n_tiles": info["n_tiles"]}
    for mode in ("cold", "warm"):
        lib.scx_timing_enable(h, 1)
        lib.scx_timing_reset(h)
        for _ in range(args.reps):
            for j in range(args.p):
                if mode == "cold":
                    l2.add_(1)
                    torch.cuda.synchronize()
                sx.gradient_hessian(dd, st, j)
        tot = C.c_double(); nl = C.c_int64()
        lib.scx_timing_get(h, 0, C.byref(tot), C.byref(nl))
        ms = tot.value / nl.value
        nnz = float(np.mean(np.diff(d.col_ptr)))
        byts = n * (8 + info["code_bytes"]) + 4 * nnz
        out[mode + "_us"] = ms * 1e3
        out[mode + "_gbs"] = byts / (ms * 1e-3) / 1e9
    lib.scx_timing_enable(h, 0)
    # loglik (K2) for reference
    lib.scx_timing_enable(h, 1)
    lib.scx_timing_reset(h)
    for _ in range(10):
        sx.log_partial_likelihood(dd, st)
    lib.scx_timing_get(h, 2, C.byref(tot), C.byref(nl))
    out["k2_us"] = tot.value / nl.value * 1e3
    print(json.dumps(out))


if __name__ == "__main__":
    main()
