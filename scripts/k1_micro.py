"""Microbenchmark of the fused scan+reduce kernel (K1) alone.

python scripts/k1_micro.py [--n 1e7] [--k 1000] [--p 64]
Prints per-launch device time (library CUDA events):
  cold   L2 flushed before each launch by writing AND then reading a 256 MiB
         buffer (so no dirty lines of the flush are written back inside K1)
  wcold  L2 flushed by a write only (dirty-line write-back lands inside K1)
  warm   back-to-back launches (D and the codes stay L2-resident)
and the effective GB/s on the algorithmic bytes N*(8 + code bytes) + 4*nnz_j.
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
    ap.add_argument("--n", type=float, nargs="+", default=[1e7])
    ap.add_argument("--k", type=int, default=1000)
    ap.add_argument("--p", type=int, default=64)
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--modes", default="cold,wcold,warm")
    ap.add_argument("--k1-mode", type=int, default=0, help="0 auto, 1 look-back, 2 chunk")
    args = ap.parse_args()
    import torch
    import paper_2310_16238_b200 as sx
    from paper_2310_16238_b200 import _capi, synthetic

    lib = _capi.load()
    l2w = torch.zeros(64 * 1024 * 1024, device="cuda")
    l2r = torch.ones(64 * 1024 * 1024, device="cuda")
    for nf in args.n:
        n = int(nf)
        syn = synthetic.generate(n, args.p, max(1, int(args.k * n / 1e7)), args.density, seed=3,
                                 device="cuda")
        d = syn.sorted_design()
        dd = sx.upload(d)
        info = dd.info()
        h = dd.handle
        rng = np.random.default_rng(1)
        beta = rng.normal(0, 0.05, args.p)
        st = sx.make_state(dd, beta)
        chunked = C.c_int()
        lib.scx_set_k1_mode(h, args.k1_mode, C.byref(chunked))
        out = {"n": n, "k": info["n_strata"], "code_bytes": info["code_bytes"],
               "n_tiles": info["n_tiles"], "dbg": os.environ.get("SCX_K1_DBG", "0"),
               "chunked": chunked.value}
        nnz = float(np.mean(np.diff(d.col_ptr)))
        byts = n * (8 + info["code_bytes"]) + 4 * nnz
        for mode in args.modes.split(","):
            lib.scx_timing_enable(h, 1)
            lib.scx_timing_reset(h)
            for _ in range(args.reps):
                for j in range(args.p):
                    if mode in ("cold", "wcold"):
                        l2w.add_(1)
                        if mode == "cold":
                            l2r.sum()
                        torch.cuda.synchronize()
                    sx.gradient_hessian(dd, st, j)
            tot = C.c_double(); nl = C.c_int64()
            lib.scx_timing_get(h, 0, C.byref(tot), C.byref(nl))
            ms = tot.value / nl.value
            out[mode + "_us"] = round(ms * 1e3, 2)
            out[mode + "_gbs"] = round(byts / (ms * 1e-3) / 1e9, 1)
        lib.scx_timing_enable(h, 0)
        lib.scx_timing_enable(h, 1)
        lib.scx_timing_reset(h)
        for _ in range(5):
            sx.log_partial_likelihood(dd, st)
        lib.scx_timing_get(h, 2, C.byref(tot), C.byref(nl))
        out["k2_us"] = round(tot.value / nl.value * 1e3, 2)
        lib.scx_timing_enable(h, 0)
        print(json.dumps(out), flush=True)
        del st
        dd.close()
        del syn, d
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
