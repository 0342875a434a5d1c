"""Microbenchmark of the refresh (make_state / refresh_xbeta) at the C4 shape
with the end-of-fit active set (about 19% of the columns nonzero).

python scripts/refresh_micro.py [--n 1e7] [--p 10000] [--active 0.19] [--reps 10]
Prints the per-call device time (CUDA events on the library stream, L2
flushed before each call) and the bytes/s of the column-tile refresh's
algorithmic traffic: 4 B (row index) per entry of an active column + 16 B per
row (eta, D written). The row-slice refresh (default when its copy of the
design was built; SCX_REFRESH_ELL=0 selects the tile refresh) reads every
entry's 2-B column id instead, whatever the active set.
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=float, default=1e7)
    ap.add_argument("--p", type=int, default=10_000)
    ap.add_argument("--k", type=int, default=1000)
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--active", type=float, default=0.19)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import torch
    import paper_2310_16238_b200 as sx
    from paper_2310_16238_b200 import _capi, synthetic

    lib = _capi.load()
    n = int(args.n)
    syn = synthetic.generate(n, args.p, args.k, args.density, seed=3, device="cuda")
    d = syn.sorted_design()
    dd = sx.upload(d)
    rng = np.random.default_rng(1)
    beta = rng.normal(0, 0.02, args.p) * (rng.random(args.p) < args.active)
    nnz_act = int(np.sum(np.diff(d.col_ptr)[beta != 0]))
    dev = torch.device("cuda", 0)
    l2 = torch.zeros(64 * 1024 * 1024, device=dev)
    stream = torch.cuda.ExternalStream(lib.scx_stream(dd.handle), device=dev)
    st = sx.make_state(dd, beta)
    times = []
    for _ in range(args.reps):
        l2.add_(1.0)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        assert lib.scx_refresh_xbeta(dd.handle) == 0
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = float(np.median(times))
    alg = 4.0 * nnz_act + 16.0 * n
    out = {"n": n, "p": args.p, "active_cols": int(np.count_nonzero(beta)), "active_nnz": nnz_act,
           "refresh_ms_median": ms, "refresh_ms_min": float(np.min(times)),
           "algorithmic_bytes": alg, "achieved_gbs": alg / (ms * 1e-3) / 1e9}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
