"""Per-tile timeline of the risk-suffix scan in CTA 0 (SCX_K1_DBG=32).

python scripts/rs_trace.py  -> for each pass / tile: cycles waiting for the TMA
stage, pass-1 compute, block scan, per-row pass, write-out.
"""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SCX_K1_DBG"] = "32"


def main():
    import paper_2310_16238_b200 as sx
    from paper_2310_16238_b200 import _capi, synthetic
    lib = _capi.load()
    syn = synthetic.generate(10_000_000, 16, 1000, 0.01, seed=3, device="cuda")
    dd = sx.upload(syn.sorted_design())
    sx.make_state(dd, np.random.default_rng(1).normal(0, 0.05, 16))
    for _ in range(3):
        assert lib.scx_risk_prefix(dd.handle) == 0
    import torch
    torch.cuda.synchronize()
    tr = np.zeros((2, 512, 8), np.int64)
    lib.scx_debug_k1_trace(tr.ctypes.data_as(C.POINTER(C.c_longlong)))
    t = tr[0]
    out = {}
    for pas in (0, 1):
        rows = []
        for i in range(64):
            e = t[pas * 64 + i]
            if e[0] == 0:
                break
            rows.append([int(e[1] - e[0]), int(e[2] - e[1]), int(e[3] - e[2]), int(e[4] - e[3]),
                         int(e[5] - e[4]), int(e[0] - t[pas * 64 + i - 1][5]) if i else 0])
        out["fwd" if pas == 0 else "bwd"] = rows
        tot = int(t[pas * 64 + len(rows) - 1][5] - t[pas * 64][0])
        out[("fwd" if pas == 0 else "bwd") + "_total_cycles"] = tot
    print("columns: wait, pass1, blockscan, perrow+smem+sync, writeout, gap_from_prev")
    base = t[0][0]
    for k in list(range(0, 4)) + list(range(64, 84)):
        print(k, [int(x - base) if x else 0 for x in t[k][:6]])
    print(json.dumps(out))


if __name__ == "__main__":
    main()
