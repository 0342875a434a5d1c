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
os.environ["SCX_K1_DBG"] = os.environ.get("SCX_K1_DBG", "32")


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
    base = t[0][0]
    print("group-0 forward tiles: [wait_start, data_ready, pass1_done, scan_done, carry_ready, perrow_done, stored] (cycles from start)")
    for k in range(20):
        if t[k][0] == 0:
            break
        print(k, [int(x - base) if x else 0 for x in t[k][:7]])


if __name__ == "__main__":
    main()
