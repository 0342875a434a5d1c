"""One risk-scan launch on the C4 shape (an ncu target).

python scripts/rs_once.py [reps]   # reps back-to-back scans in the launch (default 1)
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    import torch
    import paper_2310_16238_b200 as sx
    from paper_2310_16238_b200 import _capi, synthetic
    lib = _capi.load()
    syn = synthetic.generate(10_000_000, 64, 1000, 0.01, seed=3, device="cuda")
    dd = sx.upload(syn.sorted_design())
    assert dd.set_fit_path(0)
    sx.make_state(dd, np.random.default_rng(1).normal(0, 0.05, 64))
    torch.cuda.synchronize()
    assert lib.scx_risk_prefix_n(dd.handle, reps) == 0
    torch.cuda.synchronize()
    print("ok", reps)


if __name__ == "__main__":
    main()
