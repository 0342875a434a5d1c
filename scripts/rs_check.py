"""Risk-suffix (g', g'') vs the exact fused scan on a synthetic design.
python scripts/rs_check.py [--n 1e7] [--k 1000] [--p 32]"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=float, default=1e7)
    ap.add_argument("--k", type=int, default=1000)
    ap.add_argument("--p", type=int, default=32)
    ap.add_argument("--scale", type=float, default=0.05)
    args = ap.parse_args()
    import paper_2310_16238_b200 as sx
    from paper_2310_16238_b200 import synthetic
    syn = synthetic.generate(int(args.n), args.p, args.k, 0.01, seed=3, device="cuda")
    dd = sx.upload(syn.sorted_design())
    assert dd.set_fit_path(0)
    out = {}
    for name, scale in (("beta0", 0.0), ("beta_rand", args.scale)):
        beta = np.random.default_rng(1).normal(0, scale, args.p) if scale else np.zeros(args.p)
        st = sx.make_state(dd, beta)
        eg, eh = [], []
        for j in range(args.p):
            a = sx.gradient_hessian(dd, st, j)
            b = sx.risk_suffix_gradient_hessian(dd, st, j)
            eg.append(abs(a.gradient - b.gradient) / max(1.0, abs(a.gradient)))
            eh.append(abs(a.hessian - b.hessian) / max(1.0, abs(a.hessian)))
        out[name] = {"max_rel_g": float(max(eg)), "max_rel_h": float(max(eh)),
                     "worst_j": int(np.argmax(eh))}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
