"""One C4 fit (bench.py's design: N=1e7, p=1e4, K=1e3, 1%, L1 at 0.05 gamma_max)
for an ncu launch list: python scripts/fit_once.py [--n 1e7] [--p 10000]"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=float, default=1e7)
    ap.add_argument("--p", type=int, default=10_000)
    ap.add_argument("--k", type=int, default=1000)
    args = ap.parse_args()
    import paper_2310_16238_b200 as sx
    from paper_2310_16238_b200 import synthetic
    syn = synthetic.generate(int(args.n), args.p, args.k, 0.01, seed=11, device="cuda")
    dd = sx.upload(syn.sorted_design())
    gmax = sx.gamma_max(dd)
    t0 = time.perf_counter()
    r = sx.ccd_fit(dd, sx.PenaltySpec.shared(args.p, 0.05 * gmax), sx.OptimizerConfig())
    print(f"fit {time.perf_counter() - t0:.2f}s cycles {r.cycles_used} stats {dd.fit_path_stats()}",
          flush=True)


if __name__ == "__main__":
    main()
