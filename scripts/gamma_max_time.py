"""gamma_max at C4 (N=1e7, p=1e4, K=1e3, 1%): the risk-suffix launch (fit path 0)
vs one fused-scan pass per column (fit path 1). python scripts/gamma_max_time.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2310_16238_b200 as sx
    from paper_2310_16238_b200 import synthetic
    syn = synthetic.generate(10_000_000, 10_000, 1000, 0.01, seed=11, device="cuda")
    dd = sx.upload(syn.sorted_design())
    out = {}
    for path in (0, 1, 0):
        dd.set_fit_path(path)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        g = sx.gamma_max(dd)
        out[path] = (g, time.perf_counter() - t0)
    print(f"gamma_max risk-suffix {out[0][1] * 1e3:.1f} ms, fused scan per column "
          f"{out[1][1] * 1e3:.1f} ms, values {out[0][0]!r} {out[1][0]!r} rel "
          f"{abs(out[0][0] - out[1][0]) / out[1][0]:.2e}", flush=True)


if __name__ == "__main__":
    main()
