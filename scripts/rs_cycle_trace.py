"""Where a risk-suffix CCD cycle spends its time (SCX_K1_DBG=256).

python scripts/rs_cycle_trace.py [--n 1e7 --p 10000 --k 1000]
Runs the C4-shaped fit for a few cycles, then one more cycle with the trace on,
and prints the per-round phase totals (cycles) of CTA 0 for the first 512
rounds of the last launch: gradient round (eval, barrier+decide), full
evaluation (eval, barrier+rule), apply, scan.
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SCX_K1_DBG"] = os.environ.get("SCX_K1_DBG", "256")
os.environ.setdefault("SCX_LIB", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2310_16238_b200", "libstratcox_b200_trace.so"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=float, default=1e7)
    ap.add_argument("--p", type=int, default=10000)
    ap.add_argument("--k", type=int, default=1000)
    ap.add_argument("--cycles", type=int, default=3)
    args = ap.parse_args()
    import torch
    import paper_2310_16238_b200 as sx
    from paper_2310_16238_b200 import _capi, synthetic
    lib = _capi.load()
    syn = synthetic.generate(int(args.n), args.p, args.k, 0.01, seed=11, device="cuda")
    d = syn.sorted_design()
    dd = sx.upload(d)
    gmax = sx.gamma_max(dd)
    pen = sx.PenaltySpec.shared(args.p, 0.05 * gmax)
    r = sx.ccd_fit(dd, pen, sx.OptimizerConfig(max_cycles=args.cycles))
    torch.cuda.synchronize()
    tr = np.zeros((2, 512, 8), np.int64)
    lib.scx_debug_k1_trace(tr.ctypes.data_as(C.POINTER(C.c_longlong)))
    t = tr[1]
    # rounds of the last launch (the kernel clears the trace at launch); the
    # round index counts grid reductions, so full evaluations leave gaps
    n = int(np.max(np.nonzero(t[:, 0])[0])) + 1 if t[:, 0].any() else 0
    ph = {"grad_eval": 0, "grad_barrier_decide": 0, "full_eval": 0, "full_barrier_rule": 0,
          "apply": 0, "scan": 0}
    cnt = {k: 0 for k in ph}
    nskip = 0
    for i in range(n):
        e = t[i]
        if not e[0]:
            continue
        for key, a, b in (("grad_eval", 0, 1), ("grad_barrier_decide", 1, 2), ("full_eval", 2, 3),
                          ("full_barrier_rule", 3, 4), ("apply", 4, 5), ("scan", 5, 6)):
            if e[b] and e[a] and e[b] > e[a]:
                ph[key] += e[b] - e[a]
                cnt[key] += 1
        nskip += int(e[7])
    tot = int(t[n - 1][6] or t[n - 1][4] or t[n - 1][2]) - int(t[0][0])
    print(f"rounds={n} skipped={nskip} total_cycles={tot} ({tot / 1.965e3:.0f} us)")
    for k, v in ph.items():
        print(f"  {k:22s} {int(v):>10d} cycles {int(v) / max(1, n):8.0f}/round  {v / max(1, tot):.1%}"
              f"  n={cnt[k]} {int(v) / max(1, cnt[k]) / 1.965e3:.1f} us each")
    r0 = tr[0][:n]
    if r0[:, 0].any():  # SCX_K1_DBG bit 1024: inside the gradient rounds
        ok = (r0[:, 0] > 0) & (t[:n, 0] > 0)
        setup = (r0[ok, 0] - t[:n, 0][ok]) / 1.965e3
        ent = (r0[ok, 1] - r0[ok, 0]) / 1.965e3
        bs = (r0[ok, 2] - r0[ok, 1]) / 1.965e3
        print(f"  grad round inside: setup {setup.mean():.1f} us, entries {ent.mean():.1f} us, "
              f"block sum {bs.mean():.1f} us (n={int(ok.sum())})")
    print("stats", dd.fit_path_stats(), "cycles", r.cycles_used)


if __name__ == "__main__":
    main()
