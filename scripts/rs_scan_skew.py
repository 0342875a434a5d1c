"""Per-CTA timing of the in-fit risk scans (profiling build, SCX_K1_DBG=512).

python scripts/rs_scan_skew.py [--cycles 30]
Runs the C4-shaped fit for cycles-1 cycles, then one more with the trace on,
and prints, for the launch's first 4 scans, the spread of the CTAs' start and
end times (globaltimer, ns) and of their durations.
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["SCX_K1_DBG"] = "512"
os.environ.setdefault("SCX_LIB", os.path.join(ROOT, "paper_2310_16238_b200", "libstratcox_b200_trace.so"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cycles", type=int, default=30)
    args = ap.parse_args()
    import paper_2310_16238_b200 as sx
    from paper_2310_16238_b200 import _capi, synthetic
    lib = _capi.load()
    syn = synthetic.generate(10_000_000, 10_000, 1000, 0.01, seed=11, device="cuda")
    d = syn.sorted_design()
    dd = sx.upload(d)
    # the library's stratum-aligned chunks (capi.cu: nearest head to each share)
    off = np.asarray(syn.offsets, np.int64)
    n, k, G = int(off[-1]), len(off) - 1, 148
    ch, q = [0], 0
    for c in range(1, G):
        target = ch[-1] + (n - ch[-1]) // (G - c + 1)
        while q < k and off[q + 1] <= target:
            q += 1
        h = off[q]
        if q + 1 <= k and off[q + 1] - target < target - h:
            h = off[q + 1]
        ch.append(int(h))
    ch.append(n)
    rows = np.diff(np.array(ch))
    pen = sx.PenaltySpec.shared(10_000, 0.05 * sx.gamma_max(dd))
    r = sx.ccd_fit(dd, pen, sx.OptimizerConfig(max_cycles=args.cycles))
    tr = np.zeros((2, 512, 8), np.int64)
    lib.scx_debug_k1_trace(tr.ctypes.data_as(C.POINTER(C.c_longlong)))
    t = tr[0][:148]
    for k in range(4):
        st, en = t[:, 2 * k].astype(np.float64), t[:, 2 * k + 1].astype(np.float64)
        if not st.any():
            break
        dur = (en - st) / 1e3
        print(f"scan {k}: start spread {(st.max() - st.min()) / 1e3:.1f} us, end spread "
              f"{(en.max() - en.min()) / 1e3:.1f} us, first start -> last end "
              f"{(en.max() - st.min()) / 1e3:.1f} us; duration min/med/max "
              f"{dur.min():.1f}/{np.median(dur):.1f}/{dur.max():.1f} us, slowest CTA {int(dur.argmax())}")
        print(f"   chunk rows min/med/max {rows.min()}/{int(np.median(rows))}/{rows.max()}; "
              f"corr(rows, duration) {np.corrcoef(rows, dur)[0, 1]:.2f}; us per 1k rows "
              f"{np.median(dur / rows * 1e3):.3f}; rows of the slowest {rows[dur.argmax()]}")
    print("cycles", r.cycles_used)


if __name__ == "__main__":
    main()
