"""Per-coordinate phase timeline of one CCD cycle kernel launch (SCX_K1_DBG=16),
CTA 0: loop end -> grid barrier -> rule -> apply -> next coordinate start."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SCX_K1_DBG"] = "16"


def main():
    import paper_2310_16238_b200 as sx
    from paper_2310_16238_b200 import _capi, synthetic
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
    p = int(sys.argv[2]) if len(sys.argv) > 2 else 400
    lib = _capi.load()
    syn = synthetic.generate(n, p, max(1, n // 10000), 0.01, seed=11, device="cuda")
    d = syn.sorted_design()
    dd = sx.upload(d)
    gmax = sx.gamma_max(dd)
    pen = sx.PenaltySpec.shared(p, 0.05 * gmax)
    r = sx.ccd_fit(dd, pen, sx.OptimizerConfig(max_cycles=3))   # the last launch = cycle 3
    buf = np.zeros((2, 512, 8), dtype=np.int64)
    lib.scx_debug_k1_trace(buf.ctypes.data_as(C.POINTER(C.c_int64)))
    t = buf[0, :min(p, 511)]
    start, end, sync, rule, app = t[:, 4], t[:, 0], t[:, 1], t[:, 2], t[:, 3]
    loop = end - start
    bar = sync - end
    dec = rule - sync
    applied = app > 0
    ap = np.where(applied, app - rule, 0)
    nxt = start[1:] - np.where(applied[:-1], app[:-1], rule[:-1])
    print(f"coords {len(t)} applied {applied.sum()}  cycle beta nonzero {int(np.count_nonzero(r.beta))}")
    for name, v in [("tile loop", loop), ("grid barrier", bar), ("reduce+rule", dec),
                    ("apply (applied only)", ap[applied]), ("to next start", nxt)]:
        print(f"{name:22s} median {np.median(v):8.0f} mean {np.mean(v):8.0f} cycles")


if __name__ == "__main__":
    main()
