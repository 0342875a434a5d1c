"""Per-tile timeline of one K1 launch (SCX_K1_DBG=8): clock64 events of CTAs 0
and 73, relative to the CTA's start (cycles)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SCX_K1_DBG"] = "8"


def main():
    import paper_2310_16238_b200 as sx
    from paper_2310_16238_b200 import _capi, synthetic
    n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10_000_000
    mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    lib = _capi.load()
    syn = synthetic.generate(n, 8, max(1, n // 10000), 0.01, seed=3, device="cuda")
    d = syn.sorted_design()
    dd = sx.upload(d)
    ch = C.c_int()
    lib.scx_set_k1_mode(dd.handle, mode, C.byref(ch))
    st = sx.make_state(dd, np.random.default_rng(1).normal(0, 0.05, 8))
    for _ in range(3):
        sx.gradient_hessian(dd, st, 1)
    buf = np.zeros((2, 512, 8), dtype=np.int64)
    lib.scx_debug_k1_trace(buf.ctypes.data_as(C.POINTER(C.c_int64)))
    names = ["wg_full", "wg_pass1", "wg_carry", "wg_pass2", "lb_full", "lb_agg", "lb_done", "prod"]
    print("chunked", ch.value)
    for ci in range(2):
        t0 = buf[ci, 511, 0]
        print(f"CTA {[0, 73][ci]}: start->end {buf[ci, 511, 1] - t0} cycles")
        for i in range(0, 511):
            row = buf[ci, i]
            if not row.any():
                break
            rel = [int(x - t0) if x else -1 for x in row]
            print(i, " ".join(f"{names[k]}={rel[k]}" for k in range(8) if rel[k] >= 0))


if __name__ == "__main__":
    main()
