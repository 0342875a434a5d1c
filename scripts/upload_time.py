"""Upload phases of the C4 design from host arrays (SCX_UPLOAD_TRACE=1)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SCX_UPLOAD_TRACE"] = "1"


def main():
    import torch
    import paper_2310_16238_b200 as sx
    from paper_2310_16238_b200 import synthetic
    syn = synthetic.generate(10_000_000, 10_000, 1000, 0.01, seed=11, device="cuda")
    d = syn.sorted_design()
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dd = sx.DeviceDesign(d)
        torch.cuda.synchronize()
        print(f"DeviceDesign {time.perf_counter() - t0:.3f} s", file=sys.stderr, flush=True)
        t0 = time.perf_counter()
        g = sx.gamma_max(dd)
        print(f"gamma_max {time.perf_counter() - t0:.3f} s", file=sys.stderr, flush=True)
        dd.close()


if __name__ == "__main__":
    main()
