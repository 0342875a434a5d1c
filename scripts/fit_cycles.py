"""C4-shaped fit for a given number of cycles (a target for ncu launch ranges)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    cycles = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    import paper_2310_16238_b200 as sx
    from paper_2310_16238_b200 import synthetic
    syn = synthetic.generate(10_000_000, 10_000, 1000, 0.01, seed=11, device="cuda")
    dd = sx.upload(syn.sorted_design())
    pen = sx.PenaltySpec.shared(10_000, 0.05 * sx.gamma_max(dd))
    r = sx.ccd_fit(dd, pen, sx.OptimizerConfig(max_cycles=cycles))
    print("cycles", r.cycles_used, dd.fit_path_stats(), flush=True)


if __name__ == "__main__":
    main()
