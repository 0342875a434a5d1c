"""Parity of the BENCHMARKED configuration at full size: BASELINE config 4
(N=1e7 rows, K=1e3 strata, p=1e4 indicator covariates, 1% density, L1 at
0.05 * gamma_max) regenerated with the reference's own simulate() and
build_sorted_design (oracle/_ref), fitted on the device for the first two
CCD cycles, against the unmodified reference's two-cycle ccd_fit
(tests/golden/large_c4_p1e4_2cyc.npz, made by tests/golden/make_large_fits.py:
1363 s of reference fit on 8 cores). Writes profiles/r02_parity_c4_full.json.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2310_16238_b200 as sx
    from oracle.oracle_py import Ref
    from tests import _golden as G
    from tests.golden.make_large_fits import SPECS, fingerprint, reference_design

    z = dict(np.load(os.path.join(ROOT, "tests", "golden", "large_c4_p1e4_2cyc.npz")))
    ref = Ref()
    t0 = time.perf_counter()
    h, a = reference_design(ref, SPECS["c4_p1e4_2cyc"])
    ref.free_design(h)
    t_design = time.perf_counter() - t0
    fp = fingerprint(a)
    same = all(int(v) == int(z[k]) for k, v in fp.items())
    dd = sx.upload(G.sorted_design(a, values=False))
    del a
    rs = dd.set_fit_path(0)
    gmax = sx.gamma_max(dd)
    t0 = time.perf_counter()
    r = sx.ccd_fit(dd, sx.PenaltySpec(z["gamma"]),
                   sx.OptimizerConfig(max_cycles=int(z["max_cycles"]), tolerance=float(z["tol"])))
    t_fit = time.perf_counter() - t0
    stats = dd.fit_path_stats()
    db = np.abs(r.beta - z["beta"])
    out = {
        "design": "reference simulate(1e7, 1e4, 0.01, 0.8, 1e3, 0.3, seed 11) + build_sorted_design",
        "design_fingerprint_matches_fixture": bool(same),
        "reference": {"cycles": int(z["cycles"]), "fit_seconds_8_threads": float(z["fit_seconds"]),
                      "gamma_max_seconds": float(z["gamma_max_seconds"]),
                      "nonzero": int(np.count_nonzero(z["beta"]))},
        "device": {"cycles": r.cycles_used, "fit_seconds": t_fit, "fit_path_stats": stats,
                   "risk_suffix_cycle": bool(rs), "nonzero": int(np.count_nonzero(r.beta))},
        "gamma_max_rel_diff": abs(gmax - float(z["gamma_max"])) / float(z["gamma_max"]),
        "max_abs_dbeta": float(db.max()), "beta_atol": 1e-8,
        "supports_equal": bool(np.array_equal(r.beta != 0, z["beta"] != 0)),
        "max_rel_dtrace": float(np.max(np.abs(np.asarray(r.objective_trace) - z["trace"]) /
                                       np.abs(z["trace"]))),
        "max_abs_dtrust": float(np.abs(r.trust - z["trust"]).max()),
        "design_seconds": t_design,
    }
    out["pass"] = bool(same and r.cycles_used == int(z["cycles"]) and out["max_abs_dbeta"] <= 1e-8
                       and out["supports_equal"] and out["max_rel_dtrace"] <= 1e-10)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "r02_parity_c4_full.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out), flush=True)
    dd.close()


if __name__ == "__main__":
    main()
