"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run in the build container (needs oracle/_ref/libstratcox_ref.so, built from
/root/reference by `make -C oracle ref`):

    python tests/golden/make_golden.py

Every fixture is produced by calling the reference's own C++ API
(simulate, oracles::random_dataset, build_sorted_design, make_state,
gradient_hessian, naive_*, log_partial_likelihood, ccd_fit, gamma_max,
segmented_inclusive_scan) through oracle/ref_capi.cpp. The seeds and shapes
restate the reference tests cited beside each block.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle_py import Dataset, Ref  # noqa: E402

R = Ref()


def design_fields(prefix, a, store_values=True):
    out = {
        f"{prefix}offsets": a["offsets"],
        f"{prefix}event": a["event"],
        f"{prefix}tie_end": a["tie_end"].astype(np.int32),
        f"{prefix}head": a["head"],
        f"{prefix}time": a["time"],
        f"{prefix}perm": a["perm"].astype(np.int32),
        f"{prefix}col_ptr": a["col_ptr"],
        f"{prefix}row_idx": a["row_idx"].astype(np.int32),
    }
    if store_values:
        out[f"{prefix}values"] = a["values"]
    return out


def dataset_fields(prefix, ds: Dataset):
    return {f"{prefix}in_time": ds.time, f"{prefix}in_event": ds.event,
            f"{prefix}in_stratum": ds.stratum, f"{prefix}in_col_ptr": ds.col_ptr,
            f"{prefix}in_row_idx": ds.row_idx.astype(np.int32), f"{prefix}in_values": ds.values}


def random_instances():
    """Scan-vs-naive equivalence instances: proj/tests/test_likelihood.cpp:91-113
    (seed 31 shapes) and proj/tests/acceptance.cpp:122-168 (seed 202 shapes,
    strata {1,5,50}); each instance is oracles::random_dataset."""
    rng = np.random.default_rng(2310)
    out = {}
    specs = []
    for trial in range(40):
        strata = [1, 5, 11][trial % 3]
        n = 20 + (trial % 7) * 25
        p = 1 + trial % 5
        specs.append((31_000 + trial, n, strata, p))
    for trial in range(30):
        strata = [1, 5, 50][trial % 3]
        n = 50 + int(rng.integers(0, 151))
        p = 1 + int(rng.integers(0, 10))
        specs.append((202_000 + trial, n, strata, p))
    for i, (seed, n, strata, p) in enumerate(specs):
        ds = R.random_dataset(seed, n, strata, p)
        h, a = R.build_design(ds)
        beta = rng.normal(0.0, 0.5, size=p)
        xb, ex = R.make_state(h, beta, n)
        g = np.empty(p); hh = np.empty(p); ng = np.empty(p); nh = np.empty(p)
        for j in range(p):
            g[j], hh[j] = R.gradient_hessian(h, beta, xb, ex, j)
            ng[j], nh[j] = R.naive_gradient_hessian(h, beta, xb, ex, j)
        ll = R.log_partial_likelihood(h, beta, xb, ex)
        nll = R.naive_log_partial_likelihood(h, beta, xb, ex)
        pre = f"r{i}_"
        out.update(dataset_fields(pre, ds))
        out.update(design_fields(pre, a))
        out.update({f"{pre}beta": beta, f"{pre}xbeta": xb, f"{pre}exp_xbeta": ex,
                    f"{pre}grad": g, f"{pre}hess": hh, f"{pre}naive_grad": ng,
                    f"{pre}naive_hess": nh, f"{pre}ll": np.array(ll),
                    f"{pre}naive_ll": np.array(nll), f"{pre}spec": np.array([seed, n, strata, p])})
        R.free_design(h)
    out["count"] = np.array(len(specs))
    np.savez_compressed(os.path.join(HERE, "random_instances.npz"), **out)
    print("random_instances.npz", len(specs))


def scan_instances():
    """Segmented scan vs the reference chunked scan: worked example
    (proj/tests/test_scan.cpp:55-63, acceptance.cpp:62-68) and random flag
    patterns (test_scan.cpp:104-127 shapes), chunk 4096."""
    rng = np.random.default_rng(101)
    out = {}
    vals = np.array([3, 1, 7, 0, 4, 1, 6, 3], float)
    flags = np.array([1, 0, 1, 0, 0, 1, 0, 0], np.uint8)
    out["worked_values"] = vals
    out["worked_flags"] = flags
    out["worked_out"] = R.segmented_scan(vals, flags)
    cases = 0
    for n in [1, 2, 17, 4095, 4096, 4097, 8192 + 5, 30001, 100_003]:
        big = n > 5000
        for seg in [1, max(1, n // 100), max(1, n // 2), n]:
            integral = big or cases % 3 == 0
            v = rng.integers(0, 10, n).astype(float) if integral else rng.random(n)
            f = np.zeros(n, np.uint8)
            f[0] = 1
            f[rng.integers(0, n, seg - 1)] = 1
            out[f"s{cases}_v"] = v
            out[f"s{cases}_f"] = f
            out[f"s{cases}_out"] = R.segmented_scan(v, f)
            cases += 1
    out["count"] = np.array(cases)
    np.savez_compressed(os.path.join(HERE, "scan_instances.npz"), **out)
    print("scan_instances.npz", cases)


def fits():
    """ccd_fit trajectories: acceptance.cpp:321-389 shapes (criterion 5:
    n=2000, p=5, density 0.3, beta_sparsity 0, K in {1,10}, seed 500+K,
    tolerance 1e-8, unpenalised and shared gamma=2 at 1e-7) and
    acceptance.cpp:476-531 (criterion 7: n=3000, p=8, density 0.2,
    beta_sparsity 0.25, K=7, seed 700, gamma in {0,1})."""
    out = {}
    specs = []
    for k in (1, 10):
        specs.append(dict(name=f"c5_k{k}_none", n=2000, p=5, density=0.3, bs=0.0, strata=k,
                          seed=500 + k, gamma=0.0, tol=1e-8, max_cycles=5000))
        specs.append(dict(name=f"c5_k{k}_l1", n=2000, p=5, density=0.3, bs=0.0, strata=k,
                          seed=500 + k, gamma=2.0, tol=1e-7, max_cycles=5000))
    for gm in (0.0, 1.0):
        specs.append(dict(name=f"c7_g{int(gm)}", n=3000, p=8, density=0.2, bs=0.25, strata=7,
                          seed=700, gamma=gm, tol=1e-6, max_cycles=1000))
    # BASELINE config 1 shape (N=1e4, p=100, K=10); L2 has no reference -> L1 path
    specs.append(dict(name="cfg1_l1", n=10_000, p=100, density=0.05, bs=0.8, strata=10, seed=11,
                      gamma=None, tol=1e-8, max_cycles=1000))
    names = []
    for s in specs:
        ds = R.simulate(s["n"], s["p"], s["density"], s["bs"], s["strata"], 0.3, s["seed"])
        h, a = R.build_design(ds)
        gm = s["gamma"]
        if gm is None:
            gmax = R.gamma_max(h)
            gm = 0.05 * gmax
            out[f"{s['name']}_gamma_max"] = np.array(gmax)
        gamma = np.full(s["p"], gm)
        r = R.ccd_fit(h, gamma, s["p"], max_cycles=s["max_cycles"], tol=s["tol"])
        pre = s["name"] + "_"
        out.update(design_fields(pre, a, store_values=False))
        out.update({f"{pre}gamma": gamma, f"{pre}tol": np.array(s["tol"]),
                    f"{pre}max_cycles": np.array(s["max_cycles"]), f"{pre}beta": r["beta"],
                    f"{pre}trace": r["trace"], f"{pre}cycles": np.array(r["cycles"]),
                    f"{pre}converged": np.array(r["converged"]), f"{pre}trust": r["trust"]})
        # gradient at beta = 0 for every covariate (gamma_max building block)
        p = s["p"]
        b0 = np.zeros(p)
        xb, ex = R.make_state(h, b0, s["n"])
        g0 = np.array([R.gradient_hessian(h, b0, xb, ex, j) for j in range(p)])
        out[f"{pre}g0"] = g0
        R.free_design(h)
        names.append(s["name"])
        print("fit", s["name"], "cycles", r["cycles"], "nonzero", int(np.count_nonzero(r["beta"])))
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "fits.npz"), **out)


def known_answers():
    """Hand-worked cases re-stated from the reference unit tests."""
    out = {}
    # test_data.cpp:30-47 — sort, heads, tie groups, offsets
    def tiny(time, event, stratum, cols=None):
        n = len(time)
        cols = cols or []
        cp = [0]
        ri, va = [], []
        for c in cols:
            for r, v in c:
                ri.append(r)
                va.append(v)
            cp.append(len(ri))
        return Dataset(np.array(time, float), np.array(event, np.uint8),
                       np.array(stratum, np.int32), np.array(cp, np.int64),
                       np.array(ri, np.int64), np.array(va, float))
    cases = {
        "sort1": tiny([2, 5, 3], [1, 1, 0], [1, 1, 1]),
        "ties": tiny([4, 4, 1], [1, 1, 1], [1, 1, 1]),
        "heads": tiny([3, 7, 5], [1, 1, 1], [1, 1, 2]),
        # test_likelihood.cpp:62-75: x = 1 on the time-1 row
        "handworked": tiny([3, 2, 1], [1, 1, 1], [1, 1, 1], cols=[[(2, 1.0)]]),
        # test_likelihood.cpp:77-89: zero column
        "zerocol": tiny([3, 2, 1], [1, 1, 1], [1, 1, 1], cols=[[]]),
    }
    for name, ds in cases.items():
        h, a = R.build_design(ds)
        out.update(design_fields(name + "_", a))
        R.free_design(h)
    np.savez_compressed(os.path.join(HERE, "known_answers.npz"), **out)
    print("known_answers.npz")


if __name__ == "__main__":
    known_answers()
    scan_instances()
    random_instances()
    fits()
