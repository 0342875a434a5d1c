"""Generate the LARGE-fit parity fixtures from the UNMODIFIED reference (oracle/_ref).

TEST INFRASTRUCTURE ONLY. Run in the build container (needs
oracle/_ref/libstratcox_ref.so, built from /root/reference by `make -C oracle ref`):

    python tests/golden/make_large_fits.py c4_p200        # ~1-2 min on 8 cores
    python tests/golden/make_large_fits.py c2_1e6 c3_1e6  # lowered designs, 1e6 subjects
    python tests/golden/make_large_fits.py c4_p1e4_2cyc   # ~40 min, ~40 GB RAM

A fixture stores the reference's fit (beta, objective trace, cycles, trust,
warnings, gamma_max) and a fingerprint of the reference's SortedDesign
(CRC32 of perm / tie_group_end / stratum_offsets / col_ptr / row indices), NOT
the design itself: the GPU test regenerates the identical input with the
reference's own simulate() (simulate.cpp:9-102, deterministic under a fixed
seed with this image's libstdc++) or, for the lowered configs, with the
numpy subject generator below + the reference's lower_pipeline
(transforms.cpp:64-223), checks the fingerprint, and fits it on the device.

Reference calls: simulate / build_sorted_design (data.cpp:68-147) /
gamma_max (resample.cpp:42-55) / ccd_fit (optimizer.cpp:82-160) with
PenaltySpec::shared(p, frac * gamma_max) and the default OptimizerConfig
(max_cycles 1000, tol 1e-6, trust 1).
"""
from __future__ import annotations

import os
import sys
import time
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

# name -> spec. kind "sim": reference simulate(n, p, density, 0.8, k, 0.3, seed);
# kind "lowered": numpy subjects (subject_data below) -> reference lower_pipeline.
SPECS = {
    "c4_p200": dict(kind="sim", n=10_000_000, p=200, density=0.01, k=1000, seed=11,
                    gamma_frac=0.05, max_cycles=1000, tol=1e-6),
    "c4_p1e4_2cyc": dict(kind="sim", n=10_000_000, p=10_000, density=0.01, k=1000, seed=11,
                         gamma_frac=0.05, max_cycles=2, tol=1e-6),
    "c2_1e6": dict(kind="lowered", subjects=1_000_000, p=1000, density=0.01, bins=20,
                   split=False, seed=11, gamma_frac=0.05, max_cycles=1000, tol=1e-6),
    "c3_1e6": dict(kind="lowered", subjects=1_000_000, p=500, density=0.01, bins=20,
                   split=True, seed=11, gamma_frac=0.05, max_cycles=1000, tol=1e-6),
}


def subject_data(n, p, density, bins, seed):
    """Subjects with simulate.cpp's model (binary X, beta ~ N(0,1) x Bern(0.2),
    exponential times, censoring), integer-day times over `bins` days (heavy
    ties). Shared with bench.py's configs 2-3 (same generator, same seed)."""
    rng = np.random.default_rng(seed)
    col_ptr = [0]
    rows = []
    eta = np.zeros(n)
    beta = rng.normal(0.0, 1.0, p) * (rng.random(p) < 0.2)
    for j in range(p):
        k = rng.binomial(n, density)
        r = np.unique(rng.integers(0, n, size=k))
        rows.append(r)
        col_ptr.append(col_ptr[-1] + r.shape[0])
        eta[r] += beta[j] * 0.3
    t = rng.exponential(1.0, n) / np.exp(eta)
    t = np.minimum(np.ceil(t / np.quantile(t, 0.9) * bins * 0.8), bins)
    c = rng.integers(1, bins + 1, n).astype(float)
    time_ = np.minimum(t, c)
    event = (t <= c).astype(np.uint8)
    return dict(time=time_.astype(np.float64), event=event,
                stratum=np.ones(n, np.int32), col_ptr=np.array(col_ptr, np.int64),
                row_idx=np.concatenate(rows).astype(np.int64))


def fingerprint(a):
    """CRC32s of the SortedDesign's integer arrays (bit-exact indexing)."""
    def crc(x):
        return np.uint32(zlib.crc32(np.ascontiguousarray(x).view(np.uint8)))
    return dict(fp_perm=crc(a["perm"].astype(np.int64)),
                fp_tie_end=crc(a["tie_end"].astype(np.int64)),
                fp_offsets=crc(a["offsets"].astype(np.int64)),
                fp_col_ptr=crc(a["col_ptr"].astype(np.int64)),
                fp_row_idx=crc(a["row_idx"].astype(np.int64)),
                fp_event=crc(a["event"].astype(np.uint8)),
                n=np.int64(a["n"]), p=np.int64(a["p"]), k=np.int64(a["k"]),
                nnz=np.int64(a["col_ptr"][-1]))


def lowered_dataset(ref, spec):
    from oracle.oracle_py import Dataset
    s = subject_data(spec["subjects"], spec["p"], spec["density"], spec["bins"], spec["seed"])
    subj = Dataset(s["time"], s["event"], s["stratum"], s["col_ptr"], s["row_idx"],
                   np.ones(int(s["col_ptr"][-1])))
    cuts = np.arange(spec["bins"] + 1, dtype=np.float64)
    splits = {0: list(cuts[1:-1])} if spec["split"] else None
    return ref.lower_pipeline(subj, cuts, splits, subject=np.arange(1, spec["subjects"] + 1))


def reference_design(ref, spec):
    """(handle, arrays) of the reference's SortedDesign for a spec."""
    if spec["kind"] == "sim" and spec["p"] * spec["n"] * spec["density"] > 2e8:
        # lean path for 1e9 nonzeros: simulate and sort inside the reference
        # without a numpy copy of the input dataset
        import ctypes as C
        hd = C.c_void_p()
        ref._chk(ref.L.ref_simulate(spec["n"], spec["p"], spec["density"], 0.8, spec["k"], 0.3,
                                    spec["seed"], C.byref(hd)))
        h = C.c_void_p()
        rc = ref.L.ref_design_build(hd, C.byref(h))
        ref.L.ref_dataset_free(hd)
        ref._chk(rc)
        return h, ref.design_arrays(h)
    if spec["kind"] == "sim":
        ds = ref.simulate(spec["n"], spec["p"], spec["density"], 0.8, spec["k"], 0.3,
                          spec["seed"])
    else:
        low = lowered_dataset(ref, spec)
        ds = low[0] if isinstance(low, tuple) else low
    return ref.build_design(ds)


def make(name):
    from oracle.oracle_py import Ref
    ref = Ref()
    spec = SPECS[name]
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    h, a = reference_design(ref, spec)
    t_design = time.perf_counter() - t0
    fp = fingerprint(a)
    p = a["p"]
    del a
    t0 = time.perf_counter()
    gmax = ref.gamma_max(h, workers=threads)
    t_gmax = time.perf_counter() - t0
    gamma = np.full(p, spec["gamma_frac"] * gmax)
    t0 = time.perf_counter()
    r = ref.ccd_fit(h, gamma, p, max_cycles=spec["max_cycles"], tol=spec["tol"],
                    workers=threads)
    t_fit = time.perf_counter() - t0
    ref.free_design(h)
    out = dict(fp, gamma_max=np.float64(gmax), gamma=gamma, beta=r["beta"], trace=r["trace"],
               cycles=np.int64(r["cycles"]), converged=np.int64(r["converged"]),
               trust=r["trust"], n_warnings=np.int64(r["n_warnings"]),
               max_cycles=np.int64(spec["max_cycles"]), tol=np.float64(spec["tol"]),
               fit_seconds=np.float64(t_fit), gamma_max_seconds=np.float64(t_gmax),
               design_seconds=np.float64(t_design), threads=np.int64(threads))
    path = os.path.join(HERE, f"large_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: cycles={r['cycles']} converged={r['converged']} "
          f"nonzero={int(np.count_nonzero(r['beta']))}/{p} fit {t_fit:.1f}s "
          f"gamma_max {t_gmax:.1f}s design {t_design:.1f}s threads {threads} -> {path}",
          flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["c4_p200"]:
        make(nm)
