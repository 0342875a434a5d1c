#!/usr/bin/env python
"""Benchmark: stratified Cox L1 CCD fit at BASELINE config 4 on B200.

Workload (BASELINE.json configs[3], the shape its metric "at N=10M" is quoted
on): N = 1e7 rows, p = 1e4 sparse binary indicator covariates at 1% density
(1e9 nonzeros), K = 1e3 strata, L1 penalty gamma = 0.05 * gamma_max, full CCD
fit from beta = 0 (reference defaults: tolerance 1e-6, trust 1).

One "step" = one complete ccd_fit (every cycle: p fused scan+reduce
evaluations, on-device coordinate rule, eta/D update, cycle log-likelihood).
  value   grad+Hessian evaluations per second over the fit, design resident in
          HBM (CUDA events on the library's stream; L2 flushed by a 256 MiB
          write then a 256 MiB read before every step)
  e2e     the same metric through the public C-ABI from pinned host buffers:
          design upload (H2D) + fit + coefficient download (D2H) per step
  roofline  the fused scan+reduce kernel (K1) timed alone with L2 flushed
          before each launch, algorithmic bytes N*(8 + code bytes) + 4*nnz_j
          per launch vs the measured HBM copy bandwidth
  cpu_baseline  the reference (oracle/_ref: unmodified stratcox compiled -O3
          -fopenmp) on a bounded sample of the same workload (N=1e7, K=1e3,
          1% density, 32 covariates) with run_benchmark semantics, all cores

--impl reference runs the reference CPU arm only (rank 0), same metric.
Multi-GPU (torchrun, N>1): rows sharded at stratum boundaries, 32-byte
NCCL partial exchange per coordinate; total work fixed ("strong").
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("CCD fit wall time (s) and grad+Hessian evals/sec at N=10M; "
          "fused-scan HBM GB/s vs peak")
WORKLOAD = ("C4: stratified Cox L1 CCD fit, N=1e7 rows, p=1e4 sparse indicator covariates "
            "(1% density), K=1e3 strata, gamma=0.05*gamma_max, beta0=0, tol=1e-6")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ---------------------------------------------------------------- CPU reference arm
def reference_sample(n, p_sample, k, density, seed, threads):
    """Bounded sample of the C4 workload on the reference (oracle/_ref)."""
    from oracle.oracle_py import Ref

    ref = Ref()
    t0 = time.perf_counter()
    ds = ref.simulate(n, p_sample, density, 0.8, k, 0.3, seed)
    h, _ = ref.build_design(ds)
    del ds
    gmax = ref.gamma_max(h, workers=threads)
    return ref, h, 0.05 * gmax, time.perf_counter() - t0


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n, k, dens = args.n, args.k, args.density
    p_sample, sweep = 32, args.ref_sweep
    ref, h, gamma, setup = reference_sample(n, p_sample, k, dens, 11, threads)
    per = ref.time_iterations(h, gamma, args.warmup + args.steps, sweep, threads)
    timed = per[args.warmup:]
    sec_per_eval = float(np.mean(timed))
    value = 1.0 / sec_per_eval
    sample = (f"reference stratcox (oracle/_ref, -O3 -fopenmp) on N={n}, K={k}, density {dens}, "
              f"{p_sample} covariates; each step = {sweep} CCD coordinate iterations "
              f"(benchmark.cpp:27-41 semantics) at gamma=0.05*gamma_max; setup {setup:.1f}s excluded")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec_per_eval * sweep * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "n_rows": n, "strata": k, "density": dens,
                   "sample_covariates": p_sample, "l2_flush": "n/a (CPU)"},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "fit_wall_s_extrapolated": None,
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- configs 1-3
CONFIGS = {
    "c1": dict(workload="C1: stratified Cox, N=1e4 rows, p=100 sparse covariates (5%), K=10 strata, "
                        "L2 prior (ridge, l2=1 per coefficient: a N(0,1) prior) CCD fit; the "
                        "reference has no L2 prior, so its arm times the same evaluations "
                        "under its L1 rule",
               subjects=10_000, p=100, density=0.05, bins=None, strata=10, split=False),
    "c2": dict(workload="C2: Cox with time-varying covariates recast as stratified: 1e6 subjects, "
                        "integer-day times over 20 intervals (make_time_varying + augment_to_strata, "
                        "~4-5 counting-process rows per subject, strata = intervals), p=1e3 (1%), L1 fit",
               subjects=1_000_000, p=1000, density=0.01, bins=20, strata=None, split=False),
    "c3": dict(workload="C3: discrete-time time-varying coefficients: 1e6 subjects x 20 time bins, "
                        "covariate 0 split at all 19 interior cuts (split_time_varying_coefficient), "
                        "p=500+19 (1%), augmented to strata, L1 fit",
               subjects=1_000_000, p=500, density=0.01, bins=20, strata=None, split=True),
}


def subject_data(n, p, density, bins, strata, seed):
    """Synthetic subjects with the simulate.cpp model (binary X, beta ~ N(0,1)
    x Bern(0.2), exponential times, uniform censoring); integer-day times over
    `bins` days (heavy ties) for the time-varying configs."""
    import paper_2310_16238_b200 as sx
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
    if bins:
        t = np.minimum(np.ceil(t / np.quantile(t, 0.9) * bins * 0.8), bins)
        c = rng.integers(1, bins + 1, n).astype(float)
    else:
        c = rng.uniform(0, np.quantile(t, 0.95), n)
    time_ = np.minimum(t, c)
    event = (t <= c).astype(np.uint8)
    stratum = (np.arange(n) % (strata or 1) + 1).astype(np.int32)
    return sx.SurvivalDataset(time=time_.astype(np.float64), event=event, stratum=stratum,
                              col_ptr=np.array(col_ptr, np.int64),
                              row_idx=np.concatenate(rows).astype(np.int64), values=None,
                              subject=np.arange(1, n + 1, dtype=np.int64))


def run_small_config(args):
    """One JSON line for BASELINE config 1, 2 or 3 (1 GPU): fit wall time and
    coordinate evaluations per second, e2e from host arrays (lowering + sort +
    upload + fit), the fused-scan roofline on that design, and the reference
    CPU on the same lowered design (oracle/_ref, cpu_baseline leg)."""
    import ctypes as C

    import torch
    import paper_2310_16238_b200 as sx
    from paper_2310_16238_b200 import _capi

    cfgd = CONFIGS[args.config]
    lib = _capi.load()
    hbm_peak, peak_src = peaks()
    subj = subject_data(cfgd["subjects"], cfgd["p"], cfgd["density"], cfgd["bins"],
                        cfgd["strata"], 11)

    cuts = np.arange(cfgd["bins"] + 1, dtype=np.float64) if cfgd["bins"] else None
    splits = ({0: list(cuts[1:-1])} if cfgd["split"] else {}) if cfgd["bins"] else None

    def build():
        """Host subject arrays -> device design. Configs 2-3: only the subjects
        are uploaded; lowering (augment_to_strata + splits) and the sorted
        design are built on the device (scx_build_lowered_design)."""
        if cfgd["bins"]:
            dd_, _ = sx.build_lowered_design(subj, cuts, splits)
        else:
            dd_, _ = sx.build_design(subj)
        return dd_

    def lowered_host():  # the reference arm's input (host lowering, same arrays)
        if cfgd["bins"]:
            data_, _ = sx.lower_time_varying(subj, cuts, splits)
            return data_
        return subj

    t0 = time.perf_counter()
    dd = build()
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    data = lowered_host()
    t_lower = time.perf_counter() - t0
    info = dd.info()
    p = info["p"]
    chunked = C.c_int()
    lib.scx_set_k1_mode(dd.handle, 0, C.byref(chunked))
    gmax = sx.gamma_max(dd)
    if args.config == "c1":
        pen = sx.PenaltySpec.ridge(p, 1.0)  # BASELINE config 1: "L2 prior"
    else:
        pen = sx.PenaltySpec.shared(p, 0.05 * gmax)
    cfg = sx.OptimizerConfig()
    dev = torch.device("cuda", 0)
    l2buf = l2_buffers(dev)
    lib_stream = torch.cuda.ExternalStream(lib.scx_stream(dd.handle), device=dev)
    for _ in range(max(3, args.warmup)):
        flush_l2(l2buf)
        r = sx.ccd_fit(dd, pen, cfg)
    times, evals = [], []
    with ClockSampler(0) as clk:
        for _ in range(args.steps):
            flush_l2(l2buf)
            torch.cuda.synchronize(dev)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(lib_stream)
            r = sx.ccd_fit(dd, pen, cfg)
            e1.record(lib_stream)
            torch.cuda.synchronize(dev)
            times.append(e0.elapsed_time(e1))
            evals.append(r.n_evaluations)
    ms_step = float(np.mean(times))
    value = float(np.mean(evals)) / (ms_step / 1e3)
    # fused scan+reduce alone, L2 flushed before each launch
    cols = np.diff(data.col_ptr)
    sample = [j for j in range(p) if cols[j] > 0][:48]
    st = sx.make_state(dd, r.beta)
    lib.scx_timing_enable(dd.handle, 1)
    lib.scx_timing_reset(dd.handle)
    for j in sample:
        flush_l2(l2buf)
        torch.cuda.synchronize(dev)
        sx.gradient_hessian(dd, st, j)
    tot = C.c_double(); nl = C.c_int64()
    lib.scx_timing_get(dd.handle, 0, C.byref(tot), C.byref(nl))
    k1_ms = tot.value / max(1, nl.value)
    lib.scx_timing_enable(dd.handle, 0)
    alg = info["n_rows"] * (8 + info["code_bytes"]) + 4 * float(np.mean(cols[sample]))
    # the risk-suffix cycle's scan (when the design takes it), L2 flushed
    rs_on = dd.set_fit_path(0)
    fit_stats = dd.fit_path_stats()
    rs_roof = None
    if rs_on:
        lib.scx_timing_enable(dd.handle, 1)
        lib.scx_timing_reset(dd.handle)
        for _ in range(16):
            flush_l2(l2buf)
            torch.cuda.synchronize(dev)
            assert lib.scx_risk_prefix(dd.handle) == 0
        lib.scx_timing_get(dd.handle, 3, C.byref(tot), C.byref(nl))
        rs_ms = tot.value / max(1, nl.value)
        lib.scx_timing_enable(dd.handle, 0)
        rs_bytes = info["n_rows"] * (8 + info["code_bytes"] + 16)
        rs_roof = {"bound": "hbm", "achieved": rs_bytes / (rs_ms * 1e-3) / 1e9, "peak": hbm_peak,
                   "unit": "GB/s", "frac": rs_bytes / (rs_ms * 1e-3) / 1e9 / hbm_peak,
                   "traffic": None, "kernel": "k_rs_cycle risk scan"
                   + ("" if chunked.value else " (chunks of whole tiles, carries across CTAs)"),
                   "avg_launch_ms": rs_ms, "algorithmic_bytes_per_launch": rs_bytes,
                   "algorithmic_bytes_per_row": 8 + info["code_bytes"] + 16, "peak_source": peak_src}
    del st
    dd.close()
    # e2e: host subject arrays -> (device) lowering + sort + upload -> fit -> beta back
    e2e_runs = []
    for _ in range(3):
        t0 = time.perf_counter()
        dd2 = build()
        r2 = sx.ccd_fit(dd2, pen, cfg)
        torch.cuda.synchronize(dev)
        e2e_runs.append(time.perf_counter() - t0)
        dd2.close()
    e2e_s = min(e2e_runs)
    h2d = int(subj.col_ptr[-1]) * 8 + subj.n_rows() * 17 + subj.col_ptr.nbytes
    # reference CPU on the same lowered design (bounded: a few coordinate sweeps)
    cpu = None
    if not args.no_cpu_baseline:
        try:
            from oracle.oracle_py import Dataset, Ref
            ref = Ref()
            threads = os.cpu_count() or 1
            ds = Dataset(data.time, data.event, data.stratum, data.col_ptr, data.row_idx,
                         np.ones(int(data.col_ptr[-1])))
            h, _ = ref.build_design(ds)
            sweep = min(p, 16)
            per = ref.time_iterations(h, 0.05 * gmax, 3, sweep, threads)
            cv = 1.0 / float(np.median(per))
            cpu = {"value": cv, "unit": "evals/s", "cores": threads, "kind": "reference",
                   "sample": f"oracle/_ref on the same lowered design ({info['n_rows']} rows): "
                             f"median of 3 sweeps x {sweep} CCD coordinate iterations",
                   "fit_wall_s_extrapolated": float(np.mean(evals)) / cv}
            ref.free_design(h)
        except Exception as e:
            cpu = {"value": None, "unit": "evals/s", "kind": "reference", "sample": f"unavailable: {e}"}
    line = {
        "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": 1, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic subjects (numpy generator of simulate.cpp's model; seed 11)",
        "config": {"workload": cfgd["workload"], "subjects": cfgd["subjects"],
                   "n_rows": info["n_rows"], "p": p, "strata": info["n_strata"],
                   "code_bytes": info["code_bytes"], "chunked_scan": bool(chunked.value),
                   "gamma": 0.0 if args.config == "c1" else 0.05 * gmax,
                   "l2_prior": 1.0 if args.config == "c1" else 0.0, "fit_cycles": r.cycles_used,
                   "host_lowering_s_reference_input": t_lower,
                   "device_lower_sort_upload_s": t_build,
                   "l2_flush": "256 MiB write then 256 MiB read (another buffer) before every timed fit and K1 launch"},
        "fit_wall_s": ms_step / 1e3,
        "fit_path": "risk-suffix cycle" if fit_stats.get("risk_suffix_launches") else "fused-scan cycle",
        "fit_path_stats": fit_stats,
        "roofline": dict(rs_roof or {}, k1_fused_scan_per_coordinate={
            "kernel": "k1_grad_hess", "avg_launch_ms": k1_ms, "algorithmic_bytes_per_launch": alg,
            "achieved_gbs": alg / (k1_ms * 1e-3) / 1e9, "frac": alg / (k1_ms * 1e-3) / 1e9 / hbm_peak})
        if rs_roof else
        {"bound": "hbm", "achieved": alg / (k1_ms * 1e-3) / 1e9, "peak": hbm_peak,
         "unit": "GB/s", "frac": alg / (k1_ms * 1e-3) / 1e9 / hbm_peak,
         "traffic": None, "kernel": "k1_grad_hess", "avg_launch_ms": k1_ms,
         "algorithmic_bytes_per_launch": alg, "peak_source": peak_src},
        "cpu_baseline": cpu,
        "e2e": {"value": float(r2.n_evaluations) / e2e_s, "unit": "evals/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 8 * p, "seconds_per_step": e2e_s},
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


PARITY_P = 200  # the p=200 design of tests/golden/large_c4_p200.npz (reference converges in 9 cycles)


def cpu_baseline_and_parity(args, sx, gpu_evals):
    from oracle.oracle_py import Ref
    from oracle.oracle_py import to_sorted_design

    threads = os.cpu_count() or 1
    ref = Ref()
    t0 = time.perf_counter()
    ds = ref.simulate(args.n, PARITY_P, args.density, 0.8, args.k, 0.3, 11)
    h, a = ref.build_design(ds)
    del ds
    gmax = ref.gamma_max(h, workers=threads)
    setup = time.perf_counter() - t0
    gamma = 0.05 * gmax
    # (i) per-coordinate CCD iteration, run_benchmark semantics (benchmark.cpp:27-41, 71-98)
    per = ref.time_iterations(h, gamma, 3, args.ref_sweep, threads)
    cv = 1.0 / float(np.median(per))
    per1 = ref.time_iterations(h, gamma, 2, 2, 1)
    cv1 = 1.0 / float(np.median(per1))
    # (ii) a complete reference ccd_fit of the sample (default OptimizerConfig)
    gvec = np.full(PARITY_P, gamma)
    t0 = time.perf_counter()
    rf = ref.ccd_fit(h, gvec, PARITY_P, workers=threads)
    ref_fit_s = time.perf_counter() - t0
    ref.free_design(h)
    nzc = int(np.count_nonzero(np.diff(a["col_ptr"])))
    ref_fit_evals = rf["cycles"] * nzc
    # the library on the same design, same penalty, same path as the timed fits
    dd = sx.upload(to_sorted_design(a))
    del a
    rs_on = dd.set_fit_path(0)
    gmax_gpu = sx.gamma_max(dd)
    rg = sx.ccd_fit(dd, sx.PenaltySpec(gvec), sx.OptimizerConfig())
    stats = dd.fit_path_stats()
    dd.close()
    db = np.abs(rg.beta - rf["beta"])
    trace_rel = float(np.max(np.abs(np.asarray(rg.objective_trace) - rf["trace"]) /
                             np.maximum(1.0, np.abs(rf["trace"])))) \
        if len(rg.objective_trace) == len(rf["trace"]) else None
    parity = {
        "design": (f"reference simulate(): N={args.n}, K={args.k}, density {args.density}, "
                   f"p={PARITY_P}, seed 11; L1 at 0.05*gamma_max, default OptimizerConfig"),
        "reference_cycles": rf["cycles"], "gpu_cycles": rg.cycles_used,
        "reference_converged": rf["converged"], "gpu_converged": rg.converged,
        "max_abs_dbeta": float(db.max()), "beta_atol": 1e-8,
        "supports_equal": bool(np.array_equal(rg.beta != 0, rf["beta"] != 0)),
        "nonzero": int(np.count_nonzero(rf["beta"])),
        "max_rel_dtrace": trace_rel, "gamma_max_rel_diff": abs(gmax_gpu - gmax) / abs(gmax),
        "gpu_fit_path": "risk-suffix cycle" if rs_on else "fused-scan cycle",
        "gpu_fit_path_stats": stats,
        "pass": bool(rg.cycles_used == rf["cycles"] and float(db.max()) <= 1e-8 and
                     np.array_equal(rg.beta != 0, rf["beta"] != 0)),
        "at_scale_test": "tests/test_large_fit.py (p=200 fit to convergence, C2/C3 at 1e6 "
                         "subjects); profiles/r02_parity_c4_full.json (p=1e4, 2 cycles)",
    }
    cpu = {"value": cv, "unit": "evals/s", "cores": threads, "kind": "reference",
           "cpu_model": cpu_model(), "value_1thread": cv1,
           "sample": (f"oracle/_ref (unmodified stratcox, -O3 -fopenmp) on its own simulate() "
                      f"at N={args.n}, K={args.k}, density {args.density}, {PARITY_P} "
                      f"covariates: median of 3 sweeps x {args.ref_sweep} CCD coordinate "
                      f"iterations at gamma=0.05*gamma_max (benchmark.cpp:27-41), {threads} "
                      f"threads; 1 thread: 2 x 2 iterations; setup {setup:.1f}s excluded"),
           "reference_fit": {"p": PARITY_P, "seconds": ref_fit_s, "cycles": rf["cycles"],
                             "evals": ref_fit_evals,
                             "evals_per_s_in_fit": ref_fit_evals / ref_fit_s},
           "fit_wall_s_extrapolated": float(np.mean(gpu_evals)) / cv,
           "extrapolation": ("C4 GPU fit's coordinate evaluations / the reference's "
                             "per-evaluation rate; the same design's reference ccd_fit above "
                             "checks that rate inside a complete fit")}
    return cpu, parity


# ---------------------------------------------------------------- GPU arm
def l2_buffers(dev):
    """Two 256 MiB buffers (> the 126 MB L2): one written, one then read."""
    import torch
    return (torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev),
            torch.ones(64 * 1024 * 1024, dtype=torch.float32, device=dev))


def flush_l2(bufs):
    # write 256 MiB (the L2 holds none of our lines), then read another 256 MiB
    # so the flush's dirty lines are written back before the timed launch
    # rather than during it (the state a launch of the fit meets: no pending
    # write-backs of a foreign buffer)
    bufs[0].add_(1)
    bufs[1].sum()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=10_000_000)
    ap.add_argument("--p", type=int, default=10_000)
    ap.add_argument("--k", type=int, default=1000)
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--gamma-frac", type=float, default=0.05)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--ref-sweep", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-k1", action="store_true",
                    help="only run K1 evaluations (for ncu); prints nothing")
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4"],
                    help="BASELINE config: c4 (default, the headline) or c1-c3 (one line each)")
    args = ap.parse_args()

    for knob in ("SCX_K1_DBG", "SCX_FIT_PER_COORD"):
        if os.environ.get(knob, "0") not in ("", "0"):
            raise SystemExit(f"bench.py: {knob} is a diagnostic knob and must be unset")
    if args.config != "c4":
        run_small_config(args)
        return
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import paper_2310_16238_b200 as sx
    from paper_2310_16238_b200 import _capi, synthetic
    from paper_2310_16238_b200.sharding import plan_row_shards, shard_design

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    lib = _capi.load()
    hbm_peak, peak_src = peaks()

    # ---- data (generated on this GPU; each rank builds the same global design)
    syn = synthetic.generate(args.n, args.p, args.k, args.density, seed=11,
                             device=f"cuda:{local}")
    log(f"[bench] generated N={syn.n} p={syn.p} K={syn.k} nnz={syn.nnz} in {syn.gen_seconds:.1f}s")
    design = syn.sorted_design()
    if world > 1:
        lo, hi = plan_row_shards(design.stratum_offsets, world)[rank]
        design = shard_design(design, lo, hi)
    t0 = time.perf_counter()
    dd = sx.DeviceDesign(design, device=local)
    log(f"[bench] upload {time.perf_counter() - t0:.2f}s info={dd.info()}")
    h = dd.handle
    info = dd.info()
    p = design.n_covariates

    # ---- gamma = frac * gamma_max (global across shards: the ranks' local
    # gradients at beta = 0 summed, before the shards connect)
    if world == 1:
        gmax = sx.gamma_max(dd)
    else:
        st0 = sx.make_state(dd, np.zeros(p))
        g = np.array([sx.gradient_hessian(dd, st0, j).gradient if design.col_ptr[j + 1] >
                      design.col_ptr[j] else 0.0 for j in range(p)])
        gt = torch.tensor(g, device=f"cuda:{local}")
        dist.all_reduce(gt)
        gmax = float(gt.abs().max())
        del st0
        from paper_2310_16238_b200.sharding import connect_ipc
        connect_ipc(dd)  # device-side exchange slots over P2P (NVLink)
    gamma = args.gamma_frac * gmax
    pen = sx.PenaltySpec.shared(p, gamma)
    cfg = sx.OptimizerConfig()
    log(f"[bench] gamma_max={gmax:.6g} gamma={gamma:.6g}")

    if args.profile_k1:
        st = sx.make_state(dd, np.zeros(p))
        for j in range(0, min(p, 64)):
            sx.gradient_hessian(dd, st, j)
        return

    dev = torch.device("cuda", local)
    l2buf = l2_buffers(dev)
    lib_stream = torch.cuda.ExternalStream(lib.scx_stream(h), device=dev)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # ---- warm-up fits
    for _ in range(args.warmup):
        flush_l2(l2buf)
        r = sx.ccd_fit(dd, pen, cfg)
    if args.warmup:
        log(f"[bench] warm-up fit: cycles={r.cycles_used} converged={r.converged} "
            f"nonzero={int(np.count_nonzero(r.beta))} evals={r.n_evaluations}")

    # ---- timed fits (design resident)
    times, evals, cycles = [], [], []
    launches0 = lib.scx_launch_count(h)
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush_l2(l2buf)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(lib_stream)
            r = sx.ccd_fit(dd, pen, cfg)
            e1.record(lib_stream)
            barrier()
            ms = e0.elapsed_time(e1)
            if dist is not None:
                t = torch.tensor([ms], device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ms = float(t)
            times.append(ms)
            evals.append(r.n_evaluations)
            cycles.append(r.cycles_used)
    launches = lib.scx_launch_count(h) - launches0
    path_stats = dd.fit_path_stats()
    log(f"[bench] fit path stats {path_stats}")
    ms_step = float(np.mean(times))
    value = float(np.mean(evals)) / (ms_step / 1e3)
    beta_fit = r.beta.copy()

    # ---- roofline. The fit on the chunked layout runs the risk-suffix cycle:
    # its O(N) work is the fused risk scan (S0 -> w/S0, w/S0^2 -> within-stratum
    # prefixes U, V written per row), once per cycle launch and once per
    # applied step; a coordinate itself is O(nnz_j) gathers. The dominant
    # kernel's roofline is that scan, timed alone (scx_risk_prefix, one launch
    # = every chunk once), L2 flushed before each launch. Algorithmic bytes
    # per row: D 8 + event code + (U, V) 16 written.
    import ctypes as C
    tot = C.c_double()
    nl = C.c_int64()
    lib.scx_timing_enable(h, 1)
    st = sx.make_state(dd, beta_fit)
    rs_on = dd.set_fit_path(0)
    row_bytes_rs = 8 + info["code_bytes"] + 16
    rs = None
    if rs_on:
        lib.scx_timing_reset(h)
        for _ in range(24):
            flush_l2(l2buf)
            torch.cuda.synchronize(dev)
            assert lib.scx_risk_prefix(h) == 0
        lib.scx_timing_get(h, 3, C.byref(tot), C.byref(nl))
        rs_ms = tot.value / max(1, nl.value)
        rs_bytes = design.n_rows * row_bytes_rs
        rs = {"ms": rs_ms, "bytes": rs_bytes, "gbs": rs_bytes / (rs_ms * 1e-3) / 1e9}
        # the same scan as the fit runs it: 16 back-to-back scans in one launch
        # (no launch / pipeline fill per scan), L2 flushed before the launch
        if hasattr(lib, "scx_risk_prefix_n"):
            lib.scx_timing_reset(h)
            for _ in range(4):
                flush_l2(l2buf)
                torch.cuda.synchronize(dev)
                assert lib.scx_risk_prefix_n(h, 16) == 0
            lib.scx_timing_get(h, 3, C.byref(tot), C.byref(nl))
            ms16 = tot.value / max(1, nl.value) / 16
            rs["steady"] = {"scans_per_launch": 16, "ms_per_scan": ms16,
                            "achieved_gbs": rs_bytes / (ms16 * 1e-3) / 1e9}
    # the per-coordinate fused scan+reduce (K1: gradient_hessian, and the fit's
    # exact path), L2 flushed before each launch
    nz_cols = [j for j in range(p) if design.col_ptr[j + 1] > design.col_ptr[j]]
    sample = nz_cols[:: max(1, len(nz_cols) // 48)][:48]
    lib.scx_timing_reset(h)
    for j in sample:
        flush_l2(l2buf)
        torch.cuda.synchronize(dev)
        sx.gradient_hessian(dd, st, j)
    lib.scx_timing_get(h, 0, C.byref(tot), C.byref(nl))
    k1_ms = tot.value / max(1, nl.value)
    nnz_mean = float(np.mean([design.col_ptr[j + 1] - design.col_ptr[j] for j in sample]))
    k1_bytes = design.n_rows * (8 + info["code_bytes"]) + 4 * nnz_mean
    # inside the fit (warm): time of the cycle kernels over one full CCD cycle
    n_coords = len(nz_cols)
    lib.scx_timing_reset(h)
    sx.ccd_fit(dd, pen, sx.OptimizerConfig(max_cycles=1))
    lib.scx_timing_get(h, 3, C.byref(tot), C.byref(nl))
    rs_cycle_ms, rs_launches = tot.value, nl.value
    lib.scx_timing_get(h, 0, C.byref(tot), C.byref(nl))
    fs_cycle_ms, fs_launches = tot.value, nl.value
    lib.scx_timing_enable(h, 0)
    in_fit = {"cycle1_risk_suffix_ms": rs_cycle_ms, "cycle1_risk_suffix_launches": rs_launches,
              "cycle1_fused_scan_ms": fs_cycle_ms, "cycle1_fused_scan_launches": fs_launches,
              "cycle1_ms_per_coordinate": (rs_cycle_ms + fs_cycle_ms) / max(1, n_coords)}

    def ncu_traffic(name, rows):
        f = os.path.join(ROOT, "profiles", name)
        try:
            pj = json.load(open(f))
            return pj.get("dram_bytes_per_launch") if pj.get("n_rows") == rows else None
        except Exception:
            return None

    if rs is not None:
        roof = {"bound": "hbm", "achieved": rs["gbs"], "peak": hbm_peak, "unit": "GB/s",
                "frac": rs["gbs"] / hbm_peak,
                "traffic": ncu_traffic("ncu_rs_scan_summary.json", design.n_rows),
                "kernel": "k_rs_cycle risk scan (forward stratum-segmented S0 -> u = w/S0; "
                          "backward within-stratum suffix sums R of u and Q of u^2/w)",
                "algorithmic_bytes_per_launch": rs["bytes"],
                "algorithmic_bytes_per_row": row_bytes_rs,
                "avg_launch_ms": rs["ms"], "peak_source": peak_src}
        if "steady" in rs:
            t16 = ncu_traffic("r02_ncu_rs_scan_x16.json", design.n_rows)
            roof["steady_state"] = dict(rs["steady"], frac=rs["steady"]["achieved_gbs"] / hbm_peak,
                                        traffic_per_scan=t16 / 16 if t16 else None,
                                        note="headline frac is the single L2-flushed launch; this is "
                                             "the per-scan rate of 16 scans in one launch")
    else:
        roof = {"bound": "hbm", "achieved": k1_bytes / (k1_ms * 1e-3) / 1e9, "peak": hbm_peak,
                "unit": "GB/s", "frac": k1_bytes / (k1_ms * 1e-3) / 1e9 / hbm_peak,
                "traffic": ncu_traffic("ncu_k1_summary.json", design.n_rows),
                "kernel": "k1_grad_hess (fused segmented scan + g'/g'' reduce)",
                "algorithmic_bytes_per_launch": k1_bytes, "avg_launch_ms": k1_ms,
                "peak_source": peak_src}
    roof["in_fit"] = in_fit
    roof["k1_fused_scan_per_coordinate"] = {
        "avg_launch_ms": k1_ms, "algorithmic_bytes_per_launch": k1_bytes,
        "achieved_gbs": k1_bytes / (k1_ms * 1e-3) / 1e9,
        "frac": k1_bytes / (k1_ms * 1e-3) / 1e9 / hbm_peak,
        "traffic": ncu_traffic("ncu_k1_summary.json", design.n_rows)}

    # ---- e2e through the public API from pinned host buffers
    e2e_times = []
    h2d = (design.row_idx.nbytes + design.col_ptr.nbytes + design.stratum_offsets.nbytes +
           design.event.nbytes + design.tie_group_end.nbytes + 8 * p)
    d2h = 8 * p * 2 + 8 * (cfg.max_cycles + 1)
    e2e_evals = []
    del st
    dd.close()
    for _ in range(args.e2e_steps):
        flush_l2(l2buf)
        barrier()
        t0 = time.perf_counter()
        dd2 = sx.DeviceDesign(design, device=local)
        if world > 1:
            from paper_2310_16238_b200.sharding import connect_ipc
            connect_ipc(dd2)
        r2 = sx.ccd_fit(dd2, pen, cfg)
        barrier()
        el = time.perf_counter() - t0
        if dist is not None:
            t = torch.tensor([el], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t)
        e2e_times.append(el)
        e2e_evals.append(r2.n_evaluations)
        dd2.close()
    e2e_value = (float(np.mean(e2e_evals)) / float(np.mean(e2e_times))) if e2e_times else None
    log(f"[bench] e2e seconds per step {e2e_times}")

    # ---- CPU baseline + parity of the benchmarked fit path (rank 0, N=1 only).
    # The reference (oracle/_ref) generates a bounded sample of the same workload
    # with its own simulate() (N, K, density of C4; PARITY_P covariates), times
    # its per-coordinate CCD iteration with all host threads and with one, and
    # runs a complete reference ccd_fit on it; the library then fits the SAME
    # design (uploaded from the reference's SortedDesign) through the same
    # risk-suffix path the timed fits use, and the two fits are compared.
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu, parity = cpu_baseline_and_parity(args, sx, evals)
        except Exception as e:  # reported, never fatal
            cpu = {"value": None, "unit": "evals/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value,
            "unit": "evals/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_step,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (device generator restating simulate.cpp's model; seed 11)",
            "config": {"workload": WORKLOAD if (args.n, args.p, args.k, args.density) ==
                       (10_000_000, 10_000, 1000, 0.01) else
                       (f"C5 shape on one GPU: stratified Cox L1 CCD fit, N={args.n:.0e} rows, "
                        f"p={args.p} sparse indicator covariates ({args.density:g} density), "
                        f"K={args.k} strata, gamma=0.05*gamma_max, beta0=0, tol=1e-6"),
                       "n_rows": args.n, "p": args.p, "strata": args.k,
                       "density": args.density, "nnz": syn.nnz, "gamma": gamma,
                       "gamma_max": gmax, "fit_cycles": cycles, "evals_per_step": evals,
                       "code_bytes": info["code_bytes"],
                       "l2_flush": "256 MiB write then 256 MiB read (another buffer) before every "
                                   "timed step and before every roofline launch",
                       "parallelism": f"rows sharded at stratum boundaries x{world}"
                       if world > 1 else "single GPU"},
            "fit_wall_s": ms_step / 1e3,
            "roofline": roof,
            "fit_path": "risk-suffix cycle" if rs_on else "fused-scan cycle",
            "fit_path_stats": path_stats,
            "cpu_baseline": cpu,
            "parity": parity,
            "e2e": {"value": e2e_value, "unit": "evals/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "seconds_per_step": float(np.mean(e2e_times)) if e2e_times else None},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
