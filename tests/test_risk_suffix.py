"""GPU parity of the risk-suffix CCD cycle (the fit path on the chunked layout).

The risk-suffix cycle computes the same (g', g'') as the per-coordinate fused
scan (likelihood.cpp:129-189), summed per covariate entry instead of per row,
so it is checked the same way: gradient / Hessian against the C oracle at the
reference's 1e-10 scan-vs-naive bar (acceptance.cpp:150-160), fits against the
oracle's ccd_fit at 1e-8 on coefficients with identical cycle counts, and
against the fused-scan cycle (fit path 1) on the same device. Its two hand-offs
to the exact fused scan are exercised: a coordinate whose g'' cancels (a
covariate equal to 1 on whole strata, so S1 = S0 there) and a state whose
max|eta| bound passes 300 mid-cycle.
"""
import numpy as np
import pytest

import paper_2310_16238_b200 as sx
from tests import _golden as G

pytestmark = pytest.mark.gpu

GH_RTOL = 1e-10
LL_RTOL = 1e-10
BETA_ATOL = 1e-8


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if sx.device_count() < 1:
        pytest.fail("no CUDA device visible to libstratcox_b200.so")


def upload(a, values=True):
    return sx.upload(G.sorted_design(a, values=values))


def _design(oracle, ref, n, k, p, density, grid, values, seed):
    if values:  # real-valued X (oracles::random_dataset)
        ds = ref.random_dataset(seed, n, k, p, density, grid)
        return oracle.build_sorted_design(ds)
    ds = ref.simulate(n, p, density, 0.5, k, 0.3, seed)  # binary X (simulate.cpp)
    h0, a = ref.build_design(ds)
    ref.free_design(h0)
    return a


DESIGNS = [
    (1_500_000, 1500, 4, 0.02, 1e9, False),   # indicators, continuous times
    (1_300_000, 2000, 3, 0.15, 1e9, True),    # value columns, dense
    (1_400_000, 1500, 3, 0.01, 40, True),     # heavy ties (w >= 2, wide codes)
    (1_250_000, 20000, 2, 0.05, 1e9, False),  # small strata (135 per chunk)
    # few large strata (the lowered configs' shape): chunks of whole tiles,
    # strata across chunk ends, carries meeting across CTAs
    (1_400_000, 1, 3, 0.02, 1e9, False),      # one stratum
    (1_300_000, 7, 3, 0.15, 1e9, True),       # value columns, dense
    (1_400_000, 20, 3, 0.01, 40, True),       # heavy ties, wide codes
]


@pytest.mark.parametrize("n,k,p,density,grid,values", DESIGNS)
def test_risk_suffix_gradient_matches_oracle(oracle, ref, n, k, p, density, grid, values):
    a = _design(oracle, ref, n, k, p, density, grid, values, 31 + n + k)
    d = oracle.design(a)
    dd = upload(a, values=values)
    assert dd.set_fit_path(0), "design expected to take the risk-suffix cycle"
    rng = np.random.default_rng(k)
    beta = rng.normal(0, 0.3, p)
    st = sx.make_state(dd, beta)
    _, ex = oracle.make_state(d, beta)
    for j in range(p):
        g, h = oracle.gradient_hessian(d, ex, j)
        r1 = sx.risk_suffix_gradient_hessian(dd, st, j)
        r2 = sx.risk_suffix_gradient_hessian(dd, st, j)
        assert (r1.gradient, r1.hessian) == (r2.gradient, r2.hessian), j  # reproducible
        assert G.close_rel(r1.gradient, g, GH_RTOL), (j, r1.gradient, g)
        assert G.close_rel(r1.hessian, h, GH_RTOL), (j, r1.hessian, h)


@pytest.mark.parametrize("n,k,p,density,grid,values,gfrac", [
    (1_300_000, 1300, 4, 0.05, 1e9, False, 0.1),
    (1_300_000, 2000, 3, 0.15, 1e9, True, 0.05),
    (1_400_000, 1500, 3, 0.01, 40, True, 0.0),      # unpenalised: Newton on every coordinate
    (1_250_000, 20000, 3, 0.05, 1e9, False, 0.02),
    (1_300_000, 1, 4, 0.05, 1e9, False, 0.1),       # unaligned chunks: one stratum
    (1_300_000, 12, 3, 0.15, 1e9, True, 0.05),      # ... value columns, 12 strata
    (1_400_000, 20, 3, 0.02, 40, False, 0.05),      # ... heavy ties
])
def test_risk_suffix_fit_matches_oracle(oracle, ref, n, k, p, density, grid, values, gfrac):
    a = _design(oracle, ref, n, k, p, density, grid, values, 5 + k)
    d = oracle.design(a)
    dd = upload(a, values=values)
    assert dd.set_fit_path(0)
    gamma = np.full(p, gfrac * sx.gamma_max(dd)) if gfrac > 0 else np.zeros(p)
    cfg = dict(max_cycles=40, tol=1e-8)
    want = oracle.ccd_fit(d, gamma, **cfg)
    r = sx.ccd_fit(dd, sx.PenaltySpec(gamma), sx.OptimizerConfig(max_cycles=40, tolerance=1e-8))
    assert r.cycles_used == want["cycles"]
    assert np.max(np.abs(r.beta - want["beta"])) <= BETA_ATOL
    assert np.allclose(r.objective_trace, want["trace"], rtol=LL_RTOL, atol=0)
    # the fused-scan cycle on the same device lands on the same fit
    assert not dd.set_fit_path(1)
    r1 = sx.ccd_fit(dd, sx.PenaltySpec(gamma), sx.OptimizerConfig(max_cycles=40, tolerance=1e-8))
    assert r1.cycles_used == r.cycles_used
    assert np.max(np.abs(r1.beta - r.beta)) <= BETA_ATOL
    dd.set_fit_path(0)


def _with_extra_columns(oracle, ds, cols):
    """ds plus columns given as (rows, values) in the dataset's row space."""
    from oracle.oracle_py import Dataset
    col_ptr = list(ds.col_ptr)
    rows = [ds.row_idx]
    vals = [ds.values]
    for r, v in cols:
        rows.append(np.asarray(r, np.int64))
        vals.append(np.asarray(v, float))
        col_ptr.append(col_ptr[-1] + len(r))
    return Dataset(ds.time, ds.event, ds.stratum, np.asarray(col_ptr, np.int64),
                   np.concatenate(rows), np.concatenate(vals))


def test_risk_suffix_cancelling_hessian_goes_exact(oracle, ref):
    """A covariate equal to 1 on every row of some strata: there S1 = S0, the
    reference's g'' terms are exactly 0 and the per-entry sums cancel. The
    coordinate is handed to the exact fused scan (kRsExact) and the fit
    matches the oracle's."""
    n, k, p = 1_300_000, 1300, 3
    ds = ref.random_dataset(77, n, k, p, 0.05, 1e9)
    strat = np.asarray(ds.stratum)
    full = np.flatnonzero(np.isin(strat, np.arange(0, k, 2)))  # every even stratum, all rows
    ds2 = _with_extra_columns(oracle, ds, [(full, np.ones(len(full)))])
    a = oracle.build_sorted_design(ds2)
    d = oracle.design(a)
    dd = upload(a)
    assert dd.set_fit_path(0)
    pp = a["p"]
    gamma = np.zeros(pp)  # unpenalised: the cancelling coordinate reaches the Newton step
    want = oracle.ccd_fit(d, gamma, max_cycles=25, tol=1e-8)
    r = sx.ccd_fit(dd, sx.PenaltySpec(gamma), sx.OptimizerConfig(max_cycles=25, tolerance=1e-8))
    assert r.cycles_used == want["cycles"]
    assert np.max(np.abs(r.beta - want["beta"])) <= BETA_ATOL
    assert np.allclose(r.objective_trace, want["trace"], rtol=LL_RTOL, atol=0)


def test_risk_suffix_bound_hands_over(oracle, ref):
    """A coefficient held near eta = 299.95 on a few rows: the first applied step
    lifts the max|eta| bound past 300 and the rest of the cycle runs on the
    fused-scan cycle (kRsBound); later cycles refresh the bound. Fit vs oracle."""
    n, k, p = 1_300_000, 1300, 3
    ds = ref.random_dataset(91, n, k, p, 0.05, 1e9)
    rng = np.random.default_rng(3)
    few = np.sort(rng.choice(n, 40, replace=False)).astype(np.int64)
    ds2 = _with_extra_columns(oracle, ds, [(few, np.ones(len(few)))])
    a = oracle.build_sorted_design(ds2)
    d = oracle.design(a)
    dd = upload(a)
    assert dd.set_fit_path(0)
    pp = a["p"]
    b0 = np.zeros(pp)
    b0[pp - 1] = 299.95
    gamma = np.zeros(pp)
    gamma[: pp - 1] = 0.01 * sx.gamma_max(dd)
    want = oracle.ccd_fit(d, gamma, max_cycles=6, tol=1e-9, initial_beta=b0)
    r = sx.ccd_fit(dd, sx.PenaltySpec(gamma), sx.OptimizerConfig(max_cycles=6, tolerance=1e-9),
                   initial_beta=b0)
    assert r.cycles_used == want["cycles"]
    assert np.max(np.abs(r.beta - want["beta"])) <= BETA_ATOL
    assert np.allclose(r.objective_trace, want["trace"], rtol=LL_RTOL, atol=0)


def test_risk_suffix_mixed_penalties_match_oracle(oracle, ref):
    """Per-coordinate penalties mixing unpenalised (gamma = 0), weak and strong L1
    weights, so gradient rounds stop at coordinates that cannot be skipped
    (beta != 0 or gamma = 0) at every position of a round, and rounds of skipped
    coordinates alternate with full evaluations. Fit vs oracle."""
    n, k, p = 1_300_000, 1300, 16
    a = _design(oracle, ref, n, k, p, 0.03, 1e9, False, 4242)
    d = oracle.design(a)
    dd = upload(a, values=False)
    assert dd.set_fit_path(0)
    gmax = sx.gamma_max(dd)
    frac = np.array([0.0, 0.3, 0.02, 0.5, 0.0, 0.01, 0.9, 0.05,
                     0.2, 0.0, 0.6, 0.03, 0.4, 0.08, 0.0, 0.7])
    gamma = frac * gmax
    want = oracle.ccd_fit(d, gamma, max_cycles=40, tol=1e-8)
    r = sx.ccd_fit(dd, sx.PenaltySpec(gamma), sx.OptimizerConfig(max_cycles=40, tolerance=1e-8))
    assert r.cycles_used == want["cycles"]
    assert np.max(np.abs(r.beta - want["beta"])) <= BETA_ATOL
    assert np.allclose(r.objective_trace, want["trace"], rtol=LL_RTOL, atol=0)
    nz = np.count_nonzero(r.beta)
    assert 0 < nz < p, nz  # both kinds of coordinate present at the optimum


def test_repeated_scans_in_one_launch_are_identical():
    """scx_risk_prefix_n (the throughput probe: back-to-back scans inside one
    launch, as the fit runs them) leaves the same R, Q and tile carries as one
    scan: the stage / carry-slot sequences continue correctly across scans."""
    import ctypes as C

    from paper_2310_16238_b200 import _capi, synthetic

    lib = _capi.load()
    n = 3_000_000
    syn = synthetic.generate(n, 16, 1500, 0.02, seed=7, device="cuda")
    dd = sx.upload(syn.sorted_design())
    assert dd.set_fit_path(0)
    sx.make_state(dd, np.random.default_rng(3).normal(0, 0.1, 16))
    nt = (n + 2047) // 2048 + 1
    got = []
    for reps in (1, 4):
        arrs = [np.zeros(n), np.zeros(n), np.zeros(nt), np.zeros(nt)]
        assert lib.scx_risk_prefix_n(dd.handle, reps) == 0
        assert lib.scx_debug_risk_arrays(dd.handle, *(_capi.ptr(a, C.c_double) for a in arrs), None) == 0
        got.append(arrs)
    for a, b in zip(got[0], got[1]):
        assert np.array_equal(a, b)
    assert lib.scx_risk_prefix_n(dd.handle, 0) != 0  # reps >= 1
    dd.close()


@pytest.mark.parametrize("n,k,p,density,grid,values", DESIGNS)
def test_risk_suffix_gamma_max_matches_oracle(oracle, ref, n, k, p, density, grid, values):
    """gamma_max (resample.hpp:38-39) on the chunked layout runs as one
    risk-suffix launch (every column's g' at beta = 0 in gradient rounds): the
    oracle's value and the per-coordinate fused-scan path's within 1e-10, and a
    penalty template with unpenalised columns excludes them the same way."""
    a = _design(oracle, ref, n, k, p, density, grid, values, 99)
    d = oracle.design(a)
    dd = upload(a, values=values)
    assert dd.set_fit_path(0)
    want = oracle.gamma_max(d)
    got = sx.gamma_max(dd)
    assert G.close_rel(got, want, GH_RTOL), (got, want)
    tmpl = np.ones(p)
    tmpl[0] = 0.0  # column 0 unpenalised: left out of the max
    g_t = sx.gamma_max(dd, sx.PenaltySpec(tmpl))
    dd.set_fit_path(1)
    assert G.close_rel(sx.gamma_max(dd), want, GH_RTOL)
    assert G.close_rel(g_t, sx.gamma_max(dd, sx.PenaltySpec(tmpl)), GH_RTOL)
