"""GPU parity: the sm_100a library (through the C-ABI) against the reference.

Bars (BASELINE.json north_star): bit-exact indexing; fp64 log-likelihood
within 1e-10 relative; coefficients within 1e-8 absolute. Gradient/Hessian use
the reference's own 1e-10 scan-vs-naive bar (acceptance.cpp:150-160).
Checkers: golden fixtures from the compiled reference (tests/golden/) and the
C oracle (oracle/, itself pinned bit-exactly to the reference).
"""
import math

import numpy as np
import pytest

import paper_2310_16238_b200 as sx
from tests import _golden as G

pytestmark = pytest.mark.gpu

LL_RTOL = 1e-10   # log-likelihood, relative (north_star)
GH_RTOL = 1e-10   # gradient / Hessian, oracles::close_rel (acceptance.cpp:150-160)
BETA_ATOL = 1e-8  # coefficients, absolute (north_star)


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if sx.device_count() < 1:
        pytest.fail("no CUDA device visible to libstratcox_b200.so")


def upload(a, values=True):
    return sx.upload(G.sorted_design(a, values=values))


# ---------------------------------------------------------------- scan primitive
def test_segmented_scan_worked_example():
    v = np.array([3, 1, 7, 0, 4, 1, 6, 3], float)
    f = np.array([1, 0, 1, 0, 0, 1, 0, 0], np.uint8)
    assert sx.segmented_inclusive_scan(v, f).tolist() == [3, 4, 7, 7, 11, 1, 7, 10]
    assert sx.segmented_inclusive_scan([5, 2, 9], [1, 1, 1]).tolist() == [5, 2, 9]
    assert sx.segmented_inclusive_scan([2, 2, 2, 2], [1, 0, 0, 0]).tolist() == [2, 4, 6, 8]


def test_segmented_scan_vs_reference_fixtures():
    z = G.load("scan_instances")
    for c in range(int(z["count"])):
        v, f, want = z[f"s{c}_v"], z[f"s{c}_f"], z[f"s{c}_out"]
        got = sx.segmented_inclusive_scan(v, f)
        if np.all(v == np.round(v)):
            assert np.array_equal(got, want), c  # integer data: exact
        else:
            scale = np.maximum(1.0, np.maximum(np.abs(got), np.abs(want)))
            assert np.max(np.abs(got - want) / scale) <= 1e-12, c


def test_segmented_scan_validation():
    with pytest.raises(sx.ValidationError, match="empty scan input"):
        sx.segmented_inclusive_scan([], [])
    with pytest.raises(sx.ValidationError, match="first element must head a segment"):
        sx.segmented_inclusive_scan([1.0, 2.0, 3.0], [0, 0, 1])
    with pytest.raises(sx.ValidationError, match="non-finite input at index 1"):
        sx.segmented_inclusive_scan([1.0, np.nan, 2.0], [1, 0, 0])


def test_segmented_scan_deterministic_large():
    rng = np.random.default_rng(77)
    v = rng.uniform(-1, 1, 3_000_001)
    f = np.zeros(v.shape[0], np.uint8)
    f[0] = 1
    f[rng.integers(0, v.shape[0], 64)] = 1
    a = sx.segmented_inclusive_scan(v, f)
    b = sx.segmented_inclusive_scan(v, f)
    assert np.array_equal(a, b)


# ---------------------------------------------------------------- likelihood vs fixtures
def test_gradient_hessian_loglik_vs_reference_fixtures():
    z = G.load("random_instances")
    worst = 0.0
    for i in range(int(z["count"])):
        pre = f"r{i}_"
        a = G.design_arrays(z, pre)
        dd = upload(a)
        st = sx.make_state(dd, z[pre + "beta"])
        assert np.array_equal(st.xbeta, z[pre + "xbeta"]), i  # ascending-column sums, exact
        ex = st.exp_xbeta
        assert np.max(np.abs(ex - z[pre + "exp_xbeta"]) / z[pre + "exp_xbeta"]) <= 4e-16, i
        for j in range(a["p"]):
            gh = sx.gradient_hessian(dd, st, j)
            assert G.close_rel(gh.gradient, z[pre + "grad"][j], GH_RTOL), (i, j)
            assert G.close_rel(gh.hessian, z[pre + "hess"][j], GH_RTOL), (i, j)
            assert gh.hessian >= -1e-12
            worst = max(worst, abs(gh.gradient - z[pre + "grad"][j]) /
                        max(1, abs(gh.gradient)), abs(gh.hessian - z[pre + "hess"][j]) /
                        max(1, abs(gh.hessian)))
            nv = sx.naive_gradient_hessian(dd, st, j)
            assert G.close_rel(nv.gradient, z[pre + "naive_grad"][j], GH_RTOL), (i, j)
            assert G.close_rel(nv.hessian, z[pre + "naive_hess"][j], GH_RTOL), (i, j)
        ll = sx.log_partial_likelihood(dd, st)
        assert G.close_rel(ll, float(z[pre + "ll"]), LL_RTOL), i
        assert G.close_rel(sx.naive_log_partial_likelihood(dd, st), float(z[pre + "naive_ll"]),
                           LL_RTOL), i
        dd.close()
    assert worst < 1e-12


def test_known_answers_on_device():
    z = G.load("known_answers")
    a = G.design_arrays(z, "handworked_")
    dd = upload(a)
    st = sx.make_state(dd, [0.0])
    gh = sx.gradient_hessian(dd, st, 0)
    assert math.isclose(gh.gradient, -2.0 / 3.0, rel_tol=1e-12)
    assert math.isclose(gh.hessian, 2.0 / 9.0, rel_tol=1e-12)
    assert math.isclose(sx.log_partial_likelihood(dd, st), -math.log(6.0), rel_tol=1e-12)
    a = G.design_arrays(z, "zerocol_")
    dd = upload(a)
    st = sx.make_state(dd, [0.4])
    gh = sx.gradient_hessian(dd, st, 0)
    assert gh.gradient == 0.0 and gh.hessian == 0.0


# ---------------------------------------------------------------- state updates
def test_update_xbeta_matches_oracle(oracle):
    z = G.load("random_instances")
    for i in range(0, int(z["count"]), 7):
        pre = f"r{i}_"
        a = G.design_arrays(z, pre)
        d = oracle.design(a)
        dd = upload(a)
        beta = z[pre + "beta"].copy()
        st = sx.make_state(dd, beta)
        xb, ex = oracle.make_state(d, beta)
        u = 0
        for step, j in enumerate([0, a["p"] - 1, 0]):
            delta = 0.375 - 0.25 * step
            sx.update_xbeta(dd, st, j, delta)
            u = oracle.update_xbeta(d, beta, xb, ex, u, j, delta)
        assert np.array_equal(st.beta, beta)
        assert np.array_equal(st.xbeta, xb)
        assert np.max(np.abs(st.exp_xbeta - ex) / ex) <= 4e-16
        assert st.updates_since_refresh == u


def test_update_xbeta_overflow_leaves_state(oracle):
    z = G.load("random_instances")
    a = G.design_arrays(z, "r3_")
    dd = upload(a)
    p = a["p"]
    beta = np.zeros(p)
    st = sx.make_state(dd, beta)
    x0 = st.xbeta.copy()
    with pytest.raises(sx.NumericError, match="^step overflow$"):
        sx.update_xbeta(dd, st, 0, 800.0)
    assert np.array_equal(st.xbeta, x0) and st.beta[0] == 0.0
    with pytest.raises(sx.ValidationError, match="covariate index out of range"):
        sx.update_xbeta(dd, st, p, 0.1)


def test_make_state_overflow_message():
    from paper_2310_16238_b200.stratcox import SortedDesign
    d = SortedDesign(stratum_offsets=np.array([0, 2]), event=np.array([1, 1], np.uint8),
                     tie_group_end=np.array([0, 1]), col_ptr=np.array([0, 1]),
                     row_idx=np.array([0]), values=np.array([2.0]))
    dd = sx.upload(d)
    with pytest.raises(sx.NumericError, match="linear predictor overflow at row 0"):
        sx.make_state(dd, [400.0])


def test_refresh_after_256_updates(oracle):
    z = G.load("random_instances")
    a = G.design_arrays(z, "r12_")
    d = oracle.design(a)
    dd = upload(a)
    p = a["p"]
    beta = np.zeros(p)
    st = sx.make_state(dd, beta)
    xb, ex = oracle.make_state(d, beta)
    rng = np.random.default_rng(35)
    u = 0
    for it in range(600):
        j = it % p
        delta = float(rng.uniform(-0.01, 0.01))
        sx.update_xbeta(dd, st, j, delta)
        u = oracle.update_xbeta(d, beta, xb, ex, u, j, delta)
    assert st.updates_since_refresh == u < 256
    assert np.array_equal(st.beta, beta)
    assert np.array_equal(st.xbeta, xb)  # refresh order and increments are exact restatements


# ---------------------------------------------------------------- fits
def test_ccd_fit_vs_reference_fixtures():
    z = G.load("fits")
    for name in z["names"]:
        pre = str(name) + "_"
        a = G.design_arrays(z, pre)
        dd = upload(a, values=False)
        cfg = sx.OptimizerConfig(max_cycles=int(z[pre + "max_cycles"]), tolerance=float(z[pre + "tol"]))
        r = sx.ccd_fit(dd, sx.PenaltySpec(z[pre + "gamma"]), cfg)
        assert r.converged == bool(z[pre + "converged"]), name
        assert r.cycles_used == int(z[pre + "cycles"]), name
        assert np.max(np.abs(r.beta - z[pre + "beta"])) <= BETA_ATOL, name
        tr = np.array(r.objective_trace)
        want = z[pre + "trace"]
        assert tr.shape == want.shape, name
        assert np.max(np.abs(tr - want) / np.maximum(1, np.abs(want))) <= LL_RTOL, name
        assert np.array_equal(r.beta == 0.0, z[pre + "beta"] == 0.0), name  # same support
        dd.close()


def test_ccd_fit_bitwise_deterministic():
    z = G.load("fits")
    pre = "c7_g1_"
    a = G.design_arrays(z, pre)
    dd = upload(a, values=False)
    pen = sx.PenaltySpec(z[pre + "gamma"])
    r1 = sx.ccd_fit(dd, pen)
    r2 = sx.ccd_fit(dd, pen)
    assert r1.beta.tobytes() == r2.beta.tobytes()
    assert r1.objective_trace == r2.objective_trace
    for j in range(a["p"]):
        st = sx.make_state(dd, r1.beta)
        g1 = sx.gradient_hessian(dd, st, j)
        g2 = sx.gradient_hessian(dd, st, j)
        assert (g1.gradient, g1.hessian) == (g2.gradient, g2.hessian)


def test_ccd_fit_validation_messages():
    z = G.load("fits")
    a = G.design_arrays(z, "c7_g1_")
    dd = upload(a, values=False)
    p = a["p"]
    with pytest.raises(sx.ValidationError, match="penalty weights must be finite and non-negative"):
        sx.ccd_fit(dd, sx.PenaltySpec(np.full(p, -1.0)))
    with pytest.raises(sx.ValidationError, match="max_cycles must be >= 1"):
        sx.ccd_fit(dd, sx.PenaltySpec.none(p), sx.OptimizerConfig(max_cycles=0))
    with pytest.raises(sx.ValidationError, match="tolerance must be positive"):
        sx.ccd_fit(dd, sx.PenaltySpec.none(p), sx.OptimizerConfig(tolerance=0.0))
    r = sx.ccd_fit(dd, sx.PenaltySpec.shared(p, 1e6))  # test_optimizer.cpp:80-87
    assert r.converged and np.all(r.beta == 0.0)


def test_gamma_max_vs_reference():
    z = G.load("fits")
    pre = "cfg1_l1_"
    a = G.design_arrays(z, pre)
    dd = upload(a, values=False)
    gm = sx.gamma_max(dd)
    assert G.close_rel(gm, float(z[pre + "gamma_max"]), 1e-10)


# ---------------------------------------------------------------- edge cases vs oracle
def _compare_all(oracle, a, beta, values=True, tol=GH_RTOL):
    d = oracle.design(a)
    dd = upload(a, values=values)
    st = sx.make_state(dd, beta)
    xb, ex = oracle.make_state(d, beta)
    assert np.array_equal(st.xbeta, xb)
    for j in range(a["p"]):
        g, h = oracle.gradient_hessian(d, ex, j)
        gh = sx.gradient_hessian(dd, st, j)
        assert G.close_rel(gh.gradient, g, tol) and G.close_rel(gh.hessian, h, tol), j
    assert G.close_rel(sx.log_partial_likelihood(dd, st), oracle.log_partial_likelihood(d, xb, ex),
                       LL_RTOL)
    return dd


@pytest.mark.parametrize("n,strata,p,density,grid", [
    (1, 1, 1, 1.0, 8),          # single row
    (15, 1, 2, 0.5, 8),         # fewer rows than one thread's span
    (4095, 1, 2, 0.3, 8),       # just under one tile
    (4097, 3, 2, 0.3, 8),       # one row into the second tile
    (20000, 1, 3, 0.2, 8),      # K=1, heavy ties on an 8-point grid
    (20000, 20000, 2, 0.3, 8),  # every row its own stratum: all heads
    (50000, 997, 3, 0.05, 1e6), # many strata, nearly no ties
    (70000, 2, 2, 0.01, 2),     # two time values: tie groups of ~17k rows (u16 codes)
    (3_000_000, 1, 2, 0.01, 1e9),  # one stratum over 733 tiles: deepest look-backs
])
def test_edge_shapes_vs_oracle(oracle, ref, n, strata, p, density, grid):
    ds = ref.random_dataset(1000 + n + strata, n, strata, p, density, grid)
    a = oracle.build_sorted_design(ds)
    rng = np.random.default_rng(n)
    dd = _compare_all(oracle, a, rng.normal(0, 0.4, p))
    if grid == 2:
        assert dd.info()["code_bytes"] >= 2


def test_value_and_indicator_columns_mixed(oracle, ref):
    ds = ref.random_dataset(4242, 30000, 13, 6, 0.3, 50)
    a = oracle.build_sorted_design(ds)
    _compare_all(oracle, a, np.linspace(-0.5, 0.5, 6))


# ---------------------------------------------------------------- error paths
def test_nonfinite_state_reports_first_row():
    z = G.load("random_instances")
    a = G.design_arrays(z, "r5_")
    dd = upload(a)
    n, p = a["n"], a["p"]
    xb = np.zeros(n)
    ex = np.ones(n)
    ex[7] = np.inf
    ex[9] = np.nan
    st = sx.state_from_arrays(dd, np.zeros(p), xb, ex)
    with pytest.raises(sx.ValidationError, match="non-finite input at index 7"):
        sx.gradient_hessian(dd, st, 0)
    with pytest.raises(sx.ValidationError, match="non-finite input at index 7"):
        sx.log_partial_likelihood(dd, st)


def test_bad_denominator_is_internal_error(ref, oracle):
    ds = ref.random_dataset(99, 64, 1, 1, 0.5, 8)
    a = oracle.build_sorted_design(ds)
    d = oracle.design(a)
    dd = upload(a)
    n = a["n"]
    ex = np.ones(n)
    # zero D over the first tie group(s) so their risk-set sum is exactly 0
    first_end = int(a["tie_end"][0])
    while not a["event"][:first_end + 1].any():
        first_end = int(a["tie_end"][first_end + 1])
    ex[:first_end + 1] = 0.0
    from oracle.oracle_py import OracleError
    with pytest.raises(OracleError) as e:
        oracle.gradient_hessian(d, ex, 0)
    st = sx.state_from_arrays(dd, np.zeros(1), np.zeros(n), ex)
    with pytest.raises(sx.InternalError) as e2:
        sx.gradient_hessian(dd, st, 0)
    assert str(e2.value) == str(e.value)


# ---------------------------------------------------------------- large-N properties
@pytest.mark.parametrize("n,k,p", [(1_000_000, 1000, 8), (10_000_000, 1000, 3)])
def test_large_n_gradient_vs_oracle(oracle, ref, n, k, p):
    """BASELINE C4 row count with the oracle as checker on sampled coordinates."""
    ds = ref.simulate(n, p, 0.01, 0.5, k, 0.3, 11)
    h, a = ref.build_design(ds)
    ref.free_design(h)
    d = oracle.design(a)
    dd = upload(a, values=False)
    beta = np.linspace(-0.3, 0.3, p)
    st = sx.make_state(dd, beta)
    xb, ex = oracle.make_state(d, beta)
    assert np.array_equal(st.xbeta, xb)
    for j in range(p):
        g, hh = oracle.gradient_hessian(d, ex, j)
        gh = sx.gradient_hessian(dd, st, j)
        assert G.close_rel(gh.gradient, g, GH_RTOL) and G.close_rel(gh.hessian, hh, GH_RTOL), j
    ll = oracle.log_partial_likelihood(d, xb, ex)
    assert G.close_rel(sx.log_partial_likelihood(dd, st), ll, LL_RTOL)
    # size-independent property: stratum additivity of the log-likelihood
    g1 = sx.gradient_hessian(dd, st, 0)
    g2 = sx.gradient_hessian(dd, st, 0)
    assert (g1.gradient, g1.hessian) == (g2.gradient, g2.hessian)


# ---------------------------------------------------------------- fused-scan decompositions
def _k1_mode(dd, mode):
    """0 auto / 1 cross-CTA look-back / 2 stratum-aligned chunks; returns 1 if chunked."""
    import ctypes as C
    from paper_2310_16238_b200 import _capi
    ch = C.c_int()
    assert _capi.load().scx_set_k1_mode(dd.handle, mode, C.byref(ch)) == 0
    return ch.value


@pytest.mark.parametrize("n,k,p,density,grid,values", [
    (1_500_000, 1500, 4, 0.02, 1e9, False),  # indicators, continuous times: fast path
    (1_300_000, 2000, 3, 0.15, 1e9, True),   # value columns, > 64 entries per quarter
    (1_400_000, 1500, 3, 0.01, 40, True),    # heavy ties (general path, wide codes)
    (1_250_000, 20000, 2, 0.05, 1e9, False),  # small strata: heads in most threads' rows
])
def test_chunked_and_lookback_match_oracle(oracle, ref, n, k, p, density, grid, values):
    """The stratum-aligned chunk kernel and the look-back kernel both agree with
    the oracle (1e-10) and are each bitwise reproducible."""
    if values:  # real-valued X (oracles::random_dataset)
        ds = ref.random_dataset(31 + n + k, n, k, p, density, grid)
        a = oracle.build_sorted_design(ds)
    else:       # binary X (simulate.cpp): indicator columns
        ds = ref.simulate(n, p, density, 0.5, k, 0.3, 31 + k)
        h0, a = ref.build_design(ds)
        ref.free_design(h0)
    d = oracle.design(a)
    dd = upload(a, values=values)
    assert _k1_mode(dd, 0) == 1, "design expected to take the chunked kernel"
    rng = np.random.default_rng(k)
    beta = rng.normal(0, 0.3, p)
    st = sx.make_state(dd, beta)
    xb, ex = oracle.make_state(d, beta)
    for j in range(p):
        g, h = oracle.gradient_hessian(d, ex, j)
        for mode in (2, 1):
            _k1_mode(dd, mode)
            r1 = sx.gradient_hessian(dd, st, j)
            r2 = sx.gradient_hessian(dd, st, j)
            assert (r1.gradient, r1.hessian) == (r2.gradient, r2.hessian), (j, mode)
            assert G.close_rel(r1.gradient, g, GH_RTOL), (j, mode, r1.gradient, g)
            assert G.close_rel(r1.hessian, h, GH_RTOL), (j, mode, r1.hessian, h)
    _k1_mode(dd, 0)


def test_chunked_fit_matches_oracle(oracle, ref):
    """A full L1 CCD fit through the chunked kernel against the oracle's fit."""
    n, k, p = 1_300_000, 1300, 4
    ds = ref.simulate(n, p, 0.05, 0.5, k, 0.3, 5)
    h, a = ref.build_design(ds)
    ref.free_design(h)
    d = oracle.design(a)
    dd = upload(a, values=False)
    assert _k1_mode(dd, 0) == 1
    gmax = sx.gamma_max(dd)
    gamma = np.full(p, 0.1 * gmax)
    want = oracle.ccd_fit(d, gamma, max_cycles=50, tol=1e-8)
    r = sx.ccd_fit(dd, sx.PenaltySpec(gamma), sx.OptimizerConfig(max_cycles=50, tolerance=1e-8))
    assert r.cycles_used == want["cycles"]
    assert np.max(np.abs(r.beta - want["beta"])) <= BETA_ATOL
    assert np.allclose(r.objective_trace, want["trace"], rtol=LL_RTOL, atol=0)


@pytest.mark.parametrize("b0", [699.5, 699.95])
def test_fit_step_halving_vs_oracle(oracle, ref, b0):
    """Steps that would push eta past +-700 inside the device cycle: a column held
    at beta = b0 on the 30 latest rows (in every risk set) overlaps the other
    columns, so their steps need the exact halving level and some are skipped
    after 10 halvings with a warning (optimizer.cpp:110-123); against the oracle."""
    from oracle.oracle_py import Dataset
    ds = ref.random_dataset(7, 3000, 2, 3, 0.4, 50)
    rows_c = np.sort(np.argsort(-ds.time)[:30]).astype(np.int64)
    ds2 = Dataset(ds.time, ds.event.copy(), ds.stratum,
                  np.concatenate([ds.col_ptr, [ds.col_ptr[-1] + 30]]),
                  np.concatenate([ds.row_idx, rows_c]), np.concatenate([ds.values * 30, np.ones(30)]))
    ds2.event[rows_c] = 0
    a = oracle.build_sorted_design(ds2)
    d = oracle.design(a)
    dd = upload(a)
    p = a["p"]
    b_init = np.array([0.0, 0.0, 0.0, b0])
    want = oracle.ccd_fit(d, np.zeros(p), max_cycles=6, tol=1e-9, initial_trust=1.0,
                          initial_beta=b_init)
    assert want["n_warnings"] > 0  # the design does exercise the 10-halving skip
    r = sx.ccd_fit(dd, sx.PenaltySpec(np.zeros(p)),
                   sx.OptimizerConfig(max_cycles=6, tolerance=1e-9, initial_trust=1.0),
                   initial_beta=b_init)
    assert r.cycles_used == want["cycles"]
    assert len(r.warnings) == want["n_warnings"]
    assert np.max(np.abs(r.beta - want["beta"])) <= BETA_ATOL
    assert np.max(np.abs(r.trust - want["trust"]) / np.maximum(1, np.abs(want["trust"]))) <= 1e-12
    assert np.allclose(r.objective_trace, want["trace"], rtol=LL_RTOL, atol=0)
