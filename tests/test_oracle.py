"""CPU: pin the C oracle (oracle/stratcox_oracle.c) against the reference.

* bit-exact against the golden fixtures produced by the compiled reference
  (tests/golden/make_golden.py);
* the known-answer cases of the reference unit tests, restated;
* live bit-exact cross-checks against oracle/_ref (when built here).
"""
import math

import numpy as np
import pytest

from tests import _golden as G


# ---------------------------------------------------------------- golden, bit-exact
def test_sorted_design_matches_reference_fixtures(oracle):
    z = G.load("random_instances")
    for i in range(int(z["count"])):
        pre = f"r{i}_"
        ds = G.dataset(z, pre)
        a = oracle.build_sorted_design(ds)
        want = G.design_arrays(z, pre)
        for key in ("perm", "head", "tie_end", "offsets", "time", "event", "col_ptr", "row_idx",
                    "values"):
            assert np.array_equal(a[key], want[key]), (i, key)


def test_likelihood_matches_reference_fixtures_bitwise(oracle):
    z = G.load("random_instances")
    for i in range(int(z["count"])):
        pre = f"r{i}_"
        d = oracle.design(G.design_arrays(z, pre))
        beta = z[pre + "beta"]
        xb, ex = oracle.make_state(d, beta)
        assert np.array_equal(xb, z[pre + "xbeta"]) and np.array_equal(ex, z[pre + "exp_xbeta"])
        for j in range(d.p):
            g, h = oracle.gradient_hessian(d, ex, j)
            assert g == z[pre + "grad"][j] and h == z[pre + "hess"][j], (i, j)
            ng, nh = oracle.naive_gradient_hessian(d, ex, j)
            assert ng == z[pre + "naive_grad"][j] and nh == z[pre + "naive_hess"][j], (i, j)
        assert oracle.log_partial_likelihood(d, xb, ex) == float(z[pre + "ll"])
        assert oracle.naive_log_partial_likelihood(d, xb, ex) == float(z[pre + "naive_ll"])


def test_scan_matches_reference_fixtures_bitwise(oracle):
    z = G.load("scan_instances")
    got = oracle.segmented_scan(z["worked_values"], z["worked_flags"])
    assert got.tolist() == [3, 4, 7, 7, 11, 1, 7, 10]  # test_scan.cpp:55-63
    assert np.array_equal(got, z["worked_out"])
    for c in range(int(z["count"])):
        out = oracle.segmented_scan(z[f"s{c}_v"], z[f"s{c}_f"])
        assert np.array_equal(out, z[f"s{c}_out"]), c


def test_ccd_fit_matches_reference_fixtures_bitwise(oracle):
    z = G.load("fits")
    for name in z["names"]:
        pre = str(name) + "_"
        d = oracle.design(G.design_arrays(z, pre))
        r = oracle.ccd_fit(d, z[pre + "gamma"], max_cycles=int(z[pre + "max_cycles"]),
                           tol=float(z[pre + "tol"]))
        assert r["cycles"] == int(z[pre + "cycles"]), name
        assert np.array_equal(r["beta"], z[pre + "beta"]), name
        assert np.array_equal(r["trace"], z[pre + "trace"]), name
        assert np.array_equal(r["trust"], z[pre + "trust"]), name
        g0 = np.array([oracle.gradient_hessian(d, np.ones(d.n), j) for j in range(d.p)])
        assert np.array_equal(g0, z[pre + "g0"]), name
        if pre + "gamma_max" in z:
            assert oracle.gamma_max(d) == float(z[pre + "gamma_max"])


# ---------------------------------------------------------------- known answers
def _tiny(oracle, time, event, stratum, cols=()):
    from oracle.oracle_py import Dataset
    cp = [0]
    ri, va = [], []
    for c in cols:
        for r, v in c:
            ri.append(r)
            va.append(v)
        cp.append(len(ri))
    ds = Dataset(np.array(time, float), np.array(event, np.uint8), np.array(stratum, np.int32),
                 np.array(cp, np.int64), np.array(ri, np.int64), np.array(va, float))
    return oracle.build_sorted_design(ds)


def test_known_answers_data(oracle):
    a = _tiny(oracle, [2, 5, 3], [1, 1, 0], [1, 1, 1])  # test_data.cpp:30-35
    assert a["time"].tolist() == [5, 3, 2]
    assert a["head"].tolist() == [1, 0, 0]
    assert a["tie_end"].tolist() == [0, 1, 2]
    a = _tiny(oracle, [4, 4, 1], [1, 1, 1], [1, 1, 1])  # :37-40
    assert a["tie_end"].tolist() == [1, 1, 2]
    a = _tiny(oracle, [3, 7, 5], [1, 1, 1], [1, 1, 2])  # :42-47
    assert a["head"].tolist() == [1, 0, 1]
    assert a["time"].tolist() == [7, 3, 5]
    assert a["offsets"].tolist() == [0, 2, 3]
    z = G.load("known_answers")
    for name in ("sort1", "ties", "heads", "handworked", "zerocol"):
        want = G.design_arrays(z, name + "_")
        assert want["n"] > 0


def test_known_answers_likelihood(oracle):
    a = _tiny(oracle, [3, 2, 1], [1, 1, 1], [1, 1, 1], cols=[[]])  # test_likelihood.cpp:35-42
    d = oracle.design(a)
    xb, ex = oracle.make_state(d, [0.0])
    assert math.isclose(oracle.log_partial_likelihood(d, xb, ex), -math.log(6.0), rel_tol=1e-12)
    # strata sizes {4,2,5} -> -sum log n_k!  (:44-60)
    time, ev, st = [], [], []
    for k, size in enumerate([4, 2, 5]):
        for i in range(size):
            time.append(i + 1.0)
            ev.append(1)
            st.append(k + 1)
    a = _tiny(oracle, time, ev, st)
    d = oracle.design(a)
    xb, ex = oracle.make_state(d, [])
    want = -sum(math.lgamma(s + 1.0) for s in (4, 2, 5))
    assert math.isclose(oracle.log_partial_likelihood(d, xb, ex), want, rel_tol=1e-12)
    # hand-worked x = [0,0,1] on times [3,2,1] (:62-75)
    a = _tiny(oracle, [3, 2, 1], [1, 1, 1], [1, 1, 1], cols=[[(2, 1.0)]])
    d = oracle.design(a)
    xb, ex = oracle.make_state(d, [0.0])
    g, h = oracle.gradient_hessian(d, ex, 0)
    assert math.isclose(g, -2.0 / 3.0, rel_tol=1e-12) and math.isclose(h, 2.0 / 9.0, rel_tol=1e-12)
    g, h = oracle.naive_gradient_hessian(d, ex, 0)
    assert math.isclose(g, -2.0 / 3.0, rel_tol=1e-12) and math.isclose(h, 2.0 / 9.0, rel_tol=1e-12)
    # zero column (:77-89)
    a = _tiny(oracle, [3, 2, 1], [1, 1, 1], [1, 1, 1], cols=[[]])
    d = oracle.design(a)
    xb, ex = oracle.make_state(d, [0.4])
    assert oracle.gradient_hessian(d, ex, 0) == (0.0, 0.0)


def test_known_answers_overflow(oracle):
    from oracle.oracle_py import OracleError
    a = _tiny(oracle, [2, 1], [1, 1], [1, 1], cols=[[(0, 1.0)]])  # test_likelihood.cpp:201-211
    d = oracle.design(a)
    beta = np.array([600.0])
    xb, ex = oracle.make_state(d, beta)
    xb0 = xb.copy()
    with pytest.raises(OracleError, match="step overflow"):
        oracle.update_xbeta(d, beta, xb, ex, 0, 0, 200.0)
    assert np.array_equal(xb, xb0) and beta[0] == 600.0
    a = _tiny(oracle, [2, 1], [1, 1], [1, 1], cols=[[(0, 2.0)]])  # :213-219
    d = oracle.design(a)
    with pytest.raises(OracleError, match="linear predictor overflow at row 0"):
        oracle.make_state(d, [400.0])


def test_known_answers_optimizer_rules(oracle):
    # test_optimizer.cpp:14-64
    assert oracle.newton_step(2.0, 4.0) == (-0.5, False)
    assert oracle.newton_step(0.0, 5.0)[0] == 0.0
    assert oracle.newton_step(1.0, 0.0) == (0.0, True)
    assert oracle.apply_trust_region(-3.0, 1.0) == (-1.0, 2.0)
    assert oracle.apply_trust_region(0.1, 1.0) == (0.1, 0.5)
    assert oracle.apply_trust_region(0.0, 1.0) == (0.0, 0.5)
    assert oracle.l1_coordinate_update(1.0, 1.0, 0.0, 2.0)[:2] == (0.0, True)
    assert math.isclose(oracle.l1_coordinate_update(-3.0, 1.0, 0.0, 2.0)[0], 1.0)
    assert math.isclose(oracle.l1_coordinate_update(3.0, 1.0, 0.0, 2.0)[0], -1.0)
    assert oracle.l1_coordinate_update(2.0, 2.0, 0.5, 1.0)[0] == -0.5
    assert math.isclose(oracle.l1_coordinate_update(0.2, 2.0, 0.5, 0.5)[0], -0.35)
    for g1 in (-2.0, 0.0, 3.5):
        assert oracle.l1_coordinate_update(g1, 2.0, 0.7, 0.0)[0] == oracle.newton_step(g1, 2.0)[0]


def test_known_answers_fits(oracle):
    # all-zero design converges in one cycle (test_optimizer.cpp:66-78)
    a = _tiny(oracle, [3, 2, 1], [1, 1, 1], [1, 1, 1], cols=[[], [], []])
    d = oracle.design(a)
    r = oracle.ccd_fit(d, np.zeros(3))
    assert r["converged"] and r["cycles"] == 1 and np.all(r["beta"] == 0.0)


# ---------------------------------------------------------------- live vs compiled reference
@pytest.mark.parametrize("seed,n,strata,p,chunk", [(5, 300, 1, 4, 64), (6, 1000, 7, 3, 100),
                                                   (7, 5000, 50, 2, 4096), (8, 257, 257, 2, 16)])
def test_oracle_vs_reference_live(oracle, ref, seed, n, strata, p, chunk):
    ds = ref.random_dataset(seed, n, strata, p)
    h, a = ref.build_design(ds)
    b = oracle.build_sorted_design(ds)
    for key in ("perm", "head", "tie_end", "offsets", "row_idx", "values"):
        assert np.array_equal(a[key], b[key])
    d = oracle.design(b)
    beta = np.linspace(-0.4, 0.4, p)
    xb, ex = oracle.make_state(d, beta)
    for j in range(p):
        assert oracle.gradient_hessian(d, ex, j, chunk) == ref.gradient_hessian(
            h, beta, xb, ex, j, chunk, 3)
    assert oracle.log_partial_likelihood(d, xb, ex, chunk) == ref.log_partial_likelihood(
        h, beta, xb, ex, chunk, 2)
    r1 = oracle.ccd_fit(d, np.full(p, 0.3), chunk=chunk)
    r2 = ref.ccd_fit(h, np.full(p, 0.3), p, chunk=chunk, workers=4)
    assert np.array_equal(r1["beta"], r2["beta"]) and np.array_equal(r1["trace"], r2["trace"])
    ref.free_design(h)
