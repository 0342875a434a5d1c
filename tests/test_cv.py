"""Regularisation path / k-fold CV driver against the
compiled reference (oracle/_ref): fold labels and the gamma grid are
bit-identical (host, CPU tests); the device design build, every held-out
score and gamma* agree with the reference's kfold_select_gamma (GPU tests).
"""
import numpy as np
import pytest

import paper_2310_16238_b200 as sx
from tests import _golden as G


def _sx_dataset(ds, subject=None):
    return sx.SurvivalDataset(time=ds.time, event=ds.event, stratum=ds.stratum,
                              col_ptr=ds.col_ptr, row_idx=ds.row_idx, values=ds.values,
                              subject=subject)


def _subjects(n, rows_per_subject, seed):
    """Subject ids for augmented-style data: runs of 1..rows_per_subject rows."""
    rng = np.random.default_rng(seed)
    out = np.empty(n, np.int64)
    r, s = 0, 1
    while r < n:
        k = int(rng.integers(1, rows_per_subject + 1))
        out[r:r + k] = 1000 + 7 * s
        r += k
        s += 1
    return out


@pytest.mark.parametrize("n,folds,seed,rps", [(200, 5, 1, 1), (1000, 10, 42, 3),
                                               (57, 7, 9, 2), (5000, 2, 123456789, 4)])
def test_fold_assignment_matches_reference(ref, n, folds, seed, rps):
    ds = ref.random_dataset(seed, n, 3, 2, 0.3, 8)
    subj = _subjects(n, rps, seed) if rps > 1 else None
    want = ref.fold_assignment(ds, folds, seed, subject=subj)
    got = sx.fold_assignment(_sx_dataset(ds, subj), folds, seed)
    assert np.array_equal(got, want)
    if subj is not None:  # all rows of a subject land in one fold
        for s in np.unique(subj):
            assert len(set(got[subj == s].tolist())) == 1


def test_fold_assignment_validation(ref):
    ds = ref.random_dataset(3, 10, 1, 1, 0.5, 8)
    with pytest.raises(sx.ValidationError, match="folds must be >= 2"):
        sx.fold_assignment(_sx_dataset(ds), 1, 0)
    with pytest.raises(sx.ValidationError, match="degenerate fold"):
        sx.fold_assignment(_sx_dataset(ds), 11, 0)


def test_default_gamma_grid_matches_reference(ref):
    for gmax, size in [(57505.3679, 20), (1.0, 1), (3.5, 7)]:
        got = sx.default_gamma_grid(gmax, size)
        want = ref.default_gamma_grid(gmax, size)
        assert np.array_equal(got, want)


# ---------------------------------------------------------------- on the device
@pytest.mark.gpu
def test_build_design_matches_reference(ref, oracle):
    ds = ref.random_dataset(77, 30000, 9, 4, 0.2, 40)   # heavy ties, value columns
    h, a = ref.build_design(ds)
    ref.free_design(h)
    dd, perm = sx.build_design(_sx_dataset(ds))
    assert np.array_equal(perm, a["perm"])              # bit-exact sorted indexing
    info = dd.info()
    assert (info["n_rows"], info["n_strata"], info["p"]) == (a["n"], a["k"], a["p"])
    d = oracle.design(a)
    beta = np.array([0.3, -0.2, 0.1, 0.05])
    st = sx.make_state(dd, beta)
    xb, ex = oracle.make_state(d, beta)
    assert np.array_equal(st.xbeta, xb)
    for j in range(a["p"]):
        g, hh = oracle.gradient_hessian(d, ex, j)
        r = sx.gradient_hessian(dd, st, j)
        assert G.close_rel(r.gradient, g, 1e-10) and G.close_rel(r.hessian, hh, 1e-10)


@pytest.mark.gpu
@pytest.mark.parametrize("n,p,k,folds,ngrid,rps", [(3000, 6, 3, 5, 6, 1), (4000, 8, 5, 4, 5, 3)])
def test_kfold_select_gamma_matches_reference(ref, n, p, k, folds, ngrid, rps):
    ds = ref.simulate(n, p, 0.2, 0.5, k, 0.3, 17)
    subj = _subjects(n, rps, 5) if rps > 1 else None
    h, a = ref.build_design(ds)
    gmax = ref.gamma_max(h)
    ref.free_design(h)
    grid = ref.default_gamma_grid(gmax, ngrid)
    tmpl = np.ones(p)
    tmpl[0] = 0.0  # one unpenalized coefficient
    want = ref.kfold_select_gamma(ds, tmpl, folds, grid, 11, tol=1e-8, subject=subj)
    got = sx.kfold_select_gamma(_sx_dataset(ds, subj), sx.PenaltySpec(tmpl), folds, grid, seed=11,
                                config=sx.OptimizerConfig(tolerance=1e-8))
    assert got.gamma_star == want["gamma_star"]
    assert len(got.warnings) == want["n_warnings"]
    # held-out partial log-likelihoods of fits converged to 1e-8
    assert np.allclose(got.fold_scores, want["fold_scores"], rtol=1e-9, atol=0)
    assert np.allclose(got.mean_scores, want["mean_scores"], rtol=1e-9, atol=0)


@pytest.mark.gpu
def test_kfold_validation_messages(ref):
    ds = ref.random_dataset(5, 100, 2, 2, 0.4, 8)
    data = _sx_dataset(ds)
    with pytest.raises(sx.ValidationError, match="gamma grid is empty"):
        sx.kfold_select_gamma(data, sx.PenaltySpec(np.ones(2)), 3, [])
    with pytest.raises(sx.ValidationError, match="strictly increasing"):
        sx.kfold_select_gamma(data, sx.PenaltySpec(np.ones(2)), 3, [2.0, 1.0])
    with pytest.raises(sx.ValidationError, match="folds must be >= 2"):
        sx.kfold_select_gamma(data, sx.PenaltySpec(np.ones(2)), 1, [1.0])
