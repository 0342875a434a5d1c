"""The 256-update refresh over the row-slice copy of the design (k_refresh_ell).

make_state / refresh_xbeta (likelihood.cpp:19-58) fold eta[r] = sum_j x_rj
beta_j over the nonzero-beta columns in ascending j from 0.0, skipping
beta_j == 0. The row-slice refresh folds each row in that order, so eta must
be BIT-identical to the column-by-column fold below (numpy: per column,
eta[rows] += x * b, products rounded before the add — exactly the
reference's statement at likelihood.cpp:42) and exp_xbeta exp(eta) to 2 ulp.

Layout cases: u16 column ids with beta staged in shared memory (p <= 12800),
u32 column ids with beta read from global memory (p > 65535), value columns
mixed with indicator columns, rows without entries, a row count that is not a
multiple of the 32-row slice, and the +-700 overflow check.
"""
import numpy as np
import pytest

import paper_2310_16238_b200 as sx
from paper_2310_16238_b200 import synthetic
from paper_2310_16238_b200.stratcox import SortedDesign

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if sx.device_count() < 1:
        pytest.fail("no CUDA device visible to libstratcox_b200.so")


def _design(n, p, k, density, seed, value_frac=0.0):
    syn = synthetic.generate(n, p, k, density, seed=seed, device="cpu", pin=False)
    d = syn.sorted_design()
    vals = None
    if value_frac > 0:
        rng = np.random.default_rng(seed)
        nnz = int(d.col_ptr[-1])
        vals = np.ones(nnz)
        for j in np.flatnonzero(rng.random(p) < value_frac):
            b, e = int(d.col_ptr[j]), int(d.col_ptr[j + 1])
            vals[b:e] = rng.normal(0.0, 1.5, e - b)
        d = SortedDesign(stratum_offsets=d.stratum_offsets, event=d.event,
                         tie_group_end=d.tie_group_end, col_ptr=d.col_ptr, row_idx=d.row_idx,
                         values=vals)
    return d, vals


def _fold(d, vals, beta):
    n = d.event.shape[0]
    eta = np.zeros(n)
    cp = np.asarray(d.col_ptr)
    rows = np.asarray(d.row_idx)
    for j in np.flatnonzero(beta != 0.0):
        b, e = int(cp[j]), int(cp[j + 1])
        x = np.ones(e - b) if vals is None else vals[b:e]
        np.add.at(eta, rows[b:e], x * beta[j])  # one entry per (row, column): order = ascending j
    return eta


@pytest.mark.parametrize("n,p,k,density,value_frac,active", [
    (200_003, 300, 40, 0.05, 0.0, 0.3),      # u16 ids, beta in shared memory, ragged last slice
    (100_000, 120, 20, 0.08, 0.5, 0.6),      # value columns mixed with indicators
    (40_000, 70_000, 10, 0.0004, 0.2, 0.4),  # u32 ids, beta from global memory
    (50_000, 20_000, 10, 0.002, 0.0, 0.05),  # u16 ids, p above the shared-memory limit
])
def test_refresh_matches_column_fold_bit_exactly(n, p, k, density, value_frac, active):
    d, vals = _design(n, p, k, density, 5, value_frac)
    dd = sx.upload(d)
    try:
        rng = np.random.default_rng(7)
        beta = rng.normal(0.0, 0.05, p) * (rng.random(p) < active)
        st = sx.make_state(dd, beta)
        want = _fold(d, vals, beta)
        got = st.xbeta
        assert got.tobytes() == want.tobytes()
        ex = np.exp(want)  # CUDA exp vs libm: within 2 ulp
        assert np.max(np.abs(st.exp_xbeta - ex) / ex) <= 4.5e-16
        # a second refresh from the same beta reproduces it
        sx.refresh_xbeta(dd, st)
        assert st.xbeta.tobytes() == want.tobytes()
    finally:
        dd.close()


def test_refresh_rows_without_entries_and_overflow():
    d, _ = _design(33_000, 50, 5, 0.01, 9)  # ~60% of rows have no entry
    dd = sx.upload(d)
    try:
        beta = np.zeros(50)
        beta[3] = 0.25
        st = sx.make_state(dd, beta)
        want = _fold(d, None, beta)
        assert st.xbeta.tobytes() == want.tobytes()
        assert np.count_nonzero(want == 0.0) > 0
        beta[3] = 800.0  # every row of column 3 overflows the +-700 bound
        first = int(np.min(np.asarray(d.row_idx)[int(d.col_ptr[3]):int(d.col_ptr[4])]))
        with pytest.raises(sx.NumericError, match=f"linear predictor overflow at row {first}"):
            sx.make_state(dd, beta)
    finally:
        dd.close()
