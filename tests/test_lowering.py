"""Lowering transforms (BASELINE configs 2-3) against the
reference's make_time_varying + lower_pipeline: the augmented stratified
dataset and the column map are identical array for array (host, CPU tests);
a fit on the lowered design matches the oracle (GPU test)."""
import numpy as np
import pytest

import paper_2310_16238_b200 as sx
from tests import _golden as G


def _subjects_dataset(ref, n, p, seed, grid):
    ds = ref.random_dataset(seed, n, 1, p, 0.3, grid)
    return ds


def _sx(ds, subject=None):
    return sx.SurvivalDataset(time=ds.time, event=ds.event, stratum=ds.stratum, col_ptr=ds.col_ptr,
                              row_idx=ds.row_idx, values=ds.values, subject=subject)


@pytest.mark.parametrize("n,p,seed,cuts,splits", [
    (300, 3, 1, [0, 2, 4, 6, 8], {}),
    (500, 4, 2, [0, 1, 2.5, 4, 8], {1: [2.5], 3: [1, 4]}),
    (200, 2, 3, [0, 3, 8], {0: [3]}),
    (1000, 5, 4, list(np.linspace(0, 8, 21)), {0: list(np.linspace(0, 8, 21)[1:-1]), 2: [4.0]}),
])
def test_lowering_matches_reference(ref, n, p, seed, cuts, splits):
    ds = _subjects_dataset(ref, n, p, seed, 8)       # integer-grid times in [0, 8]: ties with cuts
    subj = np.arange(n, dtype=np.int64) * 3 + 7
    want, wsubj, wsrc, wwin = ref.lower_pipeline(ds, cuts, splits, subject=subj)
    got, cmap = sx.lower_time_varying(_sx(ds, subj), cuts, splits)
    assert np.array_equal(got.time, want.time)
    assert np.array_equal(got.event, want.event)
    assert np.array_equal(got.stratum, want.stratum)
    assert np.array_equal(got.subject, wsubj)
    assert np.array_equal(got.col_ptr, want.col_ptr)
    assert np.array_equal(got.row_idx, want.row_idx)
    assert np.array_equal(got.values, want.values)
    assert [c.source for c in cmap] == wsrc.tolist()
    assert [c.window for c in cmap] == wwin.tolist()
    assert int(got.event.sum()) == int(ds.event.sum())  # events conserved (transforms.hpp:101)


def test_lowering_validation(ref):
    ds = _subjects_dataset(ref, 50, 2, 9, 8)
    with pytest.raises(sx.ValidationError, match="first cut point must be 0"):
        sx.lower_time_varying(_sx(ds), [1, 8])
    with pytest.raises(sx.ValidationError, match="cut points do not cover follow-up"):
        sx.lower_time_varying(_sx(ds), [0, 4])
    with pytest.raises(sx.ValidationError, match="is not a cut point"):
        sx.lower_time_varying(_sx(ds), [0, 4, 8], {0: [3]})
    with pytest.raises(sx.ValidationError, match="outside the follow-up window"):
        sx.lower_time_varying(_sx(ds), [0, 4, 8], {0: [8]})


@pytest.mark.gpu
def test_fit_on_lowered_design_matches_oracle(ref, oracle):
    """BASELINE config 3 in miniature: subjects x time bins, one covariate's
    coefficient split at every interior cut, fitted on the device."""
    ds = _subjects_dataset(ref, 2000, 4, 5, 20)
    cuts = list(np.linspace(0, 20, 11))
    low, cmap = sx.lower_time_varying(_sx(ds), cuts, {0: cuts[1:-1]})
    dd, perm = sx.build_design(low)
    from oracle.oracle_py import Dataset
    h, a = ref.build_design(Dataset(low.time, low.event, low.stratum, low.col_ptr, low.row_idx,
                                    low.values))
    ref.free_design(h)
    assert np.array_equal(perm, a["perm"])
    d = oracle.design(a)
    p = a["p"]
    gamma = np.full(p, 2.0)
    want = oracle.ccd_fit(d, gamma, max_cycles=100, tol=1e-8)
    r = sx.ccd_fit(dd, sx.PenaltySpec(gamma), sx.OptimizerConfig(max_cycles=100, tolerance=1e-8))
    assert r.cycles_used == want["cycles"]
    assert np.max(np.abs(r.beta - want["beta"])) <= 1e-8
    assert np.allclose(r.objective_trace, want["trace"], rtol=1e-10, atol=0)


@pytest.mark.gpu
@pytest.mark.parametrize("n,p,seed,cuts,splits,values", [
    (500, 4, 2, [0, 1, 2.5, 4, 8], {1: [2.5], 3: [1, 4]}, False),
    (3000, 5, 4, list(np.linspace(0, 8, 21)), {0: list(np.linspace(0, 8, 21)[1:-1]), 2: [4.0]}, True),
    (200000, 6, 6, list(np.linspace(0, 20, 21)), {0: list(np.linspace(0, 20, 21)[1:-1])}, False),
])
def test_device_lowering_matches_reference(ref, n, p, seed, cuts, splits, values):
    """scx_build_lowered_design (subjects uploaded, augmentation + build on the
    device) gives the reference's lower_pipeline + build_sorted_design: perm,
    offsets, tie ends, rows and values bit for bit, and the column map."""
    from oracle.oracle_py import Dataset
    ds = ref.random_dataset(seed, n, 1, p, 0.3, 8 if n < 10000 else 20)
    subj = np.arange(n, dtype=np.int64) * 3 + 7
    if values:
        ds = Dataset(ds.time, ds.event, ds.stratum, ds.col_ptr, ds.row_idx,
                     np.round(ds.values * 3) / 2)  # some zero values: never stored
    low, wsubj, wsrc, wwin = ref.lower_pipeline(ds, cuts, splits, subject=subj)
    h, a = ref.build_design(low)
    ref.free_design(h)
    dd, cmap = sx.build_lowered_design(_sx(ds, subj), cuts, splits)
    e = dd.export()
    dd.close()
    assert [c.source for c in cmap] == wsrc.tolist() and [c.window for c in cmap] == wwin.tolist()
    for k in ("offsets", "event", "tie_end", "col_ptr", "row_idx"):
        assert np.array_equal(e[k], a[k]), k
    assert np.array_equal(e["values"], a["values"])


@pytest.mark.gpu
def test_device_lowering_validation_messages(ref):
    ds = _subjects_dataset(ref, 50, 2, 9, 8)
    for cuts, splits, msg in [([1, 8], None, "first cut point must be 0"),
                              ([0, 4], None, "cut points do not cover follow-up"),
                              ([0, 4, 8], {0: [3]}, "is not a cut point")]:
        with pytest.raises(sx.ValidationError, match=msg):
            sx.build_lowered_design(_sx(ds), cuts, splits)
