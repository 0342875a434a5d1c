"""Device build of the SortedDesign (scx_build_design, csrc/design_build.cu)
against the UNMODIFIED reference's build_sorted_design (data.cpp:68-147) and
validate_invariants (data.cpp:27-66), compiled in oracle/_ref.

Bit-exact on every integer array (perm, stratum offsets, tie-group ends, the
re-indexed CSC rows) and on the permuted event / values; the same validation
message for each kind of invalid input. Shapes cover heavy ties, -0.0 times,
one stratum, many strata, value and indicator columns, empty columns, columns
and strata spanning many 8192-entry radix tiles."""
import numpy as np
import pytest

import paper_2310_16238_b200 as sx
from oracle.oracle_py import Dataset, OracleError

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if sx.device_count() < 1:
        pytest.fail("no CUDA device visible to libstratcox_b200.so")


def _sx(ds, values=True):
    return sx.SurvivalDataset(time=ds.time, event=ds.event, stratum=ds.stratum,
                              col_ptr=ds.col_ptr, row_idx=ds.row_idx,
                              values=ds.values if values else None)


def _compare(ref, ds, values=True):
    h, a = ref.build_design(ds)
    ref.free_design(h)
    dd, perm = sx.build_design(_sx(ds, values))
    e = dd.export()
    dd.close()
    assert np.array_equal(perm, a["perm"])
    assert np.array_equal(e["offsets"], a["offsets"])
    assert np.array_equal(e["event"], a["event"])
    assert np.array_equal(e["tie_end"], a["tie_end"])
    assert np.array_equal(e["col_ptr"], a["col_ptr"])
    assert np.array_equal(e["row_idx"], a["row_idx"])
    if values:
        assert np.array_equal(e["values"], a["values"])
    return a


@pytest.mark.parametrize("seed,n,strata,p,density,grid", [
    (1, 1, 1, 1, 1.0, 4.0),            # one row
    (2, 500, 1, 3, 0.4, 3.0),          # one stratum, heavy ties
    (3, 20000, 7, 5, 0.3, 2.0),        # ties of thousands of rows
    (4, 30000, 9, 4, 0.2, 40.0),
    (5, 100000, 300, 6, 0.05, 1e9),    # continuous times, many strata
])
def test_random_datasets_match_reference(ref, seed, n, strata, p, density, grid):
    ds = ref.random_dataset(seed, n, strata, p, density, grid)
    _compare(ref, ds, values=True)
    _compare(ref, ds, values=False) if np.all(ds.values == 1.0) else None


def test_simulated_many_tiles_match_reference(ref):
    """Columns of ~5e4 entries and strata of 1e3 rows: segments over many tiles."""
    ds = ref.simulate(1_000_000, 8, 0.05, 0.5, 1000, 0.3, 21)
    a = _compare(ref, ds, values=False)
    assert a["k"] == 1000


def test_one_big_stratum_and_empty_and_dense_columns(ref):
    rng = np.random.default_rng(8)
    n = 300_000
    t = np.floor(rng.exponential(3.0, n))          # integer days: heavy ties
    t[rng.random(n) < 0.01] = -0.0                 # -0.0 ties with +0.0
    t[:5] = 0.0
    ev = (rng.random(n) < 0.6).astype(np.uint8)
    st = np.ones(n, np.int32)
    cols = [np.array([], np.int64), np.arange(n, dtype=np.int64),          # empty, dense
            np.flatnonzero(rng.random(n) < 0.3).astype(np.int64)]
    vals = [np.array([]), rng.normal(size=n), np.ones(cols[2].shape[0])]  # value, indicator
    cp = np.concatenate([[0], np.cumsum([c.shape[0] for c in cols])]).astype(np.int64)
    ds = Dataset(t, ev, st, cp, np.concatenate(cols), np.concatenate(vals))
    _compare(ref, ds, values=True)


def _bad(ref, ds):
    with pytest.raises(OracleError) as want:
        ref.build_design(ds)
    with pytest.raises(sx.ValidationError) as got:
        sx.build_design(_sx(ds))
    assert str(got.value) == str(want.value), (str(got.value), str(want.value))


def test_validation_messages_match_reference(ref):
    base = ref.random_dataset(11, 3000, 4, 3, 0.3, 6.0)

    def mod(**kw):
        d = dict(time=base.time.copy(), event=base.event.copy(), stratum=base.stratum.copy(),
                 col_ptr=base.col_ptr.copy(), row_idx=base.row_idx.copy(),
                 values=base.values.copy())
        for k, v in kw.items():
            v(d[k]) if callable(v) else d.__setitem__(k, v)
        return Dataset(d["time"], d["event"], d["stratum"], d["col_ptr"], d["row_idx"],
                       d["values"])

    def setv(i, v):
        return lambda a: a.__setitem__(i, v)

    _bad(ref, mod(time=setv(17, -1.0)))
    _bad(ref, mod(time=setv(1200, np.nan)))
    _bad(ref, mod(time=setv(5, np.inf), event=setv(3, 2)))      # first failing row wins
    _bad(ref, mod(event=setv(2999, 3)))
    _bad(ref, mod(stratum=setv(44, 0)))
    _bad(ref, mod(stratum=lambda s: s.__setitem__(s == 2, 3)))  # stratum 2 empty
    _bad(ref, mod(stratum=np.zeros(3000, np.int32)))            # no strata
    _bad(ref, mod(stratum=setv(9, 5000)))                       # max label 5000: empty 5
    r = base.row_idx
    c1 = int(base.col_ptr[1])
    _bad(ref, mod(row_idx=setv(c1 + 3, int(r[c1 + 2]))))         # not increasing (col 2)
    _bad(ref, mod(row_idx=setv(int(base.col_ptr[3]) - 1, 3000)))  # out of range (col 3)
    _bad(ref, mod(values=setv(c1 + 1, np.inf)))                  # non-finite value (col 2)
    _bad(ref, mod(values=setv(c1 + 1, np.nan), row_idx=setv(c1 + 5, -7)))


def test_fit_on_device_built_design_matches_reference_fit(ref, oracle):
    """End to end: device-built design -> device fit == reference fit."""
    ds = ref.simulate(200_000, 6, 0.05, 0.5, 400, 0.3, 4)
    h, a = ref.build_design(ds)
    gmax = ref.gamma_max(h)
    gamma = np.full(6, 0.1 * gmax)
    want = ref.ccd_fit(h, gamma, 6, max_cycles=60, tol=1e-8)
    ref.free_design(h)
    dd, _ = sx.build_design(_sx(ds, values=False))
    r = sx.ccd_fit(dd, sx.PenaltySpec(gamma), sx.OptimizerConfig(max_cycles=60, tolerance=1e-8))
    dd.close()
    assert r.cycles_used == want["cycles"]
    assert np.max(np.abs(r.beta - want["beta"])) <= 1e-8
