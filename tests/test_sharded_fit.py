"""Row-sharded fits through the library's device-side exchange, on ONE GPU
(VERDICT r1 "make multi-GPU real, without hardware").

Two (or three) scx contexts on the same B200 play the ranks: each uploads the
rows of whole strata it owns (sharding.plan_row_shards / shard_design) with
1/nranks of the SMs, the ranks' exchange slots are connected in-process
("loopback": the same device memory a P2P mapping would expose across GPUs),
and ccd_fit runs on every rank at once from its own host thread. Per
coordinate the ranks exchange only the partial sums — inside the persistent
risk-suffix cycle kernel (device flags, no host round trip) or, off that
path, through one-thread exchange kernels.

Checked: every rank ends with bit-identical coefficients; they match the
single-device fit and the oracle (the reference restatement) within 1e-8
with the same cycle count; the risk-suffix cycle really ran per shard; a
column with rows on one shard only; the per-coordinate sharded path (a
design too small for the chunked layout)."""
import numpy as np
import pytest

import paper_2310_16238_b200 as sx
from paper_2310_16238_b200 import sharding
from tests import _golden as G

pytestmark = pytest.mark.gpu

BETA_ATOL = 1e-8


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if sx.device_count() < 1:
        pytest.fail("no CUDA device visible to libstratcox_b200.so")


def _sim_design(ref, n, p, k, seed, density=0.05):
    ds = ref.simulate(n, p, density, 0.5, k, 0.3, seed)
    h, a = ref.build_design(ds)
    ref.free_design(h)
    return a


def _check(oracle, a, gamma, nranks, max_cycles=60, tol=1e-8, expect_rs=True):
    design = G.sorted_design(a, values=False)
    d = oracle.design(a)
    cfg = sx.OptimizerConfig(max_cycles=max_cycles, tolerance=tol)
    want = oracle.ccd_fit(d, gamma, max_cycles=max_cycles, tol=tol)
    dd1 = sx.upload(design)
    single = sx.ccd_fit(dd1, sx.PenaltySpec(gamma), cfg)
    dd1.close()
    dds = sharding.upload_shards(design, nranks)
    try:
        res = sharding.fit_ranks(dds, sx.PenaltySpec(gamma), cfg)
        stats = [dd.fit_path_stats() for dd in dds]
    finally:
        for dd in dds:
            dd.close()
    for r in res[1:]:
        assert r.beta.tobytes() == res[0].beta.tobytes(), "ranks disagree"
        assert r.cycles_used == res[0].cycles_used
    r0 = res[0]
    assert r0.cycles_used == want["cycles"] == single.cycles_used
    assert np.max(np.abs(r0.beta - want["beta"])) <= BETA_ATOL
    assert np.max(np.abs(r0.beta - single.beta)) <= BETA_ATOL
    assert np.allclose(r0.objective_trace, want["trace"], rtol=1e-10, atol=0)
    if expect_rs:
        assert all(s["risk_suffix_launches"] > 0 for s in stats), stats
    return r0, stats


def test_two_shards_risk_suffix_cycle_match_single_device_and_oracle(oracle, ref):
    a = _sim_design(ref, 1_300_000, 6, 1300, 7)
    dd = sx.upload(G.sorted_design(a, values=False))
    gmax = sx.gamma_max(dd)
    dd.close()
    _check(oracle, a, np.full(a["p"], 0.05 * gmax), 2)


def test_three_shards_and_a_column_on_one_shard_only(oracle, ref):
    a = _sim_design(ref, 1_500_000, 5, 1500, 8)
    # an extra column whose rows all lie in the first tenth of the rows (rank 0 only)
    n = a["n"]
    rng = np.random.default_rng(2)
    extra = np.flatnonzero(rng.random(n // 10) < 0.2).astype(np.int64)
    a["col_ptr"] = np.concatenate([a["col_ptr"], [a["col_ptr"][-1] + extra.shape[0]]])
    a["row_idx"] = np.concatenate([a["row_idx"], extra])
    a["values"] = np.ones(a["row_idx"].shape[0])
    a["p"] += 1
    dd = sx.upload(G.sorted_design(a, values=False))
    gmax = sx.gamma_max(dd)
    dd.close()
    gamma = np.full(a["p"], 0.05 * gmax)
    gamma[-1] = 0.0  # unpenalised: the one-shard column always moves
    _check(oracle, a, gamma, 3)


def test_per_coordinate_sharded_path_small_design(oracle):
    """C1-sized design: too small for the chunked layout, so every coordinate
    goes through K1 partials + the one-thread exchange kernels."""
    z = G.load("fits")
    a = G.design_arrays(z, "cfg1_l1_")
    _check(oracle, a, z["cfg1_l1_gamma"], 2, max_cycles=40, expect_rs=False)


def test_two_shards_few_large_strata(oracle, ref):
    """Four large strata: each rank's rows (two whole strata) take the
    risk-suffix cycle on chunks of whole tiles, the carries meeting across
    that rank's CTAs, and the partial sums across the ranks."""
    a = _sim_design(ref, 2_800_000, 4, 4, 9, density=0.03)
    dd = sx.upload(G.sorted_design(a, values=False))
    gmax = sx.gamma_max(dd)
    dd.close()
    _check(oracle, a, np.full(a["p"], 0.05 * gmax), 2)
