"""CPU: host logic of the multi-GPU path (rows sharded at stratum boundaries,
rank-ordered exchange of per-coordinate partials), on gloo with world size 2.

The device exchange runs inside the library (tests/test_sharded_fit.py runs
it on one GPU); here the same decomposition is checked with the oracle as
the per-shard evaluator:
  * shards start and end on stratum boundaries and cover every row once;
  * the rank-ordered sum of per-shard (gradient, Hessian) partials equals the
    single-design evaluation (1e-12 relative) — no risk set crosses shards;
  * a sharded CCD emulation (partials all-gathered over gloo, identical rule
    applied on every rank) reproduces the single-design fit.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2310_16238_b200.sharding import plan_row_shards, rank_ordered_sum, shard_design
from tests import _golden as G


def test_plan_row_shards_on_boundaries():
    off = np.array([0, 5, 9, 30, 31, 60, 100])
    for nr in (1, 2, 3, 4, 6):
        sh = plan_row_shards(off, nr)
        assert sh[0][0] == 0 and sh[-1][1] == 100
        for (a, b), (c, d) in zip(sh, sh[1:]):
            assert b == c
        for a, b in sh:
            assert a in off and b in off
    sh = plan_row_shards(np.arange(0, 1001, 10), 4)
    sizes = [b - a for a, b in sh]
    assert max(sizes) - min(sizes) <= 10


def _shard_arrays(sd):
    a = dict(offsets=np.asarray(sd.stratum_offsets, np.int64), event=np.asarray(sd.event, np.uint8),
             tie_end=np.asarray(sd.tie_group_end, np.int64),
             head=np.zeros(sd.n_rows, np.uint8), time=np.asarray(sd.time),
             col_ptr=np.asarray(sd.col_ptr, np.int64), row_idx=np.asarray(sd.row_idx, np.int64),
             values=np.ones(sd.nnz) if sd.values is None else np.asarray(sd.values))
    a["head"][a["offsets"][:-1]] = 1
    a["n"], a["p"], a["k"] = sd.n_rows, sd.n_covariates, sd.n_strata
    return a


def test_shard_partials_sum_to_full(oracle):
    z = G.load("fits")
    a = G.design_arrays(z, "c7_g1_")
    full = G.sorted_design(a)
    d = oracle.design(a)
    beta = np.linspace(-0.3, 0.4, a["p"])
    xb, ex = oracle.make_state(d, beta)
    for nr in (2, 3, 7):
        parts = []
        ll = 0.0
        for lo, hi in plan_row_shards(full.stratum_offsets, nr):
            sa = _shard_arrays(shard_design(full, lo, hi))
            sd = oracle.design(sa)
            sxb, sex = oracle.make_state(sd, beta)
            assert np.array_equal(sxb, xb[lo:hi])
            parts.append([oracle.gradient_hessian(sd, sex, j) for j in range(a["p"])])
            ll += oracle.log_partial_likelihood(sd, sxb, sex)
        for j in range(a["p"]):
            g, h = oracle.gradient_hessian(d, ex, j)
            gs = sum(p[j][0] for p in parts)
            hs = sum(p[j][1] for p in parts)
            assert G.close_rel(gs, g, 1e-12) and G.close_rel(hs, h, 1e-12)
        assert G.close_rel(ll, oracle.log_partial_likelihood(d, xb, ex), 1e-12)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch
    from oracle.oracle_py import Oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    z = G.load("fits")
    a = G.design_arrays(z, "c5_k10_l1_")
    full = G.sorted_design(a)
    lo, hi = plan_row_shards(full.stratum_offsets, world)[rank]
    sd = orc.design(_shard_arrays(shard_design(full, lo, hi)))
    p = a["p"]
    gamma = z["c5_k10_l1_gamma"]
    beta = np.zeros(p)
    trust = np.ones(p)
    xb, ex = orc.make_state(sd, beta)
    updates = 0
    local_obj_trace = []
    for cycle in range(200):
        max_step = 0.0
        for j in range(p):
            g_r, h_r = orc.gradient_hessian(sd, ex, j)
            t = torch.tensor([g_r, h_r, 0.0, 0.0], dtype=torch.float64)
            gathered = [torch.zeros(4, dtype=torch.float64) for _ in range(world)]
            dist.all_gather(gathered, t)  # the 32-byte per-coordinate exchange
            parts = np.stack([x.numpy() for x in gathered])
            # rank-ordered sum (lin folded into the gradient partial here)
            g = float(np.sum(parts[:, 0])) if world == 1 else sum(float(x) for x in parts[:, 0])
            h = sum(float(x) for x in parts[:, 1])
            step, _, _ = orc.l1_coordinate_update(g, h, beta[j], gamma[j])
            applied, _ = orc.apply_trust_region(step, trust[j])
            if applied != 0.0:
                updates = orc.update_xbeta(sd, beta, xb, ex, updates, j, applied)
            trust[j] = max(2.0 * abs(applied), trust[j] * 0.5)
            max_step = max(max_step, abs(applied))
        ll_r = orc.log_partial_likelihood(sd, xb, ex)
        t = torch.tensor([ll_r], dtype=torch.float64)
        lls = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(lls, t)
        ll = sum(float(x) for x in lls)
        local_obj_trace.append(-ll + float(np.sum(gamma * np.abs(beta))))
        if max_step < float(z["c5_k10_l1_tol"]):
            break
    out[rank] = (beta.copy(), local_obj_trace, cycle + 1)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_ccd_emulation_gloo_world2():
    z = G.load("fits")
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    b0, tr0, c0 = out[0]
    b1, tr1, c1 = out[1]
    assert b0.tobytes() == b1.tobytes()  # every rank applies identical steps
    assert tr0 == tr1 and c0 == c1
    want = z["c5_k10_l1_beta"]
    assert np.max(np.abs(b0 - want)) <= 1e-8
    assert c0 == int(z["c5_k10_l1_cycles"])


def test_rank_ordered_sum_matches_kernel_order():
    parts = np.array([[3.0, 0.5], [1.5, 0.25], [0.25, 1.0]])
    g, h = rank_ordered_sum(parts, 3.5)
    assert g == -3.5 + ((3.0 + 1.5) + 0.25) and h == (0.5 + 0.25) + 1.0


def test_combine_columns_or_sum_max_and():
    from paper_2310_16238_b200.sharding import combine_columns
    f0 = (np.array([1, 0, 0], np.uint8), np.array([1.0, 0.0, 0.0]), np.array([2.0, 0.0, 0.0]), 1)
    f1 = (np.array([1, 1, 0], np.uint8), np.array([0.5, 2.0, 0.0]), np.array([1.0, 3.0, 0.0]), 0)
    nz, lin, xmax, ok = combine_columns([f0, f1])
    assert nz.tolist() == [1, 1, 0] and lin.tolist() == [1.5, 2.0, 0.0]
    assert xmax.tolist() == [2.0, 3.0, 0.0] and ok == 0
