"""Row sharding of a SortedDesign at stratum boundaries (multi-GPU path).

Risk sets are stratum-local prefixes of the time-descending layout
(proj/include/stratcox/data.hpp:3-5), so cutting the rows between strata
leaves every segmented scan inside one device: no scan carry crosses GPUs
(SURVEY.md §8e). Each rank then evaluates its local (sum x*delta, ratio sum,
variance sum) partial of every coordinate; the partials are exchanged and
summed in rank order, so every rank applies a bit-identical coordinate step.

The exchange itself runs inside the library, on the device: each rank owns
two 128-byte slots in device memory that every rank can load (P2P-mapped
across GPUs of one process, IPC-opened across processes, plain device memory
for ranks sharing one GPU — the "loopback"), and the persistent risk-suffix
cycle kernel publishes / polls them per coordinate (scx_xchg_*). This module
plans the shards, connects the ranks (in one process, or through
torch.distributed across processes) and combines the per-column facts the
ranks must agree on (column set, sum x*delta, max |x|).
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np

from .stratcox import SortedDesign


def plan_row_shards(stratum_offsets: np.ndarray, nranks: int) -> List[Tuple[int, int]]:
    """Split [0, N) into `nranks` contiguous row ranges at stratum boundaries,
    balancing row counts (greedy on the cumulative offsets). Ranks may get an
    empty range only when there are fewer strata than ranks."""
    off = np.asarray(stratum_offsets, dtype=np.int64)
    n = int(off[-1])
    k = off.shape[0] - 1
    if nranks < 1:
        raise ValueError("nranks must be >= 1")
    cuts = [0]
    for r in range(1, nranks):
        target = (n * r) // nranks
        # stratum boundary closest to the target, never before the previous cut
        idx = int(np.searchsorted(off, target))
        cands = [c for c in (idx - 1, idx) if 0 <= c <= k]
        best = min(cands, key=lambda c: abs(int(off[c]) - target))
        best = max(int(off[best]), cuts[-1])
        cuts.append(best)
    cuts.append(n)
    return [(cuts[r], cuts[r + 1]) for r in range(nranks)]


def shard_design(d: SortedDesign, lo: int, hi: int) -> SortedDesign:
    """Rows [lo, hi) of a sorted design (lo, hi on stratum boundaries), with
    every column restricted to those rows and re-based to the shard."""
    off = np.asarray(d.stratum_offsets, dtype=np.int64)
    k_lo = int(np.searchsorted(off, lo))
    k_hi = int(np.searchsorted(off, hi))
    if off[k_lo] != lo or off[k_hi] != hi:
        raise ValueError("shard bounds must lie on stratum boundaries")
    offsets = off[k_lo:k_hi + 1] - lo
    rows = np.asarray(d.row_idx, dtype=np.int64)
    cp = np.asarray(d.col_ptr, dtype=np.int64)
    p = cp.shape[0] - 1
    new_cp = np.zeros(p + 1, np.int64)
    keep_parts = []
    for j in range(p):
        seg = rows[cp[j]:cp[j + 1]]
        a = int(np.searchsorted(seg, lo))
        b = int(np.searchsorted(seg, hi))
        keep_parts.append((cp[j] + a, cp[j] + b))
        new_cp[j + 1] = new_cp[j] + (b - a)
    idx = np.concatenate([np.arange(a, b, dtype=np.int64) for a, b in keep_parts]) \
        if p else np.zeros(0, np.int64)
    new_rows = (rows[idx] - lo).astype(d.row_idx.dtype)
    vals = None if d.values is None else np.asarray(d.values)[idx]
    te = np.asarray(d.tie_group_end, dtype=np.int64)[lo:hi] - lo
    return SortedDesign(stratum_offsets=offsets, event=np.asarray(d.event)[lo:hi],
                        tie_group_end=te, col_ptr=new_cp, row_idx=new_rows, values=vals,
                        time=None if d.time is None else np.asarray(d.time)[lo:hi],
                        covariate_names=d.covariate_names)


def rank_ordered_sum(parts: np.ndarray, lin: float) -> Tuple[float, float]:
    """(gradient, Hessian) from per-rank (ratio sum, variance sum) partials and
    the global sum x*delta, summed in rank order — the association of the
    device exchange (xchg_values) and k_shard_step / the risk-suffix cycle."""
    a1 = 0.0
    a2 = 0.0
    for r in range(parts.shape[0]):
        a1 = float(parts[r, 0]) if r == 0 else a1 + float(parts[r, 0])
        a2 = float(parts[r, 1]) if r == 0 else a2 + float(parts[r, 1])
    return -lin + a1, a2


def _local_columns(dd):
    import ctypes as C

    from . import _capi
    from ._capi import ptr

    lib = _capi.load()
    p = dd.n_covariates()
    nz = np.zeros(p, np.uint8)
    lin = np.zeros(p)
    xmax = np.zeros(p)
    ok = C.c_int()
    rc = lib.scx_shard_local_columns(dd.handle, ptr(nz, C.c_uint8), ptr(lin, C.c_double),
                                     ptr(xmax, C.c_double), C.byref(ok))
    if rc:
        raise RuntimeError(lib.scx_last_error(dd.handle).decode())
    return nz, lin, xmax, int(ok.value)


def combine_columns(facts):
    """Per-rank (nonempty, lin, xmax, rs_ok) -> the global facts: OR, sum in
    rank order, max, AND."""
    nz = np.zeros_like(facts[0][0])
    lin = np.zeros_like(facts[0][1])
    xmax = np.zeros_like(facts[0][2])
    ok = 1
    for f in facts:  # rank order
        nz |= f[0]
        lin = lin + f[1]
        xmax = np.maximum(xmax, f[2])
        ok &= f[3]
    return nz, lin, xmax, ok


def _set_columns(dd, nz, lin, xmax, ok):
    import ctypes as C

    from . import _capi
    from ._capi import ptr

    lib = _capi.load()
    nz = np.ascontiguousarray(nz, np.uint8)
    lin = np.ascontiguousarray(lin, np.float64)
    xmax = np.ascontiguousarray(xmax, np.float64)
    rc = lib.scx_shard_set_columns(dd.handle, ptr(nz, C.c_uint8), ptr(lin, C.c_double),
                                   ptr(xmax, C.c_double), int(ok))
    if rc:
        raise RuntimeError(lib.scx_last_error(dd.handle).decode())


def connect_loopback(dds):
    """Ranks in ONE process (one DeviceDesign per rank, on one GPU or on
    several peer-accessible GPUs): exchange slots connected directly."""
    import ctypes as C

    from . import _capi

    lib = _capi.load()
    n = len(dds)
    slots = (C.c_void_p * n)()
    for r, dd in enumerate(dds):
        v = C.c_void_p()
        if lib.scx_xchg_slots(dd.handle, C.byref(v)):
            raise RuntimeError(lib.scx_last_error(dd.handle).decode())
        slots[r] = v.value
    for r, dd in enumerate(dds):
        if lib.scx_xchg_connect(dd.handle, n, r, slots):
            raise RuntimeError(lib.scx_last_error(dd.handle).decode())
    g = combine_columns([_local_columns(dd) for dd in dds])
    for dd in dds:
        _set_columns(dd, *g)


def upload_shards(design: SortedDesign, nranks: int, device: int = 0):
    """Loopback ranks sharing one GPU: the design cut at stratum boundaries,
    each shard uploaded with 1/nranks of the SMs (so the ranks' persistent
    cycle kernels co-reside) and connected."""
    from .stratcox import DeviceDesign, device_count  # noqa: F401

    import torch
    sms = torch.cuda.get_device_properties(device).multi_processor_count if \
        torch.cuda.is_available() else 148
    dds = [DeviceDesign(shard_design(design, lo, hi), device, sm_budget=sms // nranks)
           for lo, hi in plan_row_shards(design.stratum_offsets, nranks)]
    connect_loopback(dds)
    return dds


def fit_ranks(dds, penalty, config=None):
    """ccd_fit on every rank at once (one host thread per rank: the ranks'
    kernels wait on each other's exchange slots). Returns the ranks' results."""
    import threading

    from .stratcox import ccd_fit

    out = [None] * len(dds)
    err = [None] * len(dds)

    def run(r):
        try:
            out[r] = ccd_fit(dds[r], penalty, config)
        except Exception as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=run, args=(r,)) for r in range(len(dds))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    bad = [(r, e) for r, e in enumerate(err) if e is not None]
    if bad:  # a timeout on one rank is usually the echo of another rank's error
        r0, e0 = bad[0]
        raise type(e0)("; ".join(f"rank {r}: {e}" for r, e in bad))
    return out


def connect_ipc(dd, group=None):
    """One rank per process (torch.distributed initialised): the ranks' slot
    IPC handles are all-gathered, opened (P2P over NVLink between GPUs) and
    the per-column facts combined with all_gather."""
    import ctypes as C

    import torch.distributed as dist

    from . import _capi

    lib = _capi.load()
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    buf = C.create_string_buffer(64)
    if lib.scx_xchg_ipc_handle(dd.handle, buf):
        raise RuntimeError(lib.scx_last_error(dd.handle).decode())
    handles = [None] * world
    dist.all_gather_object(handles, bytes(buf.raw), group=group)
    if lib.scx_xchg_connect_ipc(dd.handle, world, rank, b"".join(handles)):
        raise RuntimeError(lib.scx_last_error(dd.handle).decode())
    facts = [None] * world
    dist.all_gather_object(facts, _local_columns(dd), group=group)
    _set_columns(dd, *combine_columns(facts))
