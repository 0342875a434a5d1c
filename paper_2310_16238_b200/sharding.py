"""Row sharding of a SortedDesign at stratum boundaries (multi-GPU path).

Risk sets are stratum-local prefixes of the time-descending layout
(proj/include/stratcox/data.hpp:3-5), so cutting the rows between strata
leaves every segmented scan inside one device: no scan carry crosses GPUs
(SURVEY.md §8e). Each rank then evaluates its local (sum x*delta, ratio sum,
variance sum) partial of every coordinate; the partials are exchanged and
summed in rank order, so every rank applies a bit-identical coordinate step.

The exchange itself runs inside the library (NCCL all-gather of 32 bytes per
coordinate on the context's stream, scx_comm_init); this module only plans
the shards and bootstraps the communicator through torch.distributed.
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


def rank_ordered_sum(parts: np.ndarray) -> Tuple[float, float]:
    """(gradient, Hessian) from per-rank (lin, ratio, variance, 0) partials,
    summed in rank order — the same association as the device k4_rank_step."""
    lin = 0.0
    a1 = 0.0
    a2 = 0.0
    for r in range(parts.shape[0]):
        lin += float(parts[r, 0])
        a1 += float(parts[r, 1])
        a2 += float(parts[r, 2])
    return -lin + a1, a2


def init_comm(dd, group=None):
    """Create the library's NCCL communicator for this rank, exchanging the
    128-byte unique id through torch.distributed (rank 0 generates it)."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    from . import _capi

    lib = _capi.load()
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    buf = C.create_string_buffer(128)
    if rank == 0:
        if lib.scx_comm_unique_id(buf) != 0:
            raise RuntimeError("scx_comm_unique_id failed (libnccl.so.2 missing?)")
    # an NCCL process group only moves CUDA tensors; gloo takes CPU ones
    if dist.get_backend(group) == "nccl":
        dev = torch.device("cuda", torch.cuda.current_device())
    else:
        dev = torch.device("cpu")
    t = torch.frombuffer(bytearray(buf.raw), dtype=torch.uint8).clone().to(dev)
    dist.broadcast(t, src=0, group=group)
    raw = bytes(t.cpu().tolist())
    rc = lib.scx_comm_init(dd.handle, world, rank, raw)
    if rc != 0:
        raise RuntimeError(lib.scx_last_error(dd.handle).decode())
