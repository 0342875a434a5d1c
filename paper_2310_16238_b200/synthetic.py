"""Synthetic workloads of the BASELINE shapes, generated on the GPU.

Restates the statistical model of the reference generator
(proj/src/simulate.cpp:9-102): binary sparse X with geometric gaps
(density d), beta_true ~ N(0,1) * Bernoulli(1 - beta_sparsity),
T ~ Exp(rate exp(x'beta)), uniform censoring C ~ U(0, cmax) with cmax bisected
to a target censored fraction, strata assigned round-robin. It is not
bit-identical to the reference (libstdc++ RNG streams are implementation-
defined; the reference itself is used for every parity fixture) — it exists
to build the C4/C5 shapes (10^9 nonzeros) in seconds instead of minutes.

Then it builds the SortedDesign exactly as build_sorted_design
(proj/src/data.cpp:68-147) defines it: stable sort by (stratum asc, time
desc), stratum offsets, tie-group ends, columns re-indexed to sorted rows.
torch is used here as device plumbing for setup only; nothing here is on the
timed path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass
class SynthDesign:
    n: int
    p: int
    k: int
    offsets: np.ndarray      # int64 [K+1]
    event: np.ndarray        # uint8 [N]
    tie_end: np.ndarray      # int64 [N]
    col_ptr: np.ndarray      # int64 [P+1]
    rows: np.ndarray         # int32 [nnz] (pinned when possible)
    true_beta: np.ndarray
    gen_seconds: float = 0.0
    rows_owner: object = None  # pinned torch tensor backing `rows`

    @property
    def nnz(self) -> int:
        return int(self.col_ptr[-1])

    def sorted_design(self):
        from .stratcox import SortedDesign
        return SortedDesign(stratum_offsets=self.offsets, event=self.event,
                            tie_group_end=self.tie_end, col_ptr=self.col_ptr, row_idx=self.rows,
                            values=None)


def generate(n: int, p: int, k: int, density: float = 0.01, beta_sparsity: float = 0.8,
             censoring: float = 0.3, seed: int = 11, device: str = "cuda",
             col_chunk: int = 1000, pin: bool = True) -> SynthDesign:
    import time

    import torch

    t0 = time.perf_counter()
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    dev = torch.device(device)

    # ---- sparse binary X by geometric gaps, column by column (simulate.cpp:27-39)
    log1m = math.log1p(-density)
    mean = n * density
    m = int(mean + 8.0 * math.sqrt(mean) + 64)
    beta = torch.randn(p, generator=g, device=dev, dtype=torch.float64)
    keep = torch.rand(p, generator=g, device=dev, dtype=torch.float64) < (1.0 - beta_sparsity)
    beta = torch.where(keep, beta, torch.zeros_like(beta))
    eta = torch.zeros(n, device=dev, dtype=torch.float64)
    col_rows = []
    counts = torch.zeros(p, device=dev, dtype=torch.int64)
    for c0 in range(0, p, col_chunk):
        c1 = min(p, c0 + col_chunk)
        u = torch.rand((c1 - c0, m), generator=g, device=dev, dtype=torch.float32).clamp_min_(1e-30)
        gaps = 1 + torch.floor(torch.log(u) / log1m).to(torch.int64)
        del u
        pos = torch.cumsum(gaps, dim=1) - 1
        del gaps
        mask = pos < n
        cnt = mask.sum(dim=1)
        if bool((cnt == m).any()):
            raise RuntimeError("gap buffer too short")
        counts[c0:c1] = cnt
        rows = pos[mask]  # row-major over (column, position): per-column ascending
        del pos
        colid = torch.repeat_interleave(torch.arange(c0, c1, device=dev), cnt)
        bsel = beta[colid]
        nz = bsel != 0
        eta.index_add_(0, rows[nz], bsel[nz])
        col_rows.append(rows)
        del mask, colid, bsel, nz

    # ---- times and calibrated uniform censoring (simulate.cpp:48-97)
    u = torch.rand(n, generator=g, device=dev, dtype=torch.float64).clamp_min_(1e-300)
    t_event = -torch.log(u) / torch.exp(eta)
    del u, eta
    if censoring > 0.0:
        def frac(cmax):
            return float(torch.clamp(t_event / cmax, max=1.0).mean())
        lo, hi = 1e-12, 1.0
        while frac(hi) > censoring and hi < 1e300:
            hi *= 2.0
        for _ in range(100):
            mid = 0.5 * (lo + hi)
            if frac(mid) > censoring:
                lo = mid
            else:
                hi = mid
        cmax = 0.5 * (lo + hi)
        cens = torch.rand(n, generator=g, device=dev, dtype=torch.float64) * cmax
        event = t_event <= cens
        time_ = torch.where(event, t_event, cens)
        del cens
    else:
        event = torch.ones(n, dtype=torch.bool, device=dev)
        time_ = t_event
    del t_event
    stratum = (torch.arange(n, device=dev) % k).to(torch.int32) + 1

    # ---- build_sorted_design (data.cpp:75-145): stable sort (stratum asc, time desc)
    perm = torch.argsort(-time_, stable=True)
    perm = perm[torch.argsort(stratum[perm], stable=True)]
    inv = torch.empty_like(perm)
    inv[perm] = torch.arange(n, device=dev)
    s_time = time_[perm]
    s_str = stratum[perm]
    s_event = event[perm].to(torch.uint8)
    del time_, stratum, event
    kk = torch.bincount(s_str.to(torch.int64), minlength=k + 1)[1:]
    offsets = torch.zeros(k + 1, dtype=torch.int64, device=dev)
    offsets[1:] = torch.cumsum(kk, 0)
    # tie groups: last row sharing (stratum, time)
    is_end = torch.ones(n, dtype=torch.bool, device=dev)
    is_end[:-1] = (s_str[1:] != s_str[:-1]) | (s_time[1:] != s_time[:-1])
    idx = torch.where(is_end, torch.arange(n, device=dev), torch.full((n,), n, device=dev))
    tie_end = torch.flip(torch.cummin(torch.flip(idx, [0]), 0).values, [0])
    del idx, is_end, s_time, s_str, perm

    # ---- re-index columns to sorted rows, ascending within each column
    out_rows = []
    c0 = 0
    for rows in col_rows:
        nc = min(col_chunk, p - c0)
        cnt = counts[c0:c0 + nc]
        colid = torch.repeat_interleave(torch.arange(nc, device=dev), cnt)
        key = colid * n + inv[rows]
        del rows, colid
        key, _ = torch.sort(key)
        out_rows.append((key % n).to(torch.int32))
        del key
        c0 += nc
    del col_rows, inv
    rows_all = torch.cat(out_rows)
    del out_rows
    col_ptr = torch.zeros(p + 1, dtype=torch.int64, device=dev)
    col_ptr[1:] = torch.cumsum(counts, 0)

    if pin:
        rows_h = torch.empty(rows_all.shape, dtype=torch.int32, pin_memory=True)
        rows_h.copy_(rows_all)
        rows_np = rows_h.numpy()
    else:
        rows_h = None
        rows_np = rows_all.cpu().numpy()
    out = SynthDesign(n=n, p=p, k=k, offsets=offsets.cpu().numpy(),
                      event=s_event.cpu().numpy(), tie_end=tie_end.cpu().numpy(),
                      col_ptr=col_ptr.cpu().numpy(), rows=rows_np, true_beta=beta.cpu().numpy(),
                      rows_owner=rows_h)
    del rows_all
    if dev.type == "cuda":
        torch.cuda.synchronize()
    torch.cuda.empty_cache()
    out.gen_seconds = time.perf_counter() - t0
    return out
