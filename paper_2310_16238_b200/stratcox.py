"""Python mirror of the reference ``stratcox`` C++ API for the hot path.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/stratcox/{scan,data,likelihood,optimizer,resample}.hpp;
every call goes through the C-ABI (include/stratcox_b200.h) to the sm_100a
kernels. Exceptions mirror proj/include/stratcox/errors.hpp:9-26 and carry the
reference's exact messages.

Ownership follows the reference: a ``SortedDesign`` is
immutable host data; ``upload`` gives a ``DeviceDesign`` that owns one device
context (design + one device-resident ``CoefficientState``); results are
returned by value.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _capi
from ._capi import ptr


# ---------------------------------------------------------------- errors (errors.hpp:9-26)
class StratcoxError(RuntimeError):
    """stratcox::error"""


class ValidationError(StratcoxError):
    """stratcox::validation_error"""


class NumericError(StratcoxError):
    """stratcox::numeric_error"""


class InternalError(StratcoxError):
    """stratcox::internal_error"""


class CudaError(StratcoxError):
    """device / runtime failure (no reference equivalent)"""


_ERR = {1: ValidationError, 2: NumericError, 3: InternalError, 4: CudaError}


def _lib():
    return _capi.load()


def _check(rc: int, ctx=None, rule: bool = False):
    if rc == 0:
        return
    if rule:
        msg = _lib().scx_rule_error().decode()
    else:
        msg = _lib().scx_last_error(ctx).decode() if ctx is not None else "error"
    raise _ERR.get(rc, StratcoxError)(msg)


def device_count() -> int:
    return int(_lib().scx_device_count())


# ---------------------------------------------------------------- data (data.hpp:50-62)
@dataclass
class SortedDesign:
    """Host view of ``stratcox::SortedDesign`` in sorted row space.

    Rows are sorted stratum-major by decreasing time (stable); column row
    indices refer to sorted rows and are strictly increasing per column.
    ``values`` may be None when every stored value is 1.0.
    """

    stratum_offsets: np.ndarray  # int64 [K+1]
    event: np.ndarray            # uint8 [N]
    tie_group_end: np.ndarray    # int64 [N]
    col_ptr: np.ndarray          # int64 [P+1]
    row_idx: np.ndarray          # int64 or int32 [nnz]
    values: Optional[np.ndarray] = None  # float64 [nnz]
    time: Optional[np.ndarray] = None    # float64 [N] (optional, informational)
    perm: Optional[np.ndarray] = None    # int64 [N] sorted position -> input row
    head_flags: Optional[np.ndarray] = None  # uint8 [N]
    covariate_names: Optional[List[str]] = None

    @property
    def n_rows(self) -> int:
        return int(self.event.shape[0])

    @property
    def n_covariates(self) -> int:
        return int(self.col_ptr.shape[0] - 1)

    @property
    def n_strata(self) -> int:
        return int(self.stratum_offsets.shape[0] - 1)

    @property
    def nnz(self) -> int:
        return int(self.col_ptr[-1])

    def covariate_name(self, j: int) -> str:
        if self.covariate_names and j < len(self.covariate_names) and self.covariate_names[j]:
            return self.covariate_names[j]
        return f"x{j + 1}"


# ---------------------------------------------------------------- scan.hpp:26-29
@dataclass
class ExecutionConfig:
    """Accepted for API compatibility. On the device the bits depend on the
    fixed 4096-row tile configuration only (worker_count is meaningless)."""

    chunk_size: int = 4096
    worker_count: int = 1

    def validate(self):
        if self.chunk_size < 1:
            raise ValidationError("chunk_size must be >= 1")
        if self.worker_count < 1:
            raise ValidationError("worker_count must be >= 1")


# ---------------------------------------------------------------- device design + state
class DeviceDesign:
    """A SortedDesign uploaded to one GPU (owns one scx_ctx)."""

    def __init__(self, design: SortedDesign, device: int = 0, sm_budget: int = 0):
        lib = _lib()
        h = C.c_void_p()
        rc = lib.scx_create(int(device), C.byref(h))
        if rc != 0:
            raise CudaError(f"scx_create(device={device}) failed: no usable sm_100 device")
        if sm_budget:
            lib.scx_set_sm_budget(h, int(sm_budget))
        self._h = h
        self.device = device
        self.design = design
        self._state_owner = None
        off = np.ascontiguousarray(design.stratum_offsets, dtype=np.int64)
        ev = np.ascontiguousarray(design.event, dtype=np.uint8)
        te = np.ascontiguousarray(design.tie_group_end, dtype=np.int64)
        cp = np.ascontiguousarray(design.col_ptr, dtype=np.int64)
        vals = None if design.values is None else np.ascontiguousarray(design.values, dtype=np.float64)
        if design.row_idx.dtype == np.int32:
            rows = np.ascontiguousarray(design.row_idx)
            rc = lib.scx_upload_design_i32(h, design.n_rows, design.n_strata, ptr(off, C.c_int64),
                                           ptr(ev, C.c_uint8), ptr(te, C.c_int64),
                                           design.n_covariates, ptr(cp, C.c_int64),
                                           ptr(rows, C.c_int32), ptr(vals, C.c_double))
        else:
            rows = np.ascontiguousarray(design.row_idx, dtype=np.int64)
            rc = lib.scx_upload_design(h, design.n_rows, design.n_strata, ptr(off, C.c_int64),
                                       ptr(ev, C.c_uint8), ptr(te, C.c_int64),
                                       design.n_covariates, ptr(cp, C.c_int64),
                                       ptr(rows, C.c_int64), ptr(vals, C.c_double))
        if rc != 0:
            msg = lib.scx_last_error(h).decode()
            lib.scx_destroy(h)
            self._h = None
            raise _ERR.get(rc, StratcoxError)(msg)

    # -- housekeeping
    def close(self):
        if getattr(self, "_h", None):
            _lib().scx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def n_rows(self) -> int:
        return self.design.n_rows

    def n_covariates(self) -> int:
        return self.design.n_covariates

    def n_strata(self) -> int:
        return self.design.n_strata

    def info(self) -> dict:
        n = C.c_int64(); k = C.c_int32(); p = C.c_int64(); z = C.c_int64()
        cb = C.c_int32(); nt = C.c_int64(); ni = C.c_int64()
        _check(_lib().scx_design_info(self._h, C.byref(n), C.byref(k), C.byref(p), C.byref(z),
                                      C.byref(cb), C.byref(nt), C.byref(ni)), self._h)
        return dict(n_rows=n.value, n_strata=k.value, p=p.value, nnz=z.value,
                    code_bytes=cb.value, n_tiles=nt.value, n_indicator=ni.value)

    def stream(self) -> int:
        return int(_lib().scx_stream(self._h) or 0)

    def export(self) -> dict:
        """The device's SortedDesign arrays (scx_design_export): stratum
        offsets, event, tie_group_end, col_ptr, row_idx (sorted rows), values."""
        info = self.info()
        n, k, p, nnz = info["n_rows"], info["n_strata"], info["p"], info["nnz"]
        off = np.empty(k + 1, np.int64); ev = np.empty(n, np.uint8)
        te = np.empty(n, np.int64); cp = np.empty(p + 1, np.int64)
        ri = np.empty(max(nnz, 1), np.int64); va = np.empty(max(nnz, 1), np.float64)
        _check(_lib().scx_design_export(self._h, ptr(off, C.c_int64), ptr(ev, C.c_uint8),
                                        ptr(te, C.c_int64), ptr(cp, C.c_int64),
                                        ptr(ri, C.c_int64), ptr(va, C.c_double)), self._h)
        return dict(offsets=off, event=ev, tie_end=te, col_ptr=cp, row_idx=ri[:nnz],
                    values=va[:nnz])

    def set_fit_path(self, path: int) -> bool:
        """CCD cycle implementation: 0 automatic (risk-suffix cycle on the chunked
        layout), 1 per-coordinate fused scan only. Returns whether the
        risk-suffix cycle can run on this design."""
        rs = C.c_int()
        _check(_lib().scx_set_fit_path(self._h, int(path), C.byref(rs)), self._h)
        return bool(rs.value)

    def fit_path_stats(self) -> dict:
        """Counters of the last ccd_fit: risk-suffix cycle launches, coordinates
        handed to the exact fused scan, |eta|-bound hand-offs, fused-scan cycle
        launches."""
        out = (C.c_int64 * 4)()
        _check(_lib().scx_fit_path_stats(self._h, out), self._h)
        return dict(risk_suffix_launches=out[0], exact_handoffs=out[1], bound_handoffs=out[2],
                    fused_scan_launches=out[3])

    # -- state residency (one device-resident CoefficientState per context)
    def _activate(self, state: "CoefficientState"):
        if self._state_owner is state:
            return
        if self._state_owner is not None:
            self._state_owner._snapshot()
        if state._host is not None:
            b, x, e, u = state._host
            _check(_lib().scx_set_state(self._h, ptr(b, C.c_double), ptr(x, C.c_double),
                                        ptr(e, C.c_double), int(u)), self._h)
            state._host = None
        self._state_owner = state


def upload(design: SortedDesign, device: int = 0, sm_budget: int = 0) -> DeviceDesign:
    return DeviceDesign(design, device, sm_budget)


class CoefficientState:
    """stratcox::CoefficientState (likelihood.hpp:23-29), resident on the device."""

    def __init__(self, dd: DeviceDesign):
        self._dd = dd
        self._host = None  # (beta, xbeta, exp_xbeta, updates) when not resident
        self.objective = 0.0

    def _snapshot(self):
        b, x, e, u = self._read()
        self._host = (b, x, e, u)

    def _read(self):
        dd = self._dd
        if self._host is not None:
            return self._host
        p, n = dd.n_covariates(), dd.n_rows()
        b = np.empty(p, np.float64); x = np.empty(n, np.float64); e = np.empty(n, np.float64)
        u = C.c_uint32()
        _check(_lib().scx_get_state(dd.handle, ptr(b, C.c_double), ptr(x, C.c_double),
                                    ptr(e, C.c_double), C.byref(u)), dd.handle)
        return b, x, e, int(u.value)

    @property
    def beta(self) -> np.ndarray:
        return self._read()[0]

    @property
    def xbeta(self) -> np.ndarray:
        return self._read()[1]

    @property
    def exp_xbeta(self) -> np.ndarray:
        return self._read()[2]

    @property
    def updates_since_refresh(self) -> int:
        return self._read()[3]


def make_state(dd: DeviceDesign, beta: Sequence[float]) -> CoefficientState:
    """make_state (likelihood.hpp:33, likelihood.cpp:19-29)."""
    b = np.ascontiguousarray(beta, dtype=np.float64)
    if b.shape[0] != dd.n_covariates():
        raise ValidationError("beta length does not match covariate count")
    st = CoefficientState(dd)
    if dd._state_owner is not None:
        dd._state_owner._snapshot()
    dd._state_owner = st
    _check(_lib().scx_make_state(dd.handle, ptr(b, C.c_double)), dd.handle)
    return st


def state_from_arrays(dd: DeviceDesign, beta, xbeta, exp_xbeta, updates: int = 0) -> CoefficientState:
    """Wrap an arbitrary host CoefficientState (uploaded on first use)."""
    st = CoefficientState(dd)
    st._host = (np.ascontiguousarray(beta, np.float64), np.ascontiguousarray(xbeta, np.float64),
                np.ascontiguousarray(exp_xbeta, np.float64), int(updates))
    return st


def refresh_xbeta(dd: DeviceDesign, state: CoefficientState) -> None:
    """refresh_xbeta (likelihood.hpp:37)."""
    dd._activate(state)
    _check(_lib().scx_refresh_xbeta(dd.handle), dd.handle)


def update_xbeta(dd: DeviceDesign, state: CoefficientState, j: int, delta: float) -> None:
    """update_xbeta (likelihood.hpp:43-44)."""
    dd._activate(state)
    _check(_lib().scx_update_xbeta(dd.handle, int(j), float(delta)), dd.handle)


@dataclass
class GradHess:
    gradient: float = 0.0
    hessian: float = 0.0


def gradient_hessian(dd: DeviceDesign, state: CoefficientState, j: int,
                     workspace=None, config: Optional[ExecutionConfig] = None) -> GradHess:
    """gradient_hessian (likelihood.hpp:75-77): derivatives of the negative log
    partial likelihood w.r.t. beta[j] from one fused device pass."""
    if config is not None:
        config.validate()
    dd._activate(state)
    g = C.c_double(); h = C.c_double()
    _check(_lib().scx_gradient_hessian(dd.handle, int(j), C.byref(g), C.byref(h)), dd.handle)
    return GradHess(g.value, h.value)


def risk_suffix_gradient_hessian(dd: DeviceDesign, state: CoefficientState, j: int) -> GradHess:
    """(g', g'') of coordinate j by the risk-suffix formulation the CCD fit runs
    on the chunked layout (one fused risk scan of the state, then O(nnz_j)
    gathers); equal to gradient_hessian within rounding."""
    dd._activate(state)
    g = C.c_double(); h = C.c_double()
    _check(_lib().scx_gradient_hessian_rs(dd.handle, int(j), C.byref(g), C.byref(h)), dd.handle)
    return GradHess(g.value, h.value)


def log_partial_likelihood(dd: DeviceDesign, state: CoefficientState,
                           config: Optional[ExecutionConfig] = None, workspace=None) -> float:
    """log_partial_likelihood (likelihood.hpp:60-65)."""
    if config is not None:
        config.validate()
    dd._activate(state)
    ll = C.c_double()
    _check(_lib().scx_log_partial_likelihood(dd.handle, C.byref(ll)), dd.handle)
    return ll.value


def naive_gradient_hessian(dd: DeviceDesign, state: CoefficientState, j: int) -> GradHess:
    """naive_gradient_hessian (likelihood.hpp:80-81), literal loops on the device."""
    dd._activate(state)
    g = C.c_double(); h = C.c_double()
    _check(_lib().scx_naive_gradient_hessian(dd.handle, int(j), C.byref(g), C.byref(h)), dd.handle)
    return GradHess(g.value, h.value)


def naive_log_partial_likelihood(dd: DeviceDesign, state: CoefficientState) -> float:
    dd._activate(state)
    ll = C.c_double()
    _check(_lib().scx_naive_log_partial_likelihood(dd.handle, C.byref(ll)), dd.handle)
    return ll.value


_SCAN_CTX = {}


def segmented_inclusive_scan(values, flags, config: Optional[ExecutionConfig] = None,
                             device: int = 0) -> np.ndarray:
    """segmented_inclusive_scan (scan.hpp:71-79) on the device."""
    if config is not None:
        config.validate()
    v = np.ascontiguousarray(values, dtype=np.float64)
    f = np.ascontiguousarray(flags, dtype=np.uint8)
    if v.shape[0] == 0:
        raise ValidationError("empty scan input")
    if f.shape[0] != v.shape[0]:
        raise ValidationError("values and flags must have equal length")
    lib = _lib()
    h = _SCAN_CTX.get(device)
    if h is None:
        h = C.c_void_p()
        if lib.scx_create(int(device), C.byref(h)) != 0:
            raise CudaError("scx_create failed")
        _SCAN_CTX[device] = h
    out = np.empty_like(v)
    _check(lib.scx_segmented_inclusive_scan(h, v.shape[0], ptr(v, C.c_double), ptr(f, C.c_uint8),
                                            ptr(out, C.c_double)), h)
    return out


# ---------------------------------------------------------------- optimizer.hpp
kFlatCurvature = 1e-12
kLinearPredictorBound = 700.0


def newton_step(g1: float, g2: float):
    """newton_step (optimizer.hpp:50) -> (step, flat)."""
    s = C.c_double(); fl = C.c_int()
    _check(_lib().scx_newton_step(float(g1), float(g2), C.byref(s), C.byref(fl)), rule=True)
    return s.value, bool(fl.value)


@dataclass
class TrustOutcome:
    applied: float
    next_trust: float


def apply_trust_region(delta_proposed: float, trust: float) -> TrustOutcome:
    a = C.c_double(); n = C.c_double()
    _check(_lib().scx_apply_trust_region(float(delta_proposed), float(trust), C.byref(a),
                                         C.byref(n)), rule=True)
    return TrustOutcome(a.value, n.value)


@dataclass
class ProposedStep:
    step: float = 0.0
    skipped: bool = False
    flat: bool = False


def l1_coordinate_update(g1: float, g2: float, beta_j: float, gamma_j: float) -> ProposedStep:
    s = C.c_double(); sk = C.c_int(); fl = C.c_int()
    _check(_lib().scx_l1_coordinate_update(float(g1), float(g2), float(beta_j), float(gamma_j),
                                           C.byref(s), C.byref(sk), C.byref(fl)), rule=True)
    return ProposedStep(s.value, bool(sk.value), bool(fl.value))


def coordinate_update(g1: float, g2: float, beta_j: float, gamma_j: float,
                      l2_j: float) -> ProposedStep:
    """Elastic-net rule (extension; no reference counterpart): ridge term
    l2_j*beta_j^2/2 folded into (g', g''), then l1_coordinate_update."""
    s = C.c_double(); sk = C.c_int(); fl = C.c_int()
    _check(_lib().scx_coordinate_update(float(g1), float(g2), float(beta_j), float(gamma_j),
                                        float(l2_j), C.byref(s), C.byref(sk), C.byref(fl)),
           rule=True)
    return ProposedStep(s.value, bool(sk.value), bool(fl.value))


@dataclass
class PenaltySpec:
    """PenaltySpec (optimizer.hpp:18-28): per-coefficient L1 weight, 0 = unpenalized.

    ``l2`` (extension, not in the reference): optional per-coefficient L2
    (ridge / Gaussian) prior weight; the objective adds sum l2_j beta_j^2 / 2.
    BASELINE config 1's "L2 prior" is ``PenaltySpec.ridge(p, lam)``."""

    gamma: np.ndarray
    l2: Optional[np.ndarray] = None

    @staticmethod
    def ridge(p: int, l2_value: float, gamma_value: float = 0.0) -> "PenaltySpec":
        return PenaltySpec(np.full(p, float(gamma_value), np.float64),
                           np.full(p, float(l2_value), np.float64))

    @staticmethod
    def none(p: int) -> "PenaltySpec":
        return PenaltySpec(np.zeros(p, np.float64))

    @staticmethod
    def shared(p: int, gamma_value: float, unpenalized: Sequence[int] = ()) -> "PenaltySpec":
        g = np.full(p, float(gamma_value), np.float64)
        for j in unpenalized:
            if j >= p:
                raise ValidationError("unpenalized index out of range")
            g[j] = 0.0
        return PenaltySpec(g)

    def value(self, beta) -> float:
        total = 0.0
        for gj, bj in zip(self.gamma, beta):
            total += gj * abs(bj)
        if self.l2 is not None:
            for lj, bj in zip(self.l2, beta):
                total += 0.5 * lj * bj * bj
        return total

    def validate(self, p: int):
        if len(self.gamma) != p:
            raise ValidationError("penalty length does not match covariate count")
        g = np.asarray(self.gamma, np.float64)
        if not np.all(np.isfinite(g)) or np.any(g < 0.0):
            raise ValidationError("penalty weights must be finite and non-negative")
        if self.l2 is not None:
            lam = np.asarray(self.l2, np.float64)
            if lam.shape != (p,):
                raise ValidationError("L2 prior length does not match covariate count")
            if not np.all(np.isfinite(lam)) or np.any(lam < 0.0):
                raise ValidationError("L2 prior weights must be finite and non-negative")


@dataclass
class OptimizerConfig:
    max_cycles: int = 1000
    tolerance: float = 1e-6
    initial_trust: float = 1.0
    exec: ExecutionConfig = field(default_factory=ExecutionConfig)


@dataclass
class FitResult:
    beta: np.ndarray
    objective_trace: List[float]
    cycles_used: int
    converged: bool
    trust: np.ndarray
    warnings: List[str]
    n_evaluations: int = 0
    updates_since_refresh: int = 0


def ccd_fit(dd: DeviceDesign, penalty: PenaltySpec, config: Optional[OptimizerConfig] = None,
            initial_beta=None) -> FitResult:
    """ccd_fit (optimizer.hpp:70-73). The whole CCD cycle runs on the device;
    the host synchronises once per cycle."""
    config = config or OptimizerConfig()
    p = dd.n_covariates()
    penalty.validate(p)
    if initial_beta is not None:
        ib = np.ascontiguousarray(initial_beta, dtype=np.float64)
        if ib.shape[0] != p:
            raise ValidationError("initial beta length does not match covariate count")
    else:
        ib = None
    gamma = np.ascontiguousarray(penalty.gamma, dtype=np.float64)
    beta = np.zeros(p, np.float64)
    trust = np.zeros(p, np.float64)
    trace = np.zeros(max(1, config.max_cycles) + 1, np.float64)
    wcap = 1 << 16  # kWarnCap: the library records this many; n_warnings is exact
    wc = np.zeros(wcap, np.int64)
    res = _capi.FitResultC(ptr(beta, C.c_double), ptr(trust, C.c_double), ptr(trace, C.c_double),
                           0, 0, 0, 0, ptr(wc, C.c_int64), wcap, 0, 0)
    opt = _capi.FitOptions(int(config.max_cycles), float(config.tolerance),
                           float(config.initial_trust))
    # the fit replaces the context's device state
    if dd._state_owner is not None:
        dd._state_owner._snapshot()
        dd._state_owner = None
    lam = None if penalty.l2 is None else np.ascontiguousarray(penalty.l2, dtype=np.float64)
    _check(_lib().scx_ccd_fit_prior(dd.handle, ptr(gamma, C.c_double), ptr(lam, C.c_double),
                                    C.byref(opt), ptr(ib, C.c_double), C.byref(res)), dd.handle)
    warnings = [f"coordinate {dd.design.covariate_name(int(j))} skipped: step overflow persisted "
                f"after 10 halvings" for j in wc[:min(res.n_warnings, wcap)]]
    if res.n_warnings > wcap:
        warnings.append(f"... {res.n_warnings - wcap} more step-overflow warnings not recorded")
    return FitResult(beta=beta, objective_trace=list(trace[:res.trace_len]),
                     cycles_used=int(res.cycles_used), converged=bool(res.converged),
                     trust=trust, warnings=warnings, n_evaluations=int(res.n_evaluations),
                     updates_since_refresh=int(res.updates_since_refresh))


def gamma_max(dd: DeviceDesign, penalty_template: Optional[PenaltySpec] = None) -> float:
    """gamma_max (resample.hpp:38-39): largest |gradient| at beta = 0 over
    penalized coordinates."""
    g = None
    if penalty_template is not None:
        penalty_template.validate(dd.n_covariates())
        g = np.ascontiguousarray(penalty_template.gamma, dtype=np.float64)
    out = C.c_double()
    if dd._state_owner is not None:
        dd._state_owner._snapshot()
        dd._state_owner = None
    _check(_lib().scx_gamma_max(dd.handle, ptr(g, C.c_double), C.byref(out)), dd.handle)
    return out.value


def default_gamma_grid(gamma_max_value: float, size: int = 20) -> np.ndarray:
    """default_gamma_grid (resample.cpp:57-68): log-spaced [gmax/1e4, gmax]."""
    if size < 1:
        raise ValidationError("gamma grid size must be >= 1")
    if not gamma_max_value > 0.0:
        raise ValidationError("gamma_max must be positive")
    import math
    hi = math.log(gamma_max_value)
    lo = hi - math.log(1e4)
    out = np.empty(size, np.float64)
    for i in range(size):
        t = 1.0 if size == 1 else i / (size - 1)
        out[i] = math.exp(lo + t * (hi - lo))
    return out


# ---------------------------------------------------------------- data sets, path and CV
@dataclass
class SurvivalDataset:
    """SurvivalDataset (data.hpp:31-45) in input row order, CSC columns."""
    time: np.ndarray
    event: np.ndarray
    stratum: np.ndarray
    col_ptr: np.ndarray
    row_idx: np.ndarray
    values: Optional[np.ndarray] = None
    subject: Optional[np.ndarray] = None

    def n_rows(self) -> int:
        return int(self.time.shape[0])

    def n_covariates(self) -> int:
        return int(self.col_ptr.shape[0] - 1)

    def _c(self):
        keep = dict(time=np.ascontiguousarray(self.time, np.float64),
                    event=np.ascontiguousarray(self.event, np.uint8),
                    stratum=np.ascontiguousarray(self.stratum, np.int32),
                    col_ptr=np.ascontiguousarray(self.col_ptr, np.int64),
                    row_idx=np.ascontiguousarray(self.row_idx, np.int64),
                    values=None if self.values is None else np.ascontiguousarray(self.values, np.float64),
                    subject=None if self.subject is None else np.ascontiguousarray(self.subject, np.int64))
        ds = _capi.DatasetC(self.n_rows(), ptr(keep["time"], C.c_double), ptr(keep["event"], C.c_uint8),
                            ptr(keep["stratum"], C.c_int32), ptr(keep["subject"], C.c_int64),
                            self.n_covariates(), ptr(keep["col_ptr"], C.c_int64),
                            ptr(keep["row_idx"], C.c_int64), ptr(keep["values"], C.c_double))
        return ds, keep


class _BuiltDesign:
    """Shape of a design sorted and uploaded by the library (scx_build_design)."""

    def __init__(self, n, k, p):
        self.n_rows, self.n_strata, self.n_covariates = n, k, p

    @staticmethod
    def covariate_name(j: int) -> str:
        return f"x{j + 1}"


def build_design(data: SurvivalDataset, device: int = 0):
    """build_sorted_design (data.hpp:66, data.cpp:68-147) + upload: returns
    (DeviceDesign, perm) with perm[s] = input row of sorted row s."""
    lib = _lib()
    h = C.c_void_p()
    if lib.scx_create(int(device), C.byref(h)) != 0:
        raise CudaError(f"scx_create(device={device}) failed: no usable sm_100 device")
    ds, keep = data._c()
    perm = np.empty(data.n_rows(), np.int64)
    rc = lib.scx_build_design(h, C.byref(ds), ptr(perm, C.c_int64))
    if rc != 0:
        msg = lib.scx_last_error(h).decode()
        lib.scx_destroy(h)
        raise _ERR.get(rc, StratcoxError)(msg)
    dd = DeviceDesign.__new__(DeviceDesign)
    dd._h, dd.device, dd._state_owner = h, device, None
    info = dd.info()
    dd.design = _BuiltDesign(info["n_rows"], info["n_strata"], info["p"])
    return dd, perm


def build_lowered_design(subjects: SurvivalDataset, cut_points, splits=None, device: int = 0):
    """Device lowering + build (scx_build_lowered_design): only the subject-level
    data is uploaded; augment_to_strata / split_time_varying_coefficient and
    build_sorted_design run on the GPU. Returns (DeviceDesign, perm,
    [ColumnMapEntry]) — the design lower_time_varying + build_design give."""
    lib = _lib()
    splits = splits or {}
    cov = np.array(sorted(splits), np.int64)
    sptr = np.zeros(len(cov) + 1, np.int64)
    times: List[float] = []
    for q, j in enumerate(cov):
        times += [float(t) for t in splits[int(j)]]
        sptr[q + 1] = len(times)
    tm = np.array(times, np.float64)
    cuts = np.ascontiguousarray(cut_points, np.float64)
    pout = subjects.n_covariates() + len(times)
    src = np.empty(max(pout, 1), np.int64); win = np.empty(max(pout, 1), np.int32)
    ws = np.empty(max(pout, 1)); we = np.empty(max(pout, 1))
    h = C.c_void_p()
    if lib.scx_create(int(device), C.byref(h)) != 0:
        raise CudaError(f"scx_create(device={device}) failed: no usable sm_100 device")
    ds, keep = subjects._c()
    rc = lib.scx_build_lowered_design(h, C.byref(ds), ptr(cuts, C.c_double), cuts.shape[0],
                                      ptr(cov, C.c_int64), ptr(sptr, C.c_int64),
                                      ptr(tm, C.c_double), len(cov), None, ptr(src, C.c_int64),
                                      win.ctypes.data_as(C.POINTER(C.c_int32)),
                                      ptr(ws, C.c_double), ptr(we, C.c_double))
    if rc != 0:
        msg = lib.scx_last_error(h).decode()
        lib.scx_destroy(h)
        raise _ERR.get(rc, StratcoxError)(msg)
    dd = DeviceDesign.__new__(DeviceDesign)
    dd._h, dd.device, dd._state_owner = h, device, None
    info = dd.info()
    dd.design = _BuiltDesign(info["n_rows"], info["n_strata"], info["p"])
    cmap = [ColumnMapEntry(c, int(src[c]), int(win[c]), float(ws[c]), float(we[c]))
            for c in range(pout)]
    return dd, cmap


def fold_assignment(data: SurvivalDataset, folds: int, seed: int) -> np.ndarray:
    """fold_assignment (resample.hpp:45, resample.cpp:70-91)."""
    ds, keep = data._c()
    out = np.empty(data.n_rows(), np.int32)
    rc = _lib().scx_fold_assignment(C.byref(ds), int(folds), int(seed), ptr(out, C.c_int32))
    if rc:
        raise _ERR.get(rc, StratcoxError)(
            "folds must be >= 2" if folds < 2 else "degenerate fold; reduce folds or reseed")
    return out


@dataclass
class CvResult:
    """CvResult (resample.hpp:21-27)."""
    gamma_star: float
    grid: np.ndarray
    fold_scores: np.ndarray   # [grid index][fold]
    mean_scores: np.ndarray   # [grid index]
    warnings: List[str]


def kfold_select_gamma(data: SurvivalDataset, penalty_template: PenaltySpec, folds: int,
                       gamma_grid, seed: int = 1, config: Optional[OptimizerConfig] = None,
                       devices: Sequence[int] = (0,)) -> CvResult:
    """kfold_select_gamma (resample.hpp:53-54): warm-started gamma path per fold
    on the device(s), held-out stratified partial-likelihood scoring; folds are
    dealt round-robin over ``devices``."""
    config = config or OptimizerConfig()
    grid = np.ascontiguousarray(gamma_grid, np.float64)
    tmpl = np.ascontiguousarray(penalty_template.gamma, np.float64)
    ds, keep = data._c()
    cv = _capi.CvConfigC(int(folds), ptr(grid, C.c_double), grid.shape[0], int(seed))
    opt = _capi.FitOptions(int(config.max_cycles), float(config.tolerance),
                           float(config.initial_trust))
    fs = np.zeros((grid.shape[0], max(1, folds)), np.float64)
    ms = np.zeros(grid.shape[0], np.float64)
    res = _capi.CvResultC(0.0, ptr(fs, C.c_double), ptr(ms, C.c_double), 0)
    devs = (C.c_int * len(devices))(*devices)
    msg = C.create_string_buffer(1 << 16)
    rc = _lib().scx_kfold_select_gamma(C.byref(ds), ptr(tmpl, C.c_double), C.byref(cv),
                                       C.byref(opt), devs, len(devices), C.byref(res), msg,
                                       len(msg))
    text = msg.value.decode()
    if rc:
        raise _ERR.get(rc, StratcoxError)(text)
    return CvResult(gamma_star=res.gamma_star, grid=grid.copy(), fold_scores=fs, mean_scores=ms,
                    warnings=[w for w in text.split("\n") if w])


# ---------------------------------------------------------------- lowering (transforms.hpp)
@dataclass
class ColumnMapEntry:
    """ColumnMapEntry (transforms.hpp:52-60): window -1 = never split."""
    column: int
    source: int
    window: int
    window_start: float
    window_end: float


def lower_time_varying(subjects: SurvivalDataset, cut_points, splits=None):
    """make_time_varying (time-fixed covariates) + split_time_varying_coefficient +
    augment_to_strata (transforms.hpp:85-104, lower_pipeline): one row per
    (subject, interval at risk), interval-major, stratum = interval. ``splits``
    maps a covariate index to its effect-window boundaries (cut points).
    Returns (SurvivalDataset, [ColumnMapEntry])."""
    lib = _lib()
    splits = splits or {}
    cov = np.array(sorted(splits), np.int64)
    sptr = np.zeros(len(cov) + 1, np.int64)
    times = []
    for q, j in enumerate(cov):
        times += [float(t) for t in splits[int(j)]]
        sptr[q + 1] = len(times)
    tm = np.array(times, np.float64)
    cuts = np.ascontiguousarray(cut_points, np.float64)
    ds, keep = subjects._c()
    h = C.c_void_p()
    msg = C.create_string_buffer(4096)
    rc = lib.scx_lower_time_varying(C.byref(ds), ptr(cuts, C.c_double), cuts.shape[0],
                                    ptr(cov, C.c_int64), ptr(sptr, C.c_int64), ptr(tm, C.c_double),
                                    len(cov), C.byref(h), msg, len(msg))
    if rc:
        raise _ERR.get(rc, StratcoxError)(msg.value.decode())
    try:
        n = C.c_int64(); p = C.c_int64(); z = C.c_int64()
        lib.scx_lowered_sizes(h, C.byref(n), C.byref(p), C.byref(z))
        n, p, z = n.value, p.value, z.value
        v = _capi.DatasetC()
        lib.scx_lowered_dataset(h, C.byref(v))
        arr = lambda pt, cnt, dt: np.ctypeslib.as_array(pt, shape=(max(cnt, 1),))[:cnt].astype(dt, copy=True)
        out = SurvivalDataset(time=arr(v.time, n, np.float64), event=arr(v.event, n, np.uint8),
                              stratum=arr(v.stratum, n, np.int32), col_ptr=arr(v.col_ptr, p + 1, np.int64),
                              row_idx=arr(v.row_idx, z, np.int64), values=arr(v.values, z, np.float64),
                              subject=arr(v.subject, n, np.int64))
        src = np.empty(p, np.int64); win = np.empty(p, np.int32)
        ws = np.empty(p); we = np.empty(p)
        lib.scx_lowered_column_map(h, ptr(src, C.c_int64), win.ctypes.data_as(C.POINTER(C.c_int32)),
                                   ptr(ws, C.c_double), ptr(we, C.c_double))
        cmap = [ColumnMapEntry(c, int(src[c]), int(win[c]), float(ws[c]), float(we[c])) for c in range(p)]
        return out, cmap
    finally:
        lib.scx_lowered_free(h)
