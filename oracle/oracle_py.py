"""TEST INFRASTRUCTURE ONLY — ctypes access to the two CPU checkers.

* ``Ref``    : the UNMODIFIED reference library compiled in place
               (oracle/_ref/libstratcox_ref.so, see oracle/Makefile and
               oracle/ref_capi.cpp).
* ``Oracle`` : the plain-C restatement (oracle/liboracle.so,
               oracle/stratcox_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arm may import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PATH = os.path.join(HERE, "_ref", "libstratcox_ref.so")
ORACLE_PATH = os.path.join(HERE, "liboracle.so")

_u8 = C.POINTER(C.c_uint8)
_i32 = C.POINTER(C.c_int32)
_i64 = C.POINTER(C.c_int64)
_u32 = C.POINTER(C.c_uint32)
_d = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_vp = C.c_void_p


def _p(a, t):
    return None if a is None else a.ctypes.data_as(C.POINTER(t))


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


@dataclass
class Dataset:
    """Input-order survival data (SurvivalDataset, data.hpp:30-45)."""

    time: np.ndarray
    event: np.ndarray
    stratum: np.ndarray
    col_ptr: np.ndarray
    row_idx: np.ndarray
    values: np.ndarray
    true_beta: Optional[np.ndarray] = None

    @property
    def n(self):
        return int(self.time.shape[0])

    @property
    def p(self):
        return int(self.col_ptr.shape[0] - 1)


def to_sorted_design(arrs: dict):
    from paper_2310_16238_b200.stratcox import SortedDesign

    return SortedDesign(stratum_offsets=arrs["offsets"], event=arrs["event"],
                        tie_group_end=arrs["tie_end"], col_ptr=arrs["col_ptr"],
                        row_idx=arrs["row_idx"], values=arrs["values"], time=arrs["time"],
                        perm=arrs["perm"], head_flags=arrs["head"])


class Ref:
    """The compiled reference (stratcox C++), through oracle/ref_capi.cpp."""

    def __init__(self, path: str = REF_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_max_threads": (C.c_int, []),
            "ref_simulate": (C.c_int, [C.c_int64, C.c_int64, C.c_double, C.c_double, C.c_int32,
                                       C.c_double, C.c_uint64, C.POINTER(_vp)]),
            "ref_random_dataset": (C.c_int, [C.c_uint64, C.c_int64, C.c_int32, C.c_int64,
                                             C.c_double, C.c_double, C.POINTER(_vp)]),
            "ref_dataset_from_arrays": (C.c_int, [C.c_int64, _d, _u8, _i32, C.c_int64, _i64, _i64,
                                                  _d, C.POINTER(_vp)]),
            "ref_dataset_sizes": (None, [_vp, _i64, _i64, _i64]),
            "ref_dataset_copy": (None, [_vp, _d, _u8, _i32, _i64, _i64, _d, _d]),
            "ref_dataset_free": (None, [_vp]),
            "ref_design_build": (C.c_int, [_vp, C.POINTER(_vp)]),
            "ref_design_sizes": (None, [_vp, _i64, _i64, _i32, _i64]),
            "ref_design_copy": (None, [_vp, _i64, _u8, _i64, _i64, _d, _u8, _i32, _i64, _i64, _d]),
            "ref_design_free": (None, [_vp]),
            "ref_make_state": (C.c_int, [_vp, _d, _d, _d]),
            "ref_gradient_hessian": (C.c_int, [_vp, _d, _d, _d, C.c_int64, C.c_int64, C.c_int,
                                               _d, _d]),
            "ref_naive_gradient_hessian": (C.c_int, [_vp, _d, _d, _d, C.c_int64, _d, _d]),
            "ref_log_partial_likelihood": (C.c_int, [_vp, _d, _d, _d, C.c_int64, C.c_int, _d]),
            "ref_naive_log_partial_likelihood": (C.c_int, [_vp, _d, _d, _d, _d]),
            "ref_update_xbeta": (C.c_int, [_vp, _d, _d, _d, _u32, C.c_int64, C.c_double]),
            "ref_segmented_scan": (C.c_int, [C.c_int64, _d, _u8, C.c_int64, C.c_int, _d]),
            "ref_ccd_fit": (C.c_int, [_vp, _d, C.c_int, C.c_double, C.c_double, C.c_int64, C.c_int,
                                      _d, _d, _d, C.c_int, _ip, _ip, _ip, _d, _ip]),
            "ref_gamma_max": (C.c_int, [_vp, C.c_int64, C.c_int, _d]),
            "ref_default_gamma_grid": (C.c_int, [C.c_double, C.c_int64, _d]),
            "ref_time_iterations": (C.c_int, [_vp, C.c_double, C.c_int, C.c_int, C.c_int, _d]),
            "ref_time_fit": (C.c_int, [_vp, C.c_double, C.c_int, C.c_double, C.c_int, _d, _ip]),
            "ref_dataset_subject": (None, [_vp, _i64]),
            "ref_dataset_set_subject": (None, [_vp, _i64]),
            "ref_fold_assignment": (C.c_int, [_vp, C.c_int, C.c_uint64, _i32]),
            "ref_lower_pipeline": (C.c_int, [_vp, _d, C.c_int64, _i64, _i64, _d, C.c_int64,
                                             C.POINTER(_vp), _i64, _i32]),
            "ref_kfold_select_gamma": (C.c_int, [_vp, _d, C.c_int, _d, C.c_int64, C.c_uint64,
                                                 C.c_int, C.c_double, C.c_double, C.c_int, _d,
                                                 _d, _d, _ip]),
            "ref_read_wide_csv": (C.c_int, [C.c_char_p, C.POINTER(_vp)]),
            "ref_dataset_name": (C.c_char_p, [_vp, C.c_int64]),
            "ref_dataset_n_labels": (C.c_int32, [_vp]),
            "ref_dataset_label": (C.c_char_p, [_vp, C.c_int32]),
            "ref_write_wide_csv": (C.c_int, [_vp, C.c_char_p]),
            "ref_read_long_csv": (C.c_int, [C.c_char_p, C.POINTER(_vp)]),
            "ref_long_sizes": (None, [_vp, _i64, _i64, _i64, _d]),
            "ref_long_name": (C.c_char_p, [_vp, C.c_int64]),
            "ref_write_long_csv": (C.c_int, [_vp, C.c_char_p]),
            "ref_long_free": (None, [_vp]),
            "ref_long_lower": (C.c_int, [_vp, _d, C.c_int64, _i64, _i64, _d, C.c_int64,
                                         C.POINTER(_vp), _i64, _i32]),
            "ref_config_script": (C.c_int, [C.c_char_p, C.c_char_p, C.c_char_p, C.c_char_p,
                                            C.c_int]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        self.L = L

    def _chk(self, rc):
        if rc:
            raise OracleError(rc, self.L.ref_last_error().decode())

    # ---- datasets
    def _dataset(self, h) -> Dataset:
        n = C.c_int64(); p = C.c_int64(); z = C.c_int64()
        self.L.ref_dataset_sizes(h, C.byref(n), C.byref(p), C.byref(z))
        n, p, z = n.value, p.value, z.value
        t = np.empty(n); e = np.empty(n, np.uint8); s = np.empty(n, np.int32)
        cp = np.empty(p + 1, np.int64); r = np.empty(max(z, 1), np.int64)
        v = np.empty(max(z, 1)); tb = np.zeros(p)
        self.L.ref_dataset_copy(h, _p(t, C.c_double), _p(e, C.c_uint8), _p(s, C.c_int32),
                                _p(cp, C.c_int64), _p(r, C.c_int64), _p(v, C.c_double),
                                _p(tb, C.c_double))
        return Dataset(t, e, s, cp, r[:z], v[:z], tb)

    def simulate(self, n, p, density=0.05, beta_sparsity=0.8, strata=1, censoring=0.3, seed=0,
                 keep_handle=False):
        h = _vp()
        self._chk(self.L.ref_simulate(n, p, density, beta_sparsity, strata, censoring, seed,
                                      C.byref(h)))
        ds = self._dataset(h)
        if keep_handle:
            return ds, h
        self.L.ref_dataset_free(h)
        return ds

    def random_dataset(self, seed, n, strata, p, density=0.4, time_grid=8.0) -> Dataset:
        """oracles::random_dataset (proj/tests/oracles.hpp:58-85) with a fresh
        mt19937_64(seed)."""
        h = _vp()
        self._chk(self.L.ref_random_dataset(seed, n, strata, p, density, time_grid, C.byref(h)))
        ds = self._dataset(h)
        self.L.ref_dataset_free(h)
        return ds

    def dataset_handle(self, ds: Dataset):
        h = _vp()
        vals = np.ascontiguousarray(ds.values, np.float64)
        self._chk(self.L.ref_dataset_from_arrays(
            ds.n, _p(np.ascontiguousarray(ds.time, np.float64), C.c_double),
            _p(np.ascontiguousarray(ds.event, np.uint8), C.c_uint8),
            _p(np.ascontiguousarray(ds.stratum, np.int32), C.c_int32), ds.p,
            _p(np.ascontiguousarray(ds.col_ptr, np.int64), C.c_int64),
            _p(np.ascontiguousarray(ds.row_idx, np.int64), C.c_int64), _p(vals, C.c_double),
            C.byref(h)))
        return h

    # ---- design
    def build_design(self, ds: Dataset):
        """Returns (handle, arrays dict) of build_sorted_design."""
        dh = self.dataset_handle(ds)
        h = _vp()
        rc = self.L.ref_design_build(dh, C.byref(h))
        self.L.ref_dataset_free(dh)
        self._chk(rc)
        return h, self.design_arrays(h)

    def design_arrays(self, h) -> dict:
        n = C.c_int64(); p = C.c_int64(); k = C.c_int32(); z = C.c_int64()
        self.L.ref_design_sizes(h, C.byref(n), C.byref(p), C.byref(k), C.byref(z))
        n, p, k, z = n.value, p.value, k.value, z.value
        a = dict(perm=np.empty(n, np.int64), head=np.empty(n, np.uint8),
                 tie_end=np.empty(n, np.int64), offsets=np.empty(k + 1, np.int64),
                 time=np.empty(n), event=np.empty(n, np.uint8), stratum=np.empty(n, np.int32),
                 col_ptr=np.empty(p + 1, np.int64), row_idx=np.empty(max(z, 1), np.int64),
                 values=np.empty(max(z, 1)))
        self.L.ref_design_copy(h, _p(a["perm"], C.c_int64), _p(a["head"], C.c_uint8),
                               _p(a["tie_end"], C.c_int64), _p(a["offsets"], C.c_int64),
                               _p(a["time"], C.c_double), _p(a["event"], C.c_uint8),
                               _p(a["stratum"], C.c_int32), _p(a["col_ptr"], C.c_int64),
                               _p(a["row_idx"], C.c_int64), _p(a["values"], C.c_double))
        a["row_idx"] = a["row_idx"][:z]
        a["values"] = a["values"][:z]
        a["n"], a["p"], a["k"] = n, p, k
        return a

    def free_design(self, h):
        self.L.ref_design_free(h)

    # ---- likelihood
    def make_state(self, h, beta, n):
        x = np.empty(n); e = np.empty(n)
        b = np.ascontiguousarray(beta, np.float64)
        self._chk(self.L.ref_make_state(h, _p(b, C.c_double), _p(x, C.c_double),
                                        _p(e, C.c_double)))
        return x, e

    def gradient_hessian(self, h, beta, xb, ex, j, chunk=4096, workers=1):
        g = C.c_double(); hh = C.c_double()
        self._chk(self.L.ref_gradient_hessian(h, _p(beta, C.c_double), _p(xb, C.c_double),
                                              _p(ex, C.c_double), j, chunk, workers, C.byref(g),
                                              C.byref(hh)))
        return g.value, hh.value

    def naive_gradient_hessian(self, h, beta, xb, ex, j):
        g = C.c_double(); hh = C.c_double()
        self._chk(self.L.ref_naive_gradient_hessian(h, _p(beta, C.c_double), _p(xb, C.c_double),
                                                    _p(ex, C.c_double), j, C.byref(g),
                                                    C.byref(hh)))
        return g.value, hh.value

    def log_partial_likelihood(self, h, beta, xb, ex, chunk=4096, workers=1):
        ll = C.c_double()
        self._chk(self.L.ref_log_partial_likelihood(h, _p(beta, C.c_double), _p(xb, C.c_double),
                                                    _p(ex, C.c_double), chunk, workers,
                                                    C.byref(ll)))
        return ll.value

    def naive_log_partial_likelihood(self, h, beta, xb, ex):
        ll = C.c_double()
        self._chk(self.L.ref_naive_log_partial_likelihood(h, _p(beta, C.c_double),
                                                          _p(xb, C.c_double), _p(ex, C.c_double),
                                                          C.byref(ll)))
        return ll.value

    def update_xbeta(self, h, beta, xb, ex, updates, j, delta):
        u = C.c_uint32(updates)
        self._chk(self.L.ref_update_xbeta(h, _p(beta, C.c_double), _p(xb, C.c_double),
                                          _p(ex, C.c_double), C.byref(u), j, delta))
        return u.value

    def segmented_scan(self, values, flags, chunk=4096, workers=1):
        v = np.ascontiguousarray(values, np.float64)
        f = np.ascontiguousarray(flags, np.uint8)
        out = np.empty_like(v)
        self._chk(self.L.ref_segmented_scan(v.shape[0], _p(v, C.c_double), _p(f, C.c_uint8),
                                            chunk, workers, _p(out, C.c_double)))
        return out

    def ccd_fit(self, h, gamma, p, max_cycles=1000, tol=1e-6, initial_trust=1.0, chunk=4096,
                workers=1, initial_beta=None):
        beta = np.empty(p); trace = np.empty(max_cycles + 1); trust = np.empty(p)
        tl = C.c_int(); cy = C.c_int(); cv = C.c_int(); nw = C.c_int()
        g = np.ascontiguousarray(gamma, np.float64)
        ib = None if initial_beta is None else np.ascontiguousarray(initial_beta, np.float64)
        self._chk(self.L.ref_ccd_fit(h, _p(g, C.c_double), max_cycles, tol, initial_trust, chunk,
                                     workers, _p(ib, C.c_double), _p(beta, C.c_double),
                                     _p(trace, C.c_double), max_cycles + 1, C.byref(tl),
                                     C.byref(cy), C.byref(cv), _p(trust, C.c_double),
                                     C.byref(nw)))
        return dict(beta=beta, trace=trace[:tl.value].copy(), cycles=cy.value,
                    converged=bool(cv.value), trust=trust, n_warnings=nw.value)

    def gamma_max(self, h, chunk=4096, workers=1):
        out = C.c_double()
        self._chk(self.L.ref_gamma_max(h, chunk, workers, C.byref(out)))
        return out.value

    def default_gamma_grid(self, gmax, size=20):
        out = np.empty(size)
        self._chk(self.L.ref_default_gamma_grid(gmax, size, _p(out, C.c_double)))
        return out

    def time_iterations(self, h, gamma, reps, sweep, workers):
        out = np.empty(reps)
        self._chk(self.L.ref_time_iterations(h, gamma, reps, sweep, workers,
                                             _p(out, C.c_double)))
        return out

    def time_fit(self, h, gamma, max_cycles, tol, workers):
        s = C.c_double(); cy = C.c_int()
        self._chk(self.L.ref_time_fit(h, gamma, max_cycles, tol, workers, C.byref(s),
                                      C.byref(cy)))
        return s.value, cy.value

    def max_threads(self):
        return self.L.ref_max_threads()


def _ref_resample_methods():
    def fold_assignment(self, ds, folds, seed, subject=None):
        """fold_assignment (resample.cpp:70-91) of the reference."""
        h = self.dataset_handle(ds)
        try:
            if subject is not None:
                sj = np.ascontiguousarray(subject, np.int64)
                self.L.ref_dataset_set_subject(h, _p(sj, C.c_int64))
            out = np.empty(ds.n, np.int32)
            self._chk(self.L.ref_fold_assignment(h, int(folds), int(seed), _p(out, C.c_int32)))
            return out
        finally:
            self.L.ref_dataset_free(h)

    def kfold_select_gamma(self, ds, template, folds, grid, seed, max_cycles=1000, tol=1e-6,
                           initial_trust=1.0, workers=0, subject=None):
        """kfold_select_gamma (resample.cpp:93-172) of the reference."""
        h = self.dataset_handle(ds)
        try:
            if subject is not None:
                sj = np.ascontiguousarray(subject, np.int64)
                self.L.ref_dataset_set_subject(h, _p(sj, C.c_int64))
            g = np.ascontiguousarray(grid, np.float64)
            t = np.ascontiguousarray(template, np.float64)
            fs = np.empty((g.shape[0], folds)); ms = np.empty(g.shape[0])
            gs = C.c_double(); nw = C.c_int()
            self._chk(self.L.ref_kfold_select_gamma(
                h, _p(t, C.c_double), int(folds), _p(g, C.c_double), g.shape[0], int(seed),
                int(max_cycles), float(tol), float(initial_trust), int(workers),
                _p(fs, C.c_double), _p(ms, C.c_double), C.byref(gs), C.byref(nw)))
            return dict(gamma_star=gs.value, fold_scores=fs, mean_scores=ms, n_warnings=nw.value)
        finally:
            self.L.ref_dataset_free(h)

    # ---- io (proj/src/io.cpp)
    def read_wide_csv(self, path):
        """(Dataset, subjects, covariate names, stratum labels) of read_wide_csv."""
        h = _vp()
        self._chk(self.L.ref_read_wide_csv(str(path).encode(), C.byref(h)))
        try:
            ds = self._dataset(h)
            subj = np.empty(ds.n, np.int64)
            self.L.ref_dataset_subject(h, _p(subj, C.c_int64))
            names = [self.L.ref_dataset_name(h, j).decode() for j in range(ds.p)]
            labels = [self.L.ref_dataset_label(h, k).decode()
                      for k in range(1, self.L.ref_dataset_n_labels(h) + 1)]
            return ds, subj, names, labels
        finally:
            self.L.ref_dataset_free(h)

    def wide_roundtrip(self, path_in, path_out):
        """read_wide_csv + write_wide_csv of the reference."""
        h = _vp()
        self._chk(self.L.ref_read_wide_csv(str(path_in).encode(), C.byref(h)))
        try:
            self._chk(self.L.ref_write_wide_csv(h, str(path_out).encode()))
        finally:
            self.L.ref_dataset_free(h)

    def read_long_csv(self, path):
        h = _vp()
        self._chk(self.L.ref_read_long_csv(str(path).encode(), C.byref(h)))
        return h

    def long_info(self, h):
        ns = C.c_int64(); nr = C.c_int64(); p = C.c_int64(); mx = C.c_double()
        self.L.ref_long_sizes(h, C.byref(ns), C.byref(nr), C.byref(p), C.byref(mx))
        return dict(n_subjects=ns.value, n_records=nr.value, n_covariates=p.value,
                    max_stop=mx.value,
                    names=[self.L.ref_long_name(h, j).decode() for j in range(p.value)])

    def long_lower(self, h, cuts, splits=None):
        """to_time_varying + lower_pipeline: (Dataset, subjects, map_source, map_window, names)."""
        splits = splits or {}
        cov = np.array(sorted(splits), np.int64)
        ptr = np.zeros(len(cov) + 1, np.int64)
        times = []
        for q, j in enumerate(cov):
            times += list(splits[int(j)])
            ptr[q + 1] = len(times)
        tm = np.array(times, np.float64) if times else np.zeros(1)
        cu = np.ascontiguousarray(cuts, np.float64)
        out = _vp()
        m = 4096
        ms = np.zeros(m, np.int64)
        mw = np.zeros(m, np.int32)
        self._chk(self.L.ref_long_lower(h, _p(cu, C.c_double), cu.shape[0],
                                        _p(cov if len(cov) else np.zeros(1, np.int64), C.c_int64),
                                        _p(ptr, C.c_int64), _p(tm, C.c_double), len(cov),
                                        C.byref(out), _p(ms, C.c_int64), _p(mw, C.c_int32)))
        try:
            low = self._dataset(out)
            subj = np.empty(low.n, np.int64)
            self.L.ref_dataset_subject(out, _p(subj, C.c_int64))
            names = [self.L.ref_dataset_name(out, j).decode() for j in range(low.p)]
            return low, subj, ms[:low.p], mw[:low.p], names
        finally:
            self.L.ref_dataset_free(out)

    def config_script(self, text, script, origin="<config>"):
        buf = C.create_string_buffer(1 << 16)
        self.L.ref_config_script(text.encode(), origin.encode(), script.encode(), buf, len(buf))
        return buf.value.decode()

    def lower_pipeline(self, ds, cuts, splits=None, subject=None):
        """make_time_varying + lower_pipeline (transforms.cpp:64-231) of the
        reference; returns (Dataset, subjects, map_source, map_window)."""
        h = self.dataset_handle(ds)
        try:
            if subject is not None:
                sj = np.ascontiguousarray(subject, np.int64)
                self.L.ref_dataset_set_subject(h, _p(sj, C.c_int64))
            splits = splits or {}
            cov = np.array(sorted(splits), np.int64)
            ptr = np.zeros(len(cov) + 1, np.int64)
            times = []
            for q, j in enumerate(cov):
                times += list(splits[int(j)])
                ptr[q + 1] = len(times)
            tm = np.array(times, np.float64) if times else np.zeros(1)
            cu = np.ascontiguousarray(cuts, np.float64)
            out = _vp()
            ms = np.zeros(ds.p * (len(cuts) + 1), np.int64)
            mw = np.zeros(ds.p * (len(cuts) + 1), np.int32)
            self._chk(self.L.ref_lower_pipeline(h, _p(cu, C.c_double), cu.shape[0],
                                                _p(cov if len(cov) else np.zeros(1, np.int64), C.c_int64),
                                                _p(ptr, C.c_int64), _p(tm, C.c_double), len(cov),
                                                C.byref(out), _p(ms, C.c_int64), _p(mw, C.c_int32)))
            low = self._dataset(out)
            subj = np.empty(low.n, np.int64)
            self.L.ref_dataset_subject(out, _p(subj, C.c_int64))
            self.L.ref_dataset_free(out)
            return low, subj, ms[:low.p], mw[:low.p]
        finally:
            self.L.ref_dataset_free(h)

    Ref.lower_pipeline = lower_pipeline
    for f in (read_wide_csv, wide_roundtrip, read_long_csv, long_info, long_lower, config_script):
        setattr(Ref, f.__name__, f)
    Ref.fold_assignment = fold_assignment
    Ref.kfold_select_gamma = kfold_select_gamma


_ref_resample_methods()


class OrcDesign(C.Structure):
    _fields_ = [("n", C.c_int64), ("p", C.c_int64), ("k", C.c_int32), ("time", _d),
                ("event", _u8), ("head", _u8), ("tie_end", _i64), ("offsets", _i64),
                ("col_ptr", _i64), ("row_idx", _i64), ("values", _d)]


class Oracle:
    """The plain-C restatement (oracle/stratcox_oracle.c)."""

    def __init__(self, path: str = ORACLE_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        D = C.POINTER(OrcDesign)
        sig = {
            "orc_last_error": (C.c_char_p, []),
            "orc_build_sorted_design": (C.c_int, [C.c_int64, _d, _u8, _i32, C.c_int64, _i64, _i64,
                                                  _d, _i64, _u8, _i64, _i64, _i32, _d, _u8, _i32,
                                                  _i64, _d]),
            "orc_segmented_scan": (C.c_int, [C.c_int64, _d, _u8, C.c_int64, _d]),
            "orc_inclusive_scan": (C.c_int, [C.c_int64, _d, C.c_int64, _d]),
            "orc_make_state": (C.c_int, [D, _d, _d, _d]),
            "orc_update_xbeta": (C.c_int, [D, _d, _d, _d, _u32, C.c_int64, C.c_double]),
            "orc_log_partial_likelihood": (C.c_int, [D, _d, _d, C.c_int64, _d]),
            "orc_gradient_hessian": (C.c_int, [D, _d, C.c_int64, C.c_int64, _d, _d]),
            "orc_naive_gradient_hessian": (C.c_int, [D, _d, C.c_int64, _d, _d]),
            "orc_naive_log_partial_likelihood": (C.c_int, [D, _d, _d, _d]),
            "orc_newton_step": (C.c_int, [C.c_double, C.c_double, _d, _ip]),
            "orc_apply_trust_region": (C.c_int, [C.c_double, C.c_double, _d, _d]),
            "orc_l1_coordinate_update": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double,
                                                   _d, _ip, _ip]),
            "orc_ccd_fit": (C.c_int, [D, _d, C.c_int, C.c_double, C.c_double, C.c_int64, _d, _d,
                                      _d, _ip, _ip, _ip, _d, _ip]),
            "orc_ccd_fit_prior": (C.c_int, [D, _d, _d, C.c_int, C.c_double, C.c_double,
                                            C.c_int64, _d, _d, _d, _ip, _ip, _ip, _d, _ip]),
            "orc_coordinate_update": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double,
                                                C.c_double, _d, _ip, _ip]),
            "orc_gamma_max": (C.c_int, [D, C.c_int64, _d]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        self.L = L

    def _chk(self, rc):
        if rc:
            raise OracleError(rc, self.L.orc_last_error().decode())

    def build_sorted_design(self, ds: Dataset) -> dict:
        n, p = ds.n, ds.p
        z = int(ds.col_ptr[-1])
        a = dict(perm=np.empty(n, np.int64), head=np.empty(n, np.uint8),
                 tie_end=np.empty(n, np.int64), offsets=np.empty(n + 2, np.int64),
                 time=np.empty(n), event=np.empty(n, np.uint8), stratum=np.empty(n, np.int32),
                 col_ptr=np.ascontiguousarray(ds.col_ptr, np.int64).copy(),
                 row_idx=np.empty(max(z, 1), np.int64), values=np.empty(max(z, 1)))
        k = C.c_int32()
        vals = np.ascontiguousarray(ds.values, np.float64)
        self._chk(self.L.orc_build_sorted_design(
            n, _p(np.ascontiguousarray(ds.time, np.float64), C.c_double),
            _p(np.ascontiguousarray(ds.event, np.uint8), C.c_uint8),
            _p(np.ascontiguousarray(ds.stratum, np.int32), C.c_int32), p,
            _p(a["col_ptr"], C.c_int64), _p(np.ascontiguousarray(ds.row_idx, np.int64), C.c_int64),
            _p(vals, C.c_double), _p(a["perm"], C.c_int64), _p(a["head"], C.c_uint8),
            _p(a["tie_end"], C.c_int64), _p(a["offsets"], C.c_int64), C.byref(k),
            _p(a["time"], C.c_double), _p(a["event"], C.c_uint8), _p(a["stratum"], C.c_int32),
            _p(a["row_idx"], C.c_int64), _p(a["values"], C.c_double)))
        a["offsets"] = a["offsets"][:k.value + 1].copy()
        a["row_idx"] = a["row_idx"][:z]
        a["values"] = a["values"][:z]
        a["n"], a["p"], a["k"] = n, p, k.value
        return a

    def design(self, a: dict):
        """OrcDesign struct over a design-arrays dict (keeps references alive)."""
        keep = {key: np.ascontiguousarray(a[key]) for key in
                ("time", "event", "head", "tie_end", "offsets", "col_ptr", "row_idx", "values")}
        d = OrcDesign(a["n"], a["p"], a["k"], _p(keep["time"], C.c_double),
                      _p(keep["event"], C.c_uint8), _p(keep["head"], C.c_uint8),
                      _p(keep["tie_end"], C.c_int64), _p(keep["offsets"], C.c_int64),
                      _p(keep["col_ptr"], C.c_int64), _p(keep["row_idx"], C.c_int64),
                      _p(keep["values"], C.c_double))
        d._keep = keep
        return d

    def segmented_scan(self, values, flags, chunk=4096):
        v = np.ascontiguousarray(values, np.float64)
        f = np.ascontiguousarray(flags, np.uint8)
        out = np.empty_like(v)
        self._chk(self.L.orc_segmented_scan(v.shape[0], _p(v, C.c_double), _p(f, C.c_uint8),
                                            chunk, _p(out, C.c_double)))
        return out

    def make_state(self, d, beta):
        x = np.empty(d.n); e = np.empty(d.n)
        b = np.ascontiguousarray(beta, np.float64)
        self._chk(self.L.orc_make_state(C.byref(d), _p(b, C.c_double), _p(x, C.c_double),
                                        _p(e, C.c_double)))
        return x, e

    def update_xbeta(self, d, beta, xb, ex, updates, j, delta):
        u = C.c_uint32(updates)
        self._chk(self.L.orc_update_xbeta(C.byref(d), _p(beta, C.c_double), _p(xb, C.c_double),
                                          _p(ex, C.c_double), C.byref(u), j, delta))
        return u.value

    def log_partial_likelihood(self, d, xb, ex, chunk=4096):
        ll = C.c_double()
        self._chk(self.L.orc_log_partial_likelihood(C.byref(d), _p(xb, C.c_double),
                                                    _p(ex, C.c_double), chunk, C.byref(ll)))
        return ll.value

    def gradient_hessian(self, d, ex, j, chunk=4096):
        g = C.c_double(); h = C.c_double()
        self._chk(self.L.orc_gradient_hessian(C.byref(d), _p(ex, C.c_double), j, chunk,
                                              C.byref(g), C.byref(h)))
        return g.value, h.value

    def naive_gradient_hessian(self, d, ex, j):
        g = C.c_double(); h = C.c_double()
        self._chk(self.L.orc_naive_gradient_hessian(C.byref(d), _p(ex, C.c_double), j,
                                                    C.byref(g), C.byref(h)))
        return g.value, h.value

    def naive_log_partial_likelihood(self, d, xb, ex):
        ll = C.c_double()
        self._chk(self.L.orc_naive_log_partial_likelihood(C.byref(d), _p(xb, C.c_double),
                                                          _p(ex, C.c_double), C.byref(ll)))
        return ll.value

    def newton_step(self, g1, g2):
        s = C.c_double(); f = C.c_int()
        self._chk(self.L.orc_newton_step(g1, g2, C.byref(s), C.byref(f)))
        return s.value, bool(f.value)

    def apply_trust_region(self, d, t):
        a = C.c_double(); n = C.c_double()
        self._chk(self.L.orc_apply_trust_region(d, t, C.byref(a), C.byref(n)))
        return a.value, n.value

    def l1_coordinate_update(self, g1, g2, b, gm):
        s = C.c_double(); sk = C.c_int(); f = C.c_int()
        self._chk(self.L.orc_l1_coordinate_update(g1, g2, b, gm, C.byref(s), C.byref(sk),
                                                  C.byref(f)))
        return s.value, bool(sk.value), bool(f.value)

    def coordinate_update(self, g1, g2, b, gm, lam):
        s = C.c_double(); sk = C.c_int(); f = C.c_int()
        self._chk(self.L.orc_coordinate_update(g1, g2, b, gm, lam, C.byref(s), C.byref(sk),
                                               C.byref(f)))
        return s.value, bool(sk.value), bool(f.value)

    def ccd_fit(self, d, gamma, max_cycles=1000, tol=1e-6, initial_trust=1.0, chunk=4096,
                initial_beta=None, l2=None):
        """l2: optional per-coefficient L2 prior weights (extension, not in the
        reference; see orc_ccd_fit_prior)."""
        p = d.p
        beta = np.empty(p); trace = np.empty(max_cycles + 1); trust = np.empty(p)
        tl = C.c_int(); cy = C.c_int(); cv = C.c_int(); nw = C.c_int()
        g = np.ascontiguousarray(gamma, np.float64)
        lam = None if l2 is None else np.ascontiguousarray(l2, np.float64)
        ib = None if initial_beta is None else np.ascontiguousarray(initial_beta, np.float64)
        self._chk(self.L.orc_ccd_fit_prior(C.byref(d), _p(g, C.c_double), _p(lam, C.c_double),
                                     max_cycles, tol,
                                     initial_trust, chunk, _p(ib, C.c_double),
                                     _p(beta, C.c_double), _p(trace, C.c_double), C.byref(tl),
                                     C.byref(cy), C.byref(cv), _p(trust, C.c_double),
                                     C.byref(nw)))
        return dict(beta=beta, trace=trace[:tl.value].copy(), cycles=cy.value,
                    converged=bool(cv.value), trust=trust, n_warnings=nw.value)

    def gamma_max(self, d, chunk=4096):
        out = C.c_double()
        self._chk(self.L.orc_gamma_max(C.byref(d), chunk, C.byref(out)))
        return out.value
