"""File formats and configuration (io.hpp) over the C-ABI (csrc/io.cpp).

Same names, argument meaning and error messages as the reference:

* ``read_wide_csv(path)`` / ``write_wide_csv(path, data)`` — the wide layout
  ``subject,stratum,time,event,covariates`` (io.cpp:123-223);
* ``read_long_csv(path)`` -> ``LongData`` (io.cpp:225-272) with ``write``
  (io.cpp:274-291) and ``lower(cut_points, splits)`` = to_time_varying
  (io.cpp:293-345) + lower_pipeline (transforms.cpp:225-231);
* ``ConfigMap`` (io.cpp:347-438).

Errors are ValidationError with the reference's validation_error text.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

from . import _capi
from ._capi import ptr
from .stratcox import ColumnMapEntry, SurvivalDataset, ValidationError

_ERRCAP = 4096


def _lib():
    return _capi.load()


def _arr(pt, cnt, dt):
    if cnt == 0:
        return np.zeros(0, dt)
    return np.ctypeslib.as_array(pt, shape=(cnt,)).astype(dt, copy=True)


def _dataset_from_view(v: _capi.DatasetC) -> SurvivalDataset:
    n, p = int(v.n_rows), int(v.n_covariates)
    cp = _arr(v.col_ptr, p + 1, np.int64)
    z = int(cp[-1]) if p else 0
    return SurvivalDataset(time=_arr(v.time, n, np.float64), event=_arr(v.event, n, np.uint8),
                           stratum=_arr(v.stratum, n, np.int32), col_ptr=cp,
                           row_idx=_arr(v.row_idx, z, np.int64),
                           values=_arr(v.values, z, np.float64),
                           subject=_arr(v.subject, n, np.int64))


@dataclass
class Table:
    """A SurvivalDataset read from a wide file, with its names and labels."""
    data: SurvivalDataset
    covariate_names: List[str]
    stratum_labels: List[str]


def read_wide_csv(path: str) -> Table:
    lib = _lib()
    h = C.c_void_p()
    err = C.create_string_buffer(_ERRCAP)
    if lib.scx_read_wide_csv(str(path).encode(), C.byref(h), err, _ERRCAP):
        raise ValidationError(err.value.decode())
    try:
        v = _capi.DatasetC()
        lib.scx_table_dataset(h, C.byref(v))
        data = _dataset_from_view(v)
        names = [lib.scx_table_covariate_name(h, j).decode() for j in range(data.n_covariates())]
        labels = [lib.scx_table_stratum_label(h, k).decode()
                  for k in range(1, lib.scx_table_n_strata(h) + 1)]
        return Table(data, names, labels)
    finally:
        lib.scx_table_free(h)


def write_wide_csv(path: str, data: SurvivalDataset, covariate_names: Optional[Sequence[str]] = None,
                   stratum_labels: Optional[Sequence[str]] = None) -> None:
    lib = _lib()
    ds, keep = data._c()

    def strings(xs):
        if xs is None:
            return None
        arr = (C.c_char_p * len(xs))(*[x.encode() for x in xs])
        return arr

    nm, lb = strings(covariate_names), strings(stratum_labels)
    err = C.create_string_buffer(_ERRCAP)
    if lib.scx_write_wide_csv(str(path).encode(), C.byref(ds), nm, lb, err, _ERRCAP):
        raise ValidationError(err.value.decode())


class LongData:
    """LongData (io.hpp:32-43): per-subject interval records from a long file."""

    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib().scx_long_free(h)
            self._h = None

    def sizes(self) -> Dict[str, float]:
        ns = C.c_int64(); nr = C.c_int64(); p = C.c_int64(); mx = C.c_double()
        _lib().scx_long_sizes(self._h, C.byref(ns), C.byref(nr), C.byref(p), C.byref(mx))
        return dict(n_subjects=ns.value, n_records=nr.value, n_covariates=p.value,
                    max_stop=mx.value)

    @property
    def covariate_names(self) -> List[str]:
        p = self.sizes()["n_covariates"]
        return [_lib().scx_long_covariate_name(self._h, j).decode() for j in range(int(p))]

    @property
    def max_stop(self) -> float:
        return self.sizes()["max_stop"]

    def write(self, path: str) -> None:
        err = C.create_string_buffer(_ERRCAP)
        if _lib().scx_write_long_csv(str(path).encode(), self._h, err, _ERRCAP):
            raise ValidationError(err.value.decode())

    def lower(self, cut_points, splits: Optional[Dict[int, Sequence[float]]] = None):
        """to_time_varying + lower_pipeline: (SurvivalDataset, [ColumnMapEntry], names)."""
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
        h = C.c_void_p()
        err = C.create_string_buffer(_ERRCAP)
        if lib.scx_long_lower(self._h, ptr(cuts, C.c_double), cuts.shape[0], ptr(cov, C.c_int64),
                              ptr(sptr, C.c_int64), ptr(tm, C.c_double), len(cov), C.byref(h),
                              err, _ERRCAP):
            raise ValidationError(err.value.decode())
        try:
            v = _capi.DatasetC()
            lib.scx_lowered_dataset(h, C.byref(v))
            data = _dataset_from_view(v)
            p = data.n_covariates()
            src = np.empty(p, np.int64); win = np.empty(p, np.int32)
            ws = np.empty(p); we = np.empty(p)
            lib.scx_lowered_column_map(h, ptr(src, C.c_int64),
                                       win.ctypes.data_as(C.POINTER(C.c_int32)),
                                       ptr(ws, C.c_double), ptr(we, C.c_double))
            cmap = [ColumnMapEntry(c, int(src[c]), int(win[c]), float(ws[c]), float(we[c]))
                    for c in range(p)]
            names = [lib.scx_lowered_covariate_name(h, j).decode() for j in range(p)]
            return data, cmap, names
        finally:
            lib.scx_lowered_free(h)


def read_long_csv(path: str) -> LongData:
    h = C.c_void_p()
    err = C.create_string_buffer(_ERRCAP)
    if _lib().scx_read_long_csv(str(path).encode(), C.byref(h), err, _ERRCAP):
        raise ValidationError(err.value.decode())
    return LongData(h)


class ConfigMap:
    """ConfigMap (io.hpp:57-76): flat key = value text, '#' comments; every
    getter marks its key consumed and finish() rejects the rest."""

    def __init__(self, handle):
        self._h = handle

    @staticmethod
    def from_string(text: str, origin: str = "<config>") -> "ConfigMap":
        h = C.c_void_p()
        err = C.create_string_buffer(_ERRCAP)
        if _lib().scx_config_from_string(text.encode(), origin.encode(), C.byref(h), err, _ERRCAP):
            raise ValidationError(err.value.decode())
        return ConfigMap(h)

    @staticmethod
    def from_file(path: str) -> "ConfigMap":
        h = C.c_void_p()
        err = C.create_string_buffer(_ERRCAP)
        if _lib().scx_config_from_file(str(path).encode(), C.byref(h), err, _ERRCAP):
            raise ValidationError(err.value.decode())
        return ConfigMap(h)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            _lib().scx_config_free(h)
            self._h = None

    def has(self, key: str) -> bool:
        return bool(_lib().scx_config_has(self._h, key.encode()))

    def get_string(self, key: str, fallback: str) -> str:
        return _lib().scx_config_get_string(self._h, key.encode(), fallback.encode()).decode()

    def get_double(self, key: str, fallback: float) -> float:
        out = C.c_double()
        err = C.create_string_buffer(_ERRCAP)
        if _lib().scx_config_get_double(self._h, key.encode(), float(fallback), C.byref(out), err,
                                        _ERRCAP):
            raise ValidationError(err.value.decode())
        return out.value

    def get_int(self, key: str, fallback: int) -> int:
        out = C.c_int64()
        err = C.create_string_buffer(_ERRCAP)
        if _lib().scx_config_get_int(self._h, key.encode(), int(fallback), C.byref(out), err,
                                     _ERRCAP):
            raise ValidationError(err.value.decode())
        return out.value

    def get_double_list(self, key: str) -> List[float]:
        lib = _lib()
        n = C.c_int64()
        err = C.create_string_buffer(_ERRCAP)
        if lib.scx_config_get_double_list(self._h, key.encode(), None, 0, C.byref(n), err, _ERRCAP):
            raise ValidationError(err.value.decode())
        out = np.empty(n.value)
        lib.scx_config_get_double_list(self._h, key.encode(), ptr(out, C.c_double), n.value,
                                       C.byref(n), err, _ERRCAP)
        return [float(x) for x in out]

    def get_string_list(self, key: str) -> List[str]:
        n = C.c_int64()
        s = _lib().scx_config_get_string_list(self._h, key.encode(), C.byref(n)).decode()
        return s.split("\n") if n.value else []

    def finish(self) -> None:
        err = C.create_string_buffer(_ERRCAP)
        if _lib().scx_config_finish(self._h, err, _ERRCAP):
            raise ValidationError(err.value.decode())
