"""Helpers to turn tests/golden/*.npz fixtures into designs for the oracle and
the device library. Fixtures are produced by tests/golden/make_golden.py from
the compiled reference."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
_cache = {}


def load(name):
    if name not in _cache:
        _cache[name] = dict(np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False))
    return _cache[name]


def design_arrays(z, prefix):
    """Design-arrays dict (oracle layout) from a fixture prefix."""
    a = dict(offsets=z[prefix + "offsets"].astype(np.int64), event=z[prefix + "event"],
             tie_end=z[prefix + "tie_end"].astype(np.int64), head=z[prefix + "head"],
             time=z[prefix + "time"], perm=z[prefix + "perm"].astype(np.int64),
             col_ptr=z[prefix + "col_ptr"].astype(np.int64),
             row_idx=z[prefix + "row_idx"].astype(np.int64))
    nnz = int(a["col_ptr"][-1])
    a["values"] = z[prefix + "values"] if prefix + "values" in z else np.ones(nnz)
    a["n"] = int(a["event"].shape[0])
    a["p"] = int(a["col_ptr"].shape[0] - 1)
    a["k"] = int(a["offsets"].shape[0] - 1)
    return a


def sorted_design(a, values=True):
    from paper_2310_16238_b200.stratcox import SortedDesign
    vals = a["values"] if values else None
    if vals is not None and a["row_idx"].shape[0] and np.all(vals == 1.0):
        vals = None
    return SortedDesign(stratum_offsets=a["offsets"], event=a["event"],
                        tie_group_end=a["tie_end"], col_ptr=a["col_ptr"],
                        row_idx=a["row_idx"], values=vals, time=a["time"], perm=a["perm"],
                        head_flags=a["head"])


def dataset(z, prefix):
    from oracle.oracle_py import Dataset
    return Dataset(z[prefix + "in_time"], z[prefix + "in_event"], z[prefix + "in_stratum"],
                   z[prefix + "in_col_ptr"].astype(np.int64),
                   z[prefix + "in_row_idx"].astype(np.int64), z[prefix + "in_values"])


def close_rel(a, b, tol):
    """oracles::close_rel (proj/tests/oracles.hpp:39-41)."""
    return abs(a - b) <= tol * max(1.0, abs(a), abs(b))
