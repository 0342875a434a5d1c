"""CPU: file formats and configuration (paper_2310_16238_b200/io.py over
csrc/io.cpp) against the UNMODIFIED reference's io.cpp (oracle/_ref).

Wide and long CSV readers produce the reference's arrays, names and labels
bit for bit (also on files big enough for the parallel parser); writers are
byte-identical to the reference's; long files lower (to_time_varying +
lower_pipeline) to the same augmented design, names and column map; every
kind of malformed input fails with the reference's exact message; ConfigMap
scripts give the reference's results. Cases follow proj/tests/test_io.cpp."""
import os

import numpy as np
import pytest

from oracle.oracle_py import Dataset, OracleError
from paper_2310_16238_b200 import io as sio
from paper_2310_16238_b200.stratcox import SurvivalDataset, ValidationError


def _w(tmp_path, name, text):
    p = tmp_path / name
    p.write_bytes(text.encode())
    return str(p)


def _same_table(t, ref_out):
    ds, subj, names, labels = ref_out
    d = t.data
    assert np.array_equal(d.time, ds.time) and np.array_equal(d.event, ds.event)
    assert np.array_equal(d.stratum, ds.stratum) and np.array_equal(d.subject, subj)
    assert np.array_equal(d.col_ptr, ds.col_ptr) and np.array_equal(d.row_idx, ds.row_idx)
    assert np.array_equal(d.values, ds.values)
    assert t.covariate_names == names and t.stratum_labels == labels


def _wide_text(rng, n, p, labels, dense=0.3, zeros=True, crlf=False, blanks=True):
    names = [f"v{j}" for j in rng.permutation(p)] + ["a,b:c"]  # a name with ',' and ':'
    lines = ["subject,stratum,time,event,covariates"]
    for i in range(n):
        toks = []
        for nm in names:
            if rng.random() < dense:
                v = float(rng.normal()) if rng.random() < 0.5 else 1.0
                if zeros and rng.random() < 0.05:
                    v = 0.0
                toks.append(f"{nm}:{v!r}")
        lab = labels[rng.integers(len(labels))]
        t = float(np.round(rng.exponential(3.0), int(rng.integers(0, 4))))
        lines.append(f"{1000 + i}, {lab} ,{t!r},{int(rng.random() < 0.6)}, {' '.join(toks)}")
        if blanks and rng.random() < 0.02:
            lines.append("   ")
    eol = "\r\n" if crlf else "\n"
    return eol.join(lines) + eol


@pytest.mark.parametrize("labels,n,crlf", [
    (["3", "1", "10", "2"], 200, False),       # numeric labels: numeric order (10 after 3)
    (["b", "a", "c10", "c2"], 300, True),      # lexicographic
    (["1"], 60000, False),                      # big enough for several parser threads
])
def test_read_wide_matches_reference(ref, tmp_path, labels, n, crlf):
    rng = np.random.default_rng(n)
    path = _w(tmp_path, "w.csv", _wide_text(rng, n, 7, labels, crlf=crlf))
    _same_table(sio.read_wide_csv(path), ref.read_wide_csv(path))


def test_write_wide_byte_identical_and_roundtrip(ref, tmp_path):
    rng = np.random.default_rng(4)
    src = _w(tmp_path, "src.csv", _wide_text(rng, 500, 9, ["x", "y", "z"]))
    t = sio.read_wide_csv(src)
    ours, theirs = str(tmp_path / "ours.csv"), str(tmp_path / "theirs.csv")
    sio.write_wide_csv(ours, t.data, t.covariate_names, t.stratum_labels)
    ref.wide_roundtrip(src, theirs)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    again = str(tmp_path / "again.csv")  # write -> read -> write is byte-identical
    t2 = sio.read_wide_csv(ours)
    sio.write_wide_csv(again, t2.data, t2.covariate_names, t2.stratum_labels)
    assert open(again, "rb").read() == open(ours, "rb").read()


def test_write_wide_default_names_from_arrays(ref, tmp_path):
    ds = ref.simulate(80, 6, 0.3, 0.8, 3, 0.3, 12)
    data = SurvivalDataset(time=ds.time, event=ds.event, stratum=ds.stratum, col_ptr=ds.col_ptr,
                           row_idx=ds.row_idx, values=ds.values)
    path = str(tmp_path / "sim.csv")
    sio.write_wide_csv(path, data)
    back = ref.read_wide_csv(path)
    assert np.array_equal(back[0].time, ds.time)  # shortest round-trip decimal text
    assert back[2] == [f"x{j + 1}" for j in range(6)]


WIDE_BAD = [
    ("id,stratum,time,event,covariates\n", "header"),
    ("subject,stratum,time,event,covariates\n1,1,abc,1,\n", "time"),
    ("subject,stratum,time,event,covariates\n1,1,2.0,7,\n", "event 7"),
    ("subject,stratum,time,event,covariates\n1,1,2.0,x,\n", "event text"),
    ("subject,stratum,time,event,covariates\n1,1,2.0,1,a:1 a:2\n", "duplicate"),
    ("subject,stratum,time,event,covariates\n1,1,2.0,1,a:1 a:x\n", "bad value before dup"),
    ("subject,stratum,time,event,covariates\n", "no rows"),
    ("", "empty"),
    ("subject,stratum,time,event,covariates\n1,1,2.0\n", "few fields"),
    ("subject,stratum,time,event,covariates\nq,1,2.0,1,\n", "subject"),
    ("subject,stratum,time,event,covariates\n1,1,-2.0,1,\n", "negative time"),
    ("subject,stratum,time,event,covariates\n1,1,inf,1,\n", "inf time"),
    ("subject,stratum,time,event,covariates\n1,1,2,1,:3\n", "malformed"),
    ("subject,stratum,time,event,covariates\n1,1,2,1,b:inf\n", "inf value"),
    ("subject,stratum,time,event,covariates\n1,1,2,1,a:1\n2,1,3,1,a:1\n3,1,x,1,\n4,1,2,9,\n",
     "first failing line wins"),
]


@pytest.mark.parametrize("text,why", WIDE_BAD)
def test_wide_errors_match_reference(ref, tmp_path, text, why):
    path = _w(tmp_path, "bad.csv", text)
    with pytest.raises(OracleError) as want:
        ref.read_wide_csv(path)
    with pytest.raises(ValidationError) as got:
        sio.read_wide_csv(path)
    assert str(got.value) == str(want.value), why


def test_missing_file(ref, tmp_path):
    path = str(tmp_path / "nope.csv")
    with pytest.raises(OracleError) as want:
        ref.read_wide_csv(path)
    with pytest.raises(ValidationError) as got:
        sio.read_wide_csv(path)
    assert str(got.value) == str(want.value)


# ---------------------------------------------------------------- long format
EXAMPLE_LONG = ("subject,start,stop,event,covariates\n"
                "1,0,10,0,trt:1 age:63\n"
                "1,10,15,1,trt:0.5 age:63\n"
                "2,0,8,0,age:40\n"
                "3,0,10,0,trt:1\n"
                "3,10,20,1,trt:1\n")


def _random_long(rng, n, cuts, p=5):
    lines = ["subject,start,stop,event,covariates"]
    names = [f"c{j}" for j in range(p)]
    order = rng.permutation(n)
    for s in order:
        # records split at a random subset of the interior cut points
        end = float(rng.uniform(0.5, cuts[-1])) if rng.random() < 0.9 else float(cuts[-1])
        if rng.random() < 0.2:
            end = float(rng.choice(cuts[1:]))  # ties with cut points
        inner = [c for c in cuts[1:-1] if c < end and rng.random() < 0.5]
        edges = [0.0] + inner + [end]
        ev = int(rng.random() < 0.6)
        for r in range(len(edges) - 1):
            toks = [f"{nm}:{float(rng.integers(0, 3))!r}" for nm in names if rng.random() < 0.5]
            e = ev if r == len(edges) - 2 else 0
            lines.append(f"{s + 1},{edges[r]!r},{edges[r + 1]!r},{e},{' '.join(toks)}")
    return "\n".join(lines) + "\n"


def _same_lowered(ours, theirs):
    d, cmap, names = ours
    ds, subj, ms, mw, rnames = theirs
    assert np.array_equal(d.time, ds.time) and np.array_equal(d.event, ds.event)
    assert np.array_equal(d.stratum, ds.stratum) and np.array_equal(d.subject, subj)
    assert np.array_equal(d.col_ptr, ds.col_ptr) and np.array_equal(d.row_idx, ds.row_idx)
    assert np.array_equal(d.values, ds.values)
    assert [c.source for c in cmap] == list(ms) and [c.window for c in cmap] == list(mw)
    assert names == rnames


@pytest.mark.parametrize("cuts,splits", [([0.0, 10.0, 20.0], None), ([0.0, 10.0, 20.0], {0: [10.0]})])
def test_long_example_reads_writes_and_lowers_like_reference(ref, tmp_path, cuts, splits):
    path = _w(tmp_path, "long.csv", EXAMPLE_LONG)
    ours = sio.read_long_csv(path)
    h = ref.read_long_csv(path)
    try:
        info = ref.long_info(h)
        assert ours.covariate_names == info["names"] == ["trt", "age"]
        sz = ours.sizes()
        assert (sz["n_subjects"], sz["n_records"], sz["max_stop"]) == \
            (info["n_subjects"], info["n_records"], info["max_stop"])
        _same_lowered(ours.lower(cuts, splits), ref.long_lower(h, cuts, splits))
        o1, o2 = str(tmp_path / "o1.csv"), str(tmp_path / "o2.csv")
        ours.write(o1)
        ref.L.ref_write_long_csv(h, o2.encode())
        assert open(o1, "rb").read() == open(o2, "rb").read()
    finally:
        ref.L.ref_long_free(h)


@pytest.mark.parametrize("n,seed", [(300, 1), (40000, 2)])
def test_random_long_files_lower_like_reference(ref, tmp_path, n, seed):
    rng = np.random.default_rng(seed)
    cuts = [0.0, 2.0, 4.5, 7.0, 10.0]
    path = _w(tmp_path, "rl.csv", _random_long(rng, n, cuts))
    ours = sio.read_long_csv(path)
    h = ref.read_long_csv(path)
    try:
        assert ours.covariate_names == ref.long_info(h)["names"]
        for splits in (None, {1: [4.5]}, {0: [2.0, 7.0], 3: [4.5]}):
            _same_lowered(ours.lower(cuts, splits), ref.long_lower(h, cuts, splits))
    finally:
        ref.L.ref_long_free(h)


LONG_BAD = [
    "subject,start,stop,event,covariates\n1,5,10,1,\n",                   # must start at 0
    "subject,start,stop,event,covariates\n1,0,5,0,\n1,6,10,1,\n",         # contiguous
    "subject,start,stop,event,covariates\n1,0,5,1,\n1,5,10,0,\n",         # after event
    "subject,start,stop,event,covariates\n1,0,0,1,\n",                     # degenerate
    "subject,start,stop,event,covariates\n1,-1,3,1,\n",                    # negative
    "subject,start,stop,event,covariates\n1,0,x,1,\n",                     # bad stop
    "subject,start,stop,event,covariates\n1,0,3,1,a:q\n",                  # bad value
    "subject,start,stop,event,covariates\n1,0,5,0,\n1,6,10,1,\n2,0,x,1,\n",  # sequential error first
    "subject,stratum,time,event,covariates\n",                              # wrong header
    "subject,start,stop,event,covariates\n",                                # no rows
]


@pytest.mark.parametrize("text", LONG_BAD)
def test_long_errors_match_reference(ref, tmp_path, text):
    path = _w(tmp_path, "bad.csv", text)
    with pytest.raises(OracleError) as want:
        ref.read_long_csv(path)
    with pytest.raises(ValidationError) as got:
        sio.read_long_csv(path)
    assert str(got.value) == str(want.value)


@pytest.mark.parametrize("cuts,splits", [
    ([0.0, 20.0], None),                     # change at 10 not a cut point
    ([0.0, 10.0], None),                     # does not cover follow-up
    ([1.0, 10.0, 20.0], None),               # first cut point must be 0
    ([0.0, 10.0, 10.0, 20.0], None),         # not increasing
    ([0.0, 10.0, 20.0], {0: [5.0]}),         # split not a cut point
    ([0.0, 10.0, 20.0], {0: [20.0]}),        # outside the window
    ([0.0, 10.0, 20.0], {0: [10.0, 10.0]}),  # duplicate
    ([0.0, 10.0, 20.0], {0: []}),            # declares no times
    ([0.0, 10.0, 20.0], {5: [10.0]}),        # index out of range
])
def test_lowering_errors_match_reference(ref, tmp_path, cuts, splits):
    path = _w(tmp_path, "long.csv", EXAMPLE_LONG)
    ours = sio.read_long_csv(path)
    h = ref.read_long_csv(path)
    try:
        with pytest.raises(OracleError) as want:
            ref.long_lower(h, cuts, splits)
        with pytest.raises(ValidationError) as got:
            ours.lower(cuts, splits)
        assert str(got.value) == str(want.value)
    finally:
        ref.L.ref_long_free(h)


# ---------------------------------------------------------------- ConfigMap
def _our_script(text, script, origin="<config>"):
    out = []
    try:
        cfg = sio.ConfigMap.from_string(text, origin)
    except ValidationError as e:
        return f"ERR:{e}\n"
    for line in script.splitlines():
        parts = line.split(" ", 2)
        op, key = parts[0], parts[1]
        fb = parts[2] if len(parts) > 2 else ""
        try:
            if op == "S":
                out.append(cfg.get_string(key, fb))
            elif op == "D":
                out.append(repr(cfg.get_double(key, float(fb))))
            elif op == "I":
                out.append(str(cfg.get_int(key, int(fb))))
            elif op == "DL":
                out.append("|".join(repr(v) for v in cfg.get_double_list(key)))
            elif op == "SL":
                out.append("|".join(cfg.get_string_list(key)))
            elif op == "H":
                out.append("1" if cfg.has(key) else "0")
            elif op == "F":
                cfg.finish()
                out.append("OK")
        except ValidationError as e:
            out.append(f"ERR:{e}")
    return "\n".join(out) + "\n"


def _norm(s):  # doubles compared by value (to_chars vs repr spelling)
    res = []
    for line in s.splitlines():
        parts = []
        for x in line.split("|"):
            try:
                parts.append(repr(float(x)) if not x.startswith("ERR") else x)
            except ValueError:
                parts.append(x)
        res.append("|".join(parts))
    return res


CONFIGS = [
    ("tolerance = 1e-4\n# comment line\ngamma_grid = 0.1, 1, 10\nunpenalized = trt, age\n",
     "D tolerance 1e-6\nDL gamma_grid\nSL unpenalized\nH tolerance\nF x"),
    ("tolernace = 1e-4\n", "D tolerance 1e-6\nF x"),
    ("not a pair\n", "F x"),
    ("a = 1\na = 2\n", "F x"),
    (" = 3\n", "F x"),
    ("x = abc # trailing comment\ny=  7 \nz = 1,,2, ,3\nw = 2.5\n",
     "S x def\nI y 0\nDL z\nI w 0\nD x 0\nS missing fb\nF x"),
    ("a = 1\nb = 2\nc = 3\n", "I a 0\nF x"),
]


@pytest.mark.parametrize("text,script", CONFIGS)
def test_config_scripts_match_reference(ref, text, script):
    assert _norm(_our_script(text, script)) == _norm(ref.config_script(text, script))


def test_config_from_file(tmp_path, ref):
    path = _w(tmp_path, "c.cfg", "max_cycles = 50\nfolds = 5\n")
    cfg = sio.ConfigMap.from_file(path)
    assert cfg.get_int("max_cycles", 1000) == 50
    with pytest.raises(ValidationError, match=r"unknown config key\(s\): folds"):
        cfg.finish()
    with pytest.raises(ValidationError, match="cannot open"):
        sio.ConfigMap.from_file(str(tmp_path / "missing.cfg"))
