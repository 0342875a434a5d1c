"""CPU: the C-ABI library builds for sm_100a, loads, and exports exactly what
include/stratcox_b200.h declares; host-side scalar rules agree with the oracle.
(No device compute here — that is tests/test_gpu_parity.py.)"""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "stratcox_b200.h")
LIB = os.path.join(ROOT, "paper_2310_16238_b200", "libstratcox_b200.so")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-C", ROOT, "lib"], check=True, capture_output=True)
    from paper_2310_16238_b200 import _capi
    return _capi.load()


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(scx_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("scx_upload_design", "scx_gradient_hessian", "scx_log_partial_likelihood",
                 "scx_update_xbeta", "scx_make_state", "scx_ccd_fit", "scx_segmented_inclusive_scan",
                 "scx_naive_gradient_hessian", "scx_xchg_connect"):
        assert must in syms


def test_library_exports_every_declared_symbol(lib):
    from paper_2310_16238_b200 import _capi
    syms = declared_symbols()
    assert sorted(_capi.SIGNATURES) == syms
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (scx_[a-z0-9_]+)", out))
    assert set(syms) <= exported


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    assert "UTMALDG" in sass or "UBLKCP" in sass  # TMA / bulk-copy loads in the scan kernels


def test_version_and_no_device(lib):
    assert b"sm_100a" in lib.scx_version()
    assert lib.scx_device_count() >= 0


def test_scalar_rules_match_oracle(lib, oracle):
    import paper_2310_16238_b200 as sx
    rng = np.random.default_rng(3)
    for _ in range(2000):
        g1, g2 = rng.normal(0, 3), abs(rng.normal(0, 2)) * (rng.random() > 0.1)
        b = rng.normal(0, 1) * (rng.random() > 0.4)
        gm = abs(rng.normal(0, 1.5)) * (rng.random() > 0.2)
        try:
            want = oracle.l1_coordinate_update(g1, g2, b, gm)
        except Exception as e:  # noqa: BLE001
            with pytest.raises(sx.InternalError, match=str(e)):
                sx.l1_coordinate_update(g1, g2, b, gm)
            continue
        got = sx.l1_coordinate_update(g1, g2, b, gm)
        assert (got.step, got.skipped, got.flat) == want
        t = abs(rng.normal(0, 1)) + 1e-3
        assert sx.apply_trust_region(want[0], t).__dict__ == dict(
            zip(("applied", "next_trust"), oracle.apply_trust_region(want[0], t)))
    with pytest.raises(sx.NumericError, match="non-finite gradient or Hessian in Newton step"):
        sx.newton_step(float("nan"), 1.0)
    with pytest.raises(sx.NumericError, match="non-finite trust-region inputs"):
        sx.apply_trust_region(float("inf"), 1.0)
