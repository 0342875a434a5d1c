"""Test configuration.

Markers:
  gpu  — needs a B200 (sm_100a) and the built libstratcox_b200.so; the parity
         tests proper. Everything else runs on the CPU build container.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a B200 GPU and the sm_100a library")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle_py import Oracle, ORACLE_PATH
    if not os.path.exists(ORACLE_PATH):
        import subprocess
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle_py import Ref, REF_PATH
    if not os.path.exists(REF_PATH):
        pytest.skip("oracle/_ref/libstratcox_ref.so not built (reference sources absent)")
    return Ref()
