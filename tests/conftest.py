"""Test configuration: the `gpu` marker and shared fixtures.

`-m "not gpu"` runs here (no GPU): the oracle against the golden fixtures, host logic,
and the C-ABI library's exports. `-m gpu` runs on a B200: parity of the CUDA path
against the oracle (oracle/), always through the C-ABI (include/qcgpu.h).
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.refpy import OracleLib, oracle_available
    if not oracle_available():
        import subprocess
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True,
                       capture_output=True)
    return OracleLib()


@pytest.fixture(scope="session")
def ref():
    from oracle.refpy import RefLib, ref_available
    if not ref_available():
        pytest.skip("reference build (oracle/_ref) not present")
    return RefLib()


@pytest.fixture(scope="session")
def engine():
    from paper_2603_26232_b200 import Engine
    return Engine(0)
