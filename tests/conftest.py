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
def restatement():
    """oracle/qcut_oracle.c (the C restatement), pinned by the -m "not gpu" tests against
    the golden vectors the reference produced and against oracle/_ref directly."""
    from oracle.refpy import OracleLib, oracle_available
    if not oracle_available():
        import subprocess
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True,
                       capture_output=True)
    return OracleLib()


@pytest.fixture(scope="session")
def reference_checker(restatement):
    """The GPU parity checker: the reference build itself (oracle/_ref, which travels to
    the GPU box in the repo snapshot) whenever it is present, else the restatement."""
    from oracle.refpy import checker
    return checker()


def _is_gpu_module(module) -> bool:
    marks = getattr(module, "pytestmark", [])
    marks = marks if isinstance(marks, list) else [marks]
    return any(getattr(m, "name", "") == "gpu" for m in marks)


@pytest.fixture(scope="module")
def oracle(request, restatement, reference_checker):
    """-m gpu modules: the reference build (RefChecker); CPU modules: the restatement
    under test."""
    return reference_checker if _is_gpu_module(request.module) else restatement


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
