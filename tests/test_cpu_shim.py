"""CPU: include/qcut_gpu.hpp on the reference's own types (QCUT_GPU_REFERENCE_TYPES)
compiles against the unmodified reference headers and maps the engine's error codes to
qcut::config_error / resource_error / io_error (errors.hpp:8-24). Without a GPU the engine
refuses to start, which must surface as qcut::resource_error."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj/include/qcut/pipeline.hpp"


@pytest.mark.skipif(not os.path.exists(REF), reason="reference tree not present")
def test_reference_types_shim_builds_and_maps_errors():
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True,
                   capture_output=True, timeout=600)
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_pipeline")
    r = subprocess.run([exe, "errors"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    assert "qcut::resource_error" in r.stdout or "qcut::config_error" in r.stdout, r.stdout
