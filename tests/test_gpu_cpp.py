"""GPU: the C++ drop-in (include/qcut_gpu.hpp) reproduces config 1 end to end."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_shim_config1():
    out = os.path.join(ROOT, "build", "shim_config1")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include",
                    f"{ROOT}/tests/cpp/shim_config1.cpp", f"-L{ROOT}/paper_2603_26232_b200",
                    "-lqcgpu", f"-Wl,-rpath,{ROOT}/paper_2603_26232_b200", "-o", out], check=True)
    r = subprocess.run([out], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert "cut 296.0 leaves 8388608" in r.stdout
    assert "config_error ok" in r.stdout
