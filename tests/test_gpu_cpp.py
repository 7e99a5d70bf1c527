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


REF_PIPE = os.path.join(ROOT, "oracle", "_ref", "ref_pipeline")


@pytest.mark.parametrize("args", [["100", "0.1", "0", "10", "4", "1", "200"],
                                  ["400", "0.1", "0", "20", "2", "2", "8"],
                                  ["300", "0.05", "3", "16", "0", "1", "12"]])
def test_reference_pipeline_with_gpu_qaoa_stage(args):
    """The reference's own run_pipeline (unmodified pipeline.hpp, CPU) against the same
    stages with only the QAOA stage (pipeline.hpp:263) replaced by
    qcut_gpu::reference::solve_batch on qcut::Graph / qcut::SolveOptions: per-subgraph
    expectation, evals and retained count, then the reference's own pools and merge give
    the same cut, assignment and leaf count (config 1 at full budget; the C2 shape; top-K 0
    = every class). Built by oracle/Makefile against /root/reference."""
    if not os.path.exists(REF_PIPE):
        pytest.skip("oracle/_ref/ref_pipeline not built (needs /root/reference)")
    r = subprocess.run([REF_PIPE, "run"] + args, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("ok cut"), r.stdout


def test_reference_types_error_mapping():
    """Engine codes come back as qcut::config_error (qaoa.hpp:162-165 top_k check)."""
    if not os.path.exists(REF_PIPE):
        pytest.skip("oracle/_ref/ref_pipeline not built (needs /root/reference)")
    r = subprocess.run([REF_PIPE, "errors"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "qcut::config_error" in r.stdout, r.stdout + r.stderr
