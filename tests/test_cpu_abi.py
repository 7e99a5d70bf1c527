"""CPU: the C-ABI library (libqcgpu.so) loads, exports every symbol include/qcgpu.h
declares, and its host-only logic (ask/tell optimisers, shard ranges, records, partition
mirror) matches the reference semantics. No compute calls need a GPU here."""
import ctypes as C
import json
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2603_26232_b200 import load_library
    return load_library()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "qcgpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qc_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    syms = declared_symbols()
    assert len(syms) >= 35
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    from paper_2603_26232_b200 import EXPORTED_SYMBOLS
    assert set(EXPORTED_SYMBOLS) <= set(syms)


def test_library_is_sm100a(lib):
    from paper_2603_26232_b200 import library_path
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", library_path()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_cap(lib):
    assert lib.qc_abi_version() == 2
    assert lib.qc_qubit_cap() >= 26  # BASELINE config 5 needs 26 qubits


def test_engine_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_26232_b200 import Engine, QcError
    with pytest.raises(QcError):
        Engine(0)


def test_linear_ramp(lib, oracle):
    for p in (1, 2, 3, 7):
        g = np.zeros(p)
        b = np.zeros(p)
        assert lib.qc_linear_ramp(p, g.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p)) == 0
        g0, b0 = oracle.linear_ramp(p)
        assert np.array_equal(g, g0) and np.array_equal(b, b0)
    assert lib.qc_linear_ramp(0, None, None) == 1  # config_error (qaoa.hpp:28)


def _drive_optimizer(lib, objective, p, budget, seed, tol=1e-5):
    h = C.c_void_p()
    assert lib.qc_optimizer_create(p, budget, C.c_uint64(seed), C.c_double(tol), C.byref(h)) == 0
    xs, fs = [], []
    x = np.zeros(2 * p)
    done = C.c_int(0)
    while True:
        assert lib.qc_optimizer_ask(h, x.ctypes.data_as(C.c_void_p), C.byref(done)) == 0
        if done.value:
            break
        f = objective(x.copy())
        xs.append(x.copy())
        fs.append(f)
        assert lib.qc_optimizer_tell(h, C.c_double(f)) == 0
    params = np.zeros(2 * p)
    ex = C.c_double(0)
    ev = C.c_int(0)
    assert lib.qc_optimizer_result(h, params.ctypes.data_as(C.c_void_p), C.byref(ex), C.byref(ev)) == 0
    lib.qc_optimizer_destroy(h)
    return np.array(xs), np.array(fs), params, ex.value, ev.value


def test_ask_tell_optimizer_reproduces_reference_trajectories(lib, oracle):
    """The engine's lockstep optimiser (qc_nm.hpp) driven by the oracle objective must
    replay the reference's optimize_parameters trajectory (tests/golden/traces.npz)."""
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))
    tr = np.load(os.path.join(ROOT, "tests", "golden", "traces.npz"))
    for c in gold["optimize"]:
        n, p = c["n"], c["layers"]
        e = oracle.generate_er(n, c["p_edge"], c["seed"])

        def objective(x):
            return -oracle.run_ansatz(n, e, x[:p], x[p:], want_amps=False)[1]

        xs, fs, params, ex, ev = _drive_optimizer(lib, objective, p, c["budget"], c["seed"])
        k = c["key"]
        assert np.array_equal(xs, tr[f"x{k}"])
        assert np.array_equal(fs, tr[f"f{k}"])
        assert [float(v) for v in params] == [float.fromhex(h) for h in c["params"]]
        assert ex == float.fromhex(c["expectation"]) and ev == c["evals"]


def test_simplex_bowl_and_budget(lib):
    # test_qaoa.cpp:209-241
    def run(x0, budget, tol, f):
        x0 = np.asarray(x0, float)
        h = C.c_void_p()
        assert lib.qc_simplex_create(x0.ctypes.data_as(C.c_void_p), len(x0), budget,
                                     C.c_double(tol), C.byref(h)) == 0
        x = np.zeros(len(x0))
        done = C.c_int(0)
        calls = 0
        while True:
            lib.qc_simplex_ask(h, x.ctypes.data_as(C.c_void_p), C.byref(done))
            if done.value:
                break
            calls += 1
            lib.qc_simplex_tell(h, C.c_double(f(x)))
        bx = np.zeros(len(x0))
        val = C.c_double(0)
        ev = C.c_int(0)
        conv = C.c_int(0)
        lib.qc_simplex_result(h, bx.ctypes.data_as(C.c_void_p), C.byref(val), C.byref(ev), C.byref(conv))
        lib.qc_simplex_destroy(h)
        return bx, val.value, ev.value, bool(conv.value), calls

    bx, val, ev, conv, calls = run([0, 0], 500, 1e-10, lambda x: (x[0] - 2) ** 2 + (x[1] + 1) ** 2)
    assert conv and val < 1e-8 and abs(bx[0] - 2) < 1e-3 and abs(bx[1] + 1) < 1e-3
    for budget in (1, 2, 5, 37):
        _, _, ev, conv, calls = run([1, 1], budget, 1e-5, lambda x: x[0] ** 2 + np.sin(x[1]))
        assert calls == ev <= budget
        if budget <= 3:
            assert not conv
    h = C.c_void_p()
    assert lib.qc_simplex_create(None, 0, 10, C.c_double(1e-5), C.byref(h)) == 1  # config_error


def test_records_and_shards(lib):
    from paper_2603_26232_b200 import kcap_for
    lib.qc_record_bytes.restype = C.c_int64
    assert lib.qc_record_bytes(4, 1) == 24 + 16 + 32 + 16
    b, e = C.c_int32(0), C.c_int32(0)
    spans = []
    for i in range(8):
        assert lib.qc_shard_range(527, i, 8, C.byref(b), C.byref(e)) == 0
        spans.append((b.value, e.value))
    assert spans[0] == (0, 66) and spans[-1][1] == 527
    assert all(spans[i][1] == spans[i + 1][0] for i in range(7))
    assert max(e - b for b, e in spans) - min(e - b for b, e in spans) <= 1
    assert lib.qc_shard_range(10, 3, 2, C.byref(b), C.byref(e)) == 1
    assert kcap_for(20, 4) == 4 and kcap_for(3, 0) == 4


def test_python_partition_mirror_matches_oracle(oracle):
    from paper_2603_26232_b200 import partition_chain, derive_subgraph_count
    e = oracle.generate_er(100, 0.1, 0)
    for M, mode in [(11, 0), (5, 1), (1, 0), (33, 0)]:
        P = partition_chain(100, e, M, mode)
        f, l, lm, inter = oracle.partition(100, e, M, mode)
        assert np.array_equal(P.first, f) and np.array_equal(P.last, l) and P.inter == inter
        assert [len(x[1]) for x in P.local] == list(lm)
    assert derive_subgraph_count(100, 10) == oracle.derive_subgraph_count(100, 10) == 11
    assert derive_subgraph_count(16000, 26) == 640 and derive_subgraph_count(10000, 20) == 527


def test_product_generators_match_oracle(oracle):
    """bench.py builds its inputs with the PRODUCT's host generators (qc_generate_er,
    graph.hpp:146-160; qc_generate_regular for config 3); they equal the oracle's."""
    from paper_2603_26232_b200 import generate_er, generate_regular
    for n, p, seed in [(100, 0.1, 0), (400, 0.1, 0), (37, 0.5, 9)]:
        assert np.array_equal(generate_er(n, p, seed), oracle.generate_er(n, p, seed))
    g = generate_regular(1000, 3, 0, 1, 10)
    assert np.array_equal(g, oracle.generate_regular(1000, 3, 0, 1, 10))
    assert len(g) == 1500
    deg = np.bincount(np.concatenate([g["u"], g["v"]]), minlength=1000)
    assert (deg == 3).all() and (g["u"] < g["v"]).all()
    assert set(np.unique(g["w"])) <= set(float(x) for x in range(1, 11))


def _big_edges(n=3000, m=400_000, seed=5):
    """m distinct (u < v) pairs over n vertices as an EDGE_DTYPE array (integer weights)."""
    from paper_2603_26232_b200 import EDGE_DTYPE
    rng = np.random.default_rng(seed)
    keys = np.unique(rng.integers(0, n * (n - 1) // 2, size=int(m * 1.2)))[:m]
    rng.shuffle(keys)
    # index k of the row-major upper triangle -> (u, v)
    u = (n - 2 - np.floor(np.sqrt(-8 * keys + 4 * n * (n - 1) - 7) / 2.0 - 0.5)).astype(np.int64)
    v = keys + u + 1 - n * (n - 1) // 2 + (n - u) * ((n - u) - 1) // 2
    e = np.zeros(len(keys), dtype=EDGE_DTYPE)
    e["u"], e["v"], e["w"] = u, v, rng.integers(1, 4, size=len(keys)).astype(np.float64)
    flip = rng.random(len(keys)) < 0.5
    e["u"][flip], e["v"][flip] = v[flip], u[flip]
    return e


def _load_error(n, e):
    from paper_2603_26232_b200 import QcError, run_record_bytes
    try:
        run_record_bytes(n, e, qubit_cap=20, layers=1, top_k=2)
    except QcError as ex:
        return str(ex)
    return None


def test_large_graph_validation_first_error():
    """load_graph's parallel validation (m >= 2^18) accepts a valid large edge list and, on any
    problem, reports exactly the first error in edge order as graph.hpp:37-50 add_edge does
    (qc_engine.cpp load_graph falls back to the serial loop)."""
    n = 3000
    e = _big_edges(n)
    assert len(e) == 400_000 and np.all(e["u"] != e["v"])
    assert _load_error(n, e) is None
    # a duplicate late in the list, then a self-loop after it: the duplicate is reported
    d = e.copy()
    d[350_000] = (d[10]["v"], d[10]["u"], 1.0)
    d[390_000] = (7, 7, 1.0)
    lo, hi = sorted((int(d[10]["u"]), int(d[10]["v"])))
    assert f"duplicate edge ({lo},{hi})" in _load_error(n, d)
    # the self-loop first: it is reported
    d2 = e.copy()
    d2[300_000] = (7, 7, 1.0)
    d2[350_000] = (d2[10]["v"], d2[10]["u"], 1.0)
    assert "self-loop rejected at vertex 7" in _load_error(n, d2)
    # out-of-range endpoint and negative weight
    d3 = e.copy()
    d3[200_000] = (1, n, 1.0)
    assert "out of range" in _load_error(n, d3)
    d4 = e.copy()
    d4[399_999]["w"] = -1.0
    assert "negative or NaN" in _load_error(n, d4)
