"""GPU parity at the BASELINE subgraph sizes: 20-26 qubits (2 and 3 passes per layer,
several high passes, mirror in the last one). Bit-exact amplitudes / expectation / top-K
against the oracle (kQubitCap raised to 26 like oracle/_ref/libqcut_ref26.so)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
THREADS = max(1, min(32, os.cpu_count() or 1))


@pytest.fixture(scope="module")
def oracle26(oracle):
    oracle.set_qubit_cap(26)
    yield oracle
    oracle.set_qubit_cap(24)


@pytest.mark.parametrize("q,layers", [(21, 1), (22, 2), (24, 1), (26, 1)])
def test_large_run_ansatz_bit_exact(engine, oracle26, q, layers):
    e = oracle26.generate_er(q, 0.15, q)
    rng = np.random.default_rng(q)
    g = rng.uniform(0, np.pi, layers)
    b = rng.uniform(0, np.pi, layers)
    a0, x0 = oracle26.run_ansatz(q, e, g, b, threads=THREADS)
    a1, x1 = engine.run_ansatz(q, e, g, b)
    assert x1 == x0
    assert np.array_equal(a1, a0)
    for k in (1, 8):
        b0, p0 = oracle26.top_candidates(a0, k, True)
        b1, p1 = engine.top_candidates(a1, k, True)
        assert np.array_equal(b1, b0) and np.array_equal(p1, p0)
    del a0, a1


def test_large_solve_short_budget(engine, oracle26):
    q = 24
    e = oracle26.generate_er(q, 0.1, 7)
    ref = oracle26.solve_subgraph(q, e, top_k=4, layers=1, budget=6, seed=3, qubit_cap=26,
                                  threads=THREADS)
    got = engine.solve_subgraph(q, e, top_k=4, layers=1, budget=6, seed=3, qubit_cap=26)
    assert np.array_equal(got.bits, ref.bits) and np.array_equal(got.probs, ref.probs)
    assert got.expectation == ref.expectation and got.evals == ref.evals
    assert np.array_equal(got.params, ref.params[:2])


def test_weighted_integral_c3_like(engine, oracle):
    # config-3-like piece: integer weights U{1..10} on a sparse 3-regular-ish graph
    rng = np.random.default_rng(3)
    n = 16
    edges = []
    for u in range(n):
        for v in (u + 1, u + 5):
            if v < n:
                edges.append((u, v, float(rng.integers(1, 11))))
    ref = oracle.solve_subgraph(n, edges, top_k=3, layers=2, budget=40, seed=1, qubit_cap=24)
    got = engine.solve_subgraph(n, edges, top_k=3, layers=2, budget=40, seed=1, qubit_cap=24)
    assert np.array_equal(got.bits, ref.bits) and got.expectation == ref.expectation


@pytest.mark.parametrize("q", [14, 20, 22])
def test_large_lut_from_global_memory(engine, oracle26, q):
    """Integer weights with a total above the pass kernels' shared-memory LUT cache (224
    entries): the phase table is read from global memory (qc_pass.cu lut_sm == false).
    Bit-exact amplitudes and expectation against the oracle, and eval_batch."""
    rng = np.random.default_rng(q)
    edges = [(u, v, float(rng.integers(20, 60))) for u in range(q) for v in range(u + 1, q)
             if rng.random() < 0.25]
    assert sum(w for _, _, w in edges) + 1 > 224
    g = rng.uniform(0.05, 0.3, 2)
    b = rng.uniform(0.1, 3.0, 2)
    a0, x0 = oracle26.run_ansatz(q, edges, g, b, threads=THREADS)
    a1, x1 = engine.run_ansatz(q, edges, g, b)
    assert x1 == x0 and np.array_equal(a1, a0)
    got = engine.eval_batch([(q, edges)], 2, np.zeros(1, np.int32), np.concatenate([g, b])[None, :])
    assert got[0] == x0
    del a0, a1
