"""CPU: the C restatement (oracle/qcut_oracle.c) is pinned against the reference.

1. against the committed golden vectors (tests/golden/, generated from the unmodified
   reference by oracle/gen_golden.py) — runs everywhere, including the GPU box;
2. against the compiled reference itself (oracle/_ref) on seeded sweeps — runs where
   the reference build exists.
Everything is bit-exact (== on float64 bit patterns).
"""
import hashlib
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(GOLD, "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def traces():
    return np.load(os.path.join(GOLD, "traces.npz"))


def fx(h):
    return float.fromhex(h)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_config1_pipeline(oracle, gold):
    g = gold["config1"]
    e = oracle.generate_er(100, 0.1, 0)
    assert len(e) == g["edges"] and sha(e) == g["edges_sha"]
    rep = oracle.run_pipeline(100, e, qubit_cap=10, top_k=4, layers=1, budget=200, seed=0)
    assert rep["cut"] == g["cut"] == 296.0
    assert rep["assignment"] == g["assignment"]
    assert rep["leaves"] == g["leaves"]
    first, last, _, inter = oracle.partition(100, e, 11, 0, 10)
    assert list(first) == g["first"] and list(last) == g["last"] and inter == g["inter_edges"]


def test_config1_subgraph_solves(oracle, gold):
    g = gold["config1"]
    e = oracle.generate_er(100, 0.1, 0)
    for i, s in enumerate(g["subgraphs"]):
        a, b = g["first"][i], g["last"][i]
        sel = (e["u"] >= a) & (e["v"] <= b)
        le = e[sel].copy()
        le["u"] -= a
        le["v"] -= a
        r = oracle.solve_subgraph(b - a + 1, le, top_k=4, layers=1, budget=200, seed=i,
                                  qubit_cap=10)
        assert r.expectation == fx(s["expectation"])
        assert [float(x) for x in r.params[:2]] == [fx(x) for x in s["params"]]
        assert list(r.bits) == s["bits"]
        assert [float(x) for x in r.probs] == [fx(x) for x in s["probs"]]
        assert r.evals == s["evals"] == 200


def test_ansatz_amplitudes(oracle, gold):
    for c in gold["ansatz"]:
        e = oracle.generate_er(c["q"], c["p_edge"], c["seed"])
        g = [fx(x) for x in c["gammas"]]
        b = [fx(x) for x in c["betas"]]
        a, ex = oracle.run_ansatz(c["q"], e, g, b)
        assert sha(a) == c["amps_sha"], c
        assert ex == fx(c["expectation"])
        assert oracle.norm_sq(a) == fx(c["norm"])


def test_optimize_traces(oracle, gold, traces):
    for c in gold["optimize"]:
        e = oracle.generate_er(c["n"], c["p_edge"], c["seed"])
        o = oracle.optimize(c["n"], e, c["layers"], c["budget"], c["seed"], trace=True)
        k = c["key"]
        assert np.array_equal(o["trace_x"], traces[f"x{k}"])
        assert np.array_equal(o["trace_f"], traces[f"f{k}"])
        assert [float(x) for x in o["params"]] == [fx(x) for x in c["params"]]
        assert o["expectation"] == fx(c["expectation"]) and o["evals"] == c["evals"]


def test_topk_plateaus(oracle, gold):
    t = gold["topk"]
    e = oracle.generate_er(10, 0.1, 0)
    a, _ = oracle.run_ansatz(10, e, [fx(t["gamma"])], [fx(t["beta"])])
    for c in t["cases"]:
        bits, probs = oracle.top_candidates(a, c["k"], c["fold"])
        assert list(bits) == c["bits"]
        assert sha(probs) == c["probs_sha"]


def test_merges(oracle, gold):
    from oracle.refpy import edges_array
    for c in gold["merge"]:
        if "edges" in c:
            e = edges_array([(u, v, fx(w)) for u, v, w in c["edges"]])
        else:
            n_p = {"er13": (13, 0.4, 3), "er21": (21, 0.3, 9), "er400": (400, 0.1, 0)}[c["name"]]
            e = oracle.generate_er(*n_p)
        assert sha(e) == c["edges_sha"]
        pool = [(w, b) for w, b in c["pool"]]
        for inc in (0, 1):
            key = f"level_inc{inc}"
            if key in c:
                r = oracle.level_merge(c["n"], e, c["M"], pool, incremental=bool(inc))
                assert r.value == fx(c[key]["value"])
                assert "".join(map(str, r.assignment)) == c[key]["assignment"]
                assert r.leaves == c[key]["leaves"]
        r = oracle.chained_merge(c["n"], e, c["M"], pool)
        assert r.value == fx(c["chained"]["value"])
        assert "".join(map(str, r.assignment)) == c["chained"]["assignment"]
        assert r.leaves == c["chained"]["leaves"]


# ---- reference-backed sweeps (only where oracle/_ref was built) --------------------------
@pytest.mark.parametrize("seed", range(6))
def test_vs_reference_statevector(oracle, ref, seed):
    rng = np.random.default_rng(seed)
    q = int(rng.integers(2, 15))
    e = ref.generate_er(q, float(rng.uniform(0.1, 0.9)), seed)
    p = int(rng.integers(1, 4))
    g, b = rng.uniform(0, np.pi, p), rng.uniform(0, np.pi, p)
    a0, e0 = ref.run_ansatz(q, e, g, b)
    a1, e1 = oracle.run_ansatz(q, e, g, b)
    assert np.array_equal(a0, a1) and e0 == e1
    for k, fold in [(1, True), (3, False), (min(16, 1 << (q - 1)), True)]:
        r0 = ref.top_candidates(a0, k, fold)
        r1 = oracle.top_candidates(a0, k, fold)
        assert np.array_equal(r0[0], r1[0]) and np.array_equal(r0[1], r1[1])


def test_vs_reference_fractional(oracle, ref):
    from oracle.refpy import edges_array
    rng = np.random.default_rng(3)
    e = edges_array([(u, v, float(0.1 + rng.uniform())) for u in range(9) for v in range(u + 1, 9)
                     if rng.uniform() < 0.5])
    t0 = ref.cost_table(9, e)
    t1 = oracle.cost_table(9, e)
    assert np.array_equal(t0[0], t1[0]) and t0[1:] == t1[1:] and not t0[1]
    a0, e0 = ref.run_ansatz(9, e, [0.4, 1.2], [0.9, 0.3])
    a1, e1 = oracle.run_ansatz(9, e, [0.4, 1.2], [0.9, 0.3])
    assert np.array_equal(a0, a1) and e0 == e1
    heavy = edges_array([(0, 1, 40000.0), (2, 3, 40000.0)])  # test_statevector.cpp:72-80
    assert not oracle.cost_table(4, heavy)[1]


@pytest.mark.parametrize("n,p,pe,budget,seed", [(8, 2, 0.4, 120, 7), (11, 2, 0.3, 200, 1),
                                                (7, 3, 0.6, 90, 5)])
def test_vs_reference_optimize(oracle, ref, n, p, pe, budget, seed):
    e = ref.generate_er(n, pe, seed)
    o0 = ref.optimize(n, e, p, budget, seed, trace=True)
    o1 = oracle.optimize(n, e, p, budget, seed, trace=True)
    assert np.array_equal(o0["trace_x"], o1["trace_x"]) and np.array_equal(o0["trace_f"], o1["trace_f"])
    assert np.array_equal(o0["params"], o1["params"]) and o0["evals"] == o1["evals"]


def test_vs_reference_pipeline_windowed(oracle, ref):
    e = ref.generate_er(120, 0.2, 5)
    kw = dict(qubit_cap=8, top_k=3, layers=1, budget=30, seed=2, path_budget=1e5)
    r0 = ref.run_pipeline(120, e, **kw)
    r1 = oracle.run_pipeline(120, e, **kw)
    assert r0["windowed"] and r1["windowed"]
    assert r0["cut"] == r1["cut"] and r0["assignment"] == r1["assignment"]
    assert r0["leaves"] == r1["leaves"]


def test_vs_reference_partition_modes(oracle, ref):
    e = ref.generate_er(50, 0.2, 1)
    for M, mode in [(1, 0), (3, 0), (7, 0), (7, 1), (24, 0), (49, 0)]:
        assert all(np.array_equal(x, y) if isinstance(x, np.ndarray) else x == y
                   for x, y in zip(ref.partition(50, e, M, mode), oracle.partition(50, e, M, mode)))
    from oracle.refpy import ConfigError, ResourceError
    for lib in (ref, oracle):
        with pytest.raises(ConfigError):
            lib.partition(50, e, 50, 0)
        with pytest.raises(ResourceError):
            lib.partition(50, e, 3, 0, 10)
