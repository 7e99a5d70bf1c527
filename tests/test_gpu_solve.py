"""GPU parity: optimize_parameters / solve_subgraph / merges / pipeline vs the oracle.

The lockstep ask/tell Nelder-Mead must reproduce every (x, f) of the reference
trajectory; SolveResults, merge results and the config-1 cut must be identical.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def oracle_trace(oracle, n, e, p, budget, seed):
    return oracle.optimize(n, e, p, budget, seed, trace=True)


@pytest.mark.parametrize("n,pe,p,budget,seed", [(2, 1.0, 1, 200, 0), (6, 0.5, 2, 120, 7),
                                                (10, 0.3, 1, 200, 3), (10, 0.3, 3, 200, 4),
                                                (12, 0.5, 3, 150, 0), (15, 0.3, 2, 60, 1)])
def test_optimize_trajectory_bit_exact(engine, oracle, n, pe, p, budget, seed):
    e = oracle.generate_er(n, pe, seed)
    ref = oracle_trace(oracle, n, e, p, budget, seed)
    out = engine.optimize_batch([(n, e)], p, budget, [seed], trace=True)
    L = len(ref["trace_f"])
    assert L == budget
    assert np.array_equal(out["trace_x"][0, :L], ref["trace_x"])
    assert np.array_equal(out["trace_f"][0, :L], ref["trace_f"])
    assert np.array_equal(out["params"][0], ref["params"])
    assert out["expectation"][0] == ref["expectation"]
    assert out["evals"][0] == ref["evals"]


def test_optimize_batch_is_placement_independent(engine, oracle):
    graphs = [(10, oracle.generate_er(10, 0.3, s)) for s in range(5)]
    seeds = [11, 12, 13, 14, 15]
    batch = engine.optimize_batch(graphs, 2, 80, seeds)
    for i, (n, e) in enumerate(graphs):
        one = engine.optimize_batch([(n, e)], 2, 80, [seeds[i]])
        assert np.array_equal(batch["params"][i], one["params"][0])
        assert batch["expectation"][i] == one["expectation"][0]


def test_tiny_budgets(engine, oracle):
    e = oracle.generate_er(6, 0.5, 1)
    for budget in (1, 3, 10):
        ref = oracle.optimize(6, e, 2, budget, 0)
        out = engine.optimize_batch([(6, e)], 2, budget, [0])
        assert out["evals"][0] == ref["evals"] and np.array_equal(out["params"][0], ref["params"])


def test_edgeless_keeps_ramp(engine):
    out = engine.optimize_batch([(3, [])], 2, 50, [0])
    g, b = engine.linear_ramp(2)
    assert out["expectation"][0] == 0.0
    assert np.array_equal(out["params"][0], np.concatenate([g, b]))


@pytest.mark.parametrize("n,pe,k,layers,fold", [(2, 1.0, 1, 1, True), (7, 0.5, 3, 3, True),
                                                (10, 0.2, 4, 1, True), (9, 0.4, 5, 2, False),
                                                (14, 0.2, 4, 1, True)])
def test_solve_subgraph_matches(engine, oracle, n, pe, k, layers, fold):
    e = oracle.generate_er(n, pe, n)
    budget = 100 if n >= 14 else 200
    ref = oracle.solve_subgraph(n, e, top_k=k, layers=layers, budget=budget, seed=n, fold=fold)
    got = engine.solve_subgraph(n, e, top_k=k, layers=layers, budget=budget, seed=n, fold=fold)
    assert np.array_equal(got.bits, ref.bits)
    assert np.array_equal(got.probs, ref.probs)
    assert np.array_equal(got.params, ref.params[: 2 * layers])
    assert got.expectation == ref.expectation and got.evals == ref.evals


def test_single_edge_solve(engine):
    r = engine.solve_subgraph(2, [(0, 1)], top_k=1, layers=1, budget=200)
    assert list(r.bits) == [2] and r.probs[0] >= 0.99 and r.expectation >= 0.99


# ---- merge ---------------------------------------------------------------------------
def full_pool(first, last):
    pool = []
    for a, b in zip(first, last):
        w = b - a + 1
        pool.append((w, [x for rep in range(0, 1 << w, 2) for x in (rep, rep ^ ((1 << w) - 1))]))
    return pool


def random_pool(first, last, k, rng):
    pool = []
    for a, b in zip(first, last):
        w = b - a + 1
        reps = set()
        while len(reps) < k:
            reps.add(int(rng.integers(0, 1 << w)) & ~1)
        bits = []
        for r in sorted(reps):
            for x in (r, r ^ ((1 << w) - 1)):
                if x not in bits:
                    bits.append(x)
        pool.append((w, bits))
    return pool


def weighted(n, p, seed):
    rng = np.random.default_rng(seed)
    out = []
    for u in range(n):
        for v in range(u + 1, n):
            if rng.uniform() < p:
                out.append((u, v, 0.1 + rng.uniform()))
    return out


def check_merge(engine, oracle, n, e, M, pool, **kw):
    first, last, _, _ = oracle.partition(n, e, M)
    ref = oracle.level_merge(n, e, M, pool, **kw)
    got = engine.level_merge(n, e, (first, last), pool, **kw)
    assert got.best_value == ref.value
    assert np.array_equal(got.assignment, ref.assignment)
    assert got.candidates_evaluated == ref.leaves


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("M", [2, 3])
def test_exhaustive_pool_is_brute_force(engine, oracle, seed, M):
    n = 10
    e = oracle.generate_er(n, 0.5, seed)
    first, last, _, _ = oracle.partition(n, e, M)
    pool = full_pool(first, last)
    for halve in (False, True):
        check_merge(engine, oracle, n, e, M, pool, halve=halve)


@pytest.mark.parametrize("incremental", [False, True])
def test_weighted_merge_exact_order(engine, oracle, incremental):
    from oracle.refpy import edges_array
    e = edges_array(weighted(14, 0.5, 4))
    rng = np.random.default_rng(5)
    first, last, _, _ = oracle.partition(14, e, 4)
    pool = random_pool(first, last, 2, rng)
    check_merge(engine, oracle, 14, e, 4, pool, incremental=incremental)


def test_merge_invariance_and_counts(engine, oracle):
    rng = np.random.default_rng(7)
    e = oracle.generate_er(13, 0.4, 3)
    first, last, _, _ = oracle.partition(13, e, 3)
    pool = random_pool(first, last, 3, rng)
    for level in (1, 2, 3):
        for inc in (False, True):
            for halve in (False, True):
                check_merge(engine, oracle, 13, e, 3, pool, start_level=level, incremental=inc,
                            halve=halve)


def test_chained_merge_matches(engine, oracle):
    rng = np.random.default_rng(17)
    e = oracle.generate_er(21, 0.3, 9)
    first, last, _, _ = oracle.partition(21, e, 5)
    pool = random_pool(first, last, 2, rng)
    for window in (0, 1, 2, 5):
        ref = oracle.chained_merge(21, e, 5, pool, window=window)
        got = engine.chained_merge(21, e, (first, last), pool, window=window)
        assert got.best_value == ref.value
        assert np.array_equal(got.assignment, ref.assignment)
        assert got.candidates_evaluated == ref.leaves


def test_chained_merge_windowed_large(engine, oracle):
    rng = np.random.default_rng(3)
    n, M = 400, 21
    e = oracle.generate_er(n, 0.1, 0)
    first, last, _, _ = oracle.partition(n, e, M)
    pool = random_pool(first, last, 4, rng)
    ref = oracle.chained_merge(n, e, M, pool)
    got = engine.chained_merge(n, e, (first, last), pool)
    assert got.best_value == ref.value
    assert np.array_equal(got.assignment, ref.assignment)
    assert got.candidates_evaluated == ref.leaves


def test_merge_errors(engine, oracle):
    from paper_2603_26232_b200 import ConfigError, ResourceError
    e = [(0, 1), (1, 2)]
    with pytest.raises(ConfigError):  # dead end (test_merge.cpp:259-266)
        engine.level_merge(3, e, ([0, 1], [1, 2]), [(2, [3]), (2, [0])])
    e10 = [(i, i + 1) for i in range(9)]
    first, last, _, _ = oracle.partition(10, e10, 3)
    pool = full_pool(first, last)
    paths = 2 * 16 * 16 * 16 / 2 / 2  # estimate_paths
    with pytest.raises(ResourceError):
        engine.level_merge(10, e10, (first, last), pool, path_budget=float(len(pool[0][1]) *
                           (len(pool[1][1]) / 2) * (len(pool[2][1]) / 2) - 1))
    del paths


# ---- pipeline (config 1) ----------------------------------------------------------------
def test_config1_pipeline(engine, oracle):
    e = oracle.generate_er(100, 0.1, 0)
    rep = engine.run_pipeline(100, e, qubit_cap=10, top_k=4, layers=1, budget=200, seed=0)
    assert rep.cut == 296.0  # SURVEY Appendix E (reference canonical build)
    assert rep.assignment == ("0001001001111010100000001001101111111111001010001010100001010101"
                              "101110001111110110000000101100001011")
    assert rep.candidates_evaluated == 8388608
    assert rep.subgraphs == 11 and not rep.windowed


# ---- multi-GPU record path, emulated in one process -------------------------------------
@pytest.mark.parametrize("shards", [2, 3, 8])
def test_sharded_records_equal_single_gpu(engine, oracle, shards):
    from paper_2603_26232_b200 import kcap_for
    e = oracle.generate_er(100, 0.1, 0)
    cfg = dict(qubit_cap=10, top_k=4, layers=1, budget=200, seed=0)
    M = engine.subgraph_count(100, e, **cfg)
    rb = engine.record_bytes(kcap_for(10, 4), 1)
    recs = []
    for r in range(shards):
        b, en = engine.shard_range(M, r, shards)
        recs.append(engine.shard_solve(100, e, b, en, rb, **cfg))
    rep = engine.merge_records(100, e, np.concatenate(recs), M, **cfg)
    single = engine.run_pipeline(100, e, **cfg)
    assert rep.cut == single.cut == 296.0
    assert rep.assignment == single.assignment
    assert rep.candidates_evaluated == single.candidates_evaluated
    assert rep.evals == single.evals == 11 * 200


def test_pipeline_windowed_matches_oracle(engine, oracle):
    e = oracle.generate_er(120, 0.2, 5)
    kw = dict(qubit_cap=8, top_k=3, layers=1, budget=30, seed=2, path_budget=1e5)
    ref = oracle.run_pipeline(120, e, **kw)
    got = engine.run_pipeline(120, e, **kw)
    assert ref["windowed"] and got.windowed
    assert got.cut == ref["cut"] and got.assignment == ref["assignment"]
    assert got.candidates_evaluated == ref["leaves"]


def test_pipeline_c2_shape_matches_oracle(engine, oracle):
    """config-2 shape (400 vertices, 20-qubit pieces) with a short NM budget so the
    oracle finishes quickly; the full budget runs in bench.py."""
    e = oracle.generate_er(400, 0.1, 0)
    kw = dict(qubit_cap=20, top_k=2, layers=2, budget=8, seed=0)
    ref = oracle.run_pipeline(400, e, workers=os.cpu_count() or 1, **kw)
    got = engine.run_pipeline(400, e, **kw)
    assert got.cut == ref["cut"] and got.assignment == ref["assignment"]
    assert got.candidates_evaluated == ref["leaves"]
    assert np.array_equal(np.array([got.evals]), np.array([int(ref["sub_evals"].sum())]))


def test_sweep_rows_match_oracle_pipeline(engine, oracle):
    """paper_2603_26232_b200.sweep on the GPU: one CSV row per grid point, in the CLI's
    axis order, with the cut the oracle's run_pipeline finds for the same instance."""
    import io
    from paper_2603_26232_b200.sweep import run_sweep
    grid = {"qubits": 8, "layers": 1, "budget": 20, "n": [40], "p": [0.2, 0.4], "seed": [3],
            "top_k": [2, 3]}
    out = io.StringIO()
    assert run_sweep(grid, out, engine=engine) == 4
    rows = [r.split(",") for r in out.getvalue().splitlines()[1:]]
    for row, (p, k) in zip(rows, [(0.2, 2), (0.2, 3), (0.4, 2), (0.4, 3)]):
        e = oracle.generate_er(40, p, 3)
        ref = oracle.run_pipeline(40, e, qubit_cap=8, top_k=k, layers=1, budget=20, seed=0)
        assert row[0] == "40" and float(row[1]) == p and row[4] == str(k)
        assert float(row[6]) == ref["cut"]
