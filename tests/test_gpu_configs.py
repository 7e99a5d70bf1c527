"""GPU parity at the benchmarked configurations, against the reference build itself
(oracle/_ref: the unmodified qcut headers; libqcut_ref26.so for 26-qubit pieces).

SURVEY 8(c) parity plan: configs 3-5 are too large to solve end to end on the CPU inside a
test, so sampled subgraphs of the real instance get full solves (the reference's own
partition, the pipeline's per-index options: seed = base + idx, top_k clamp) and every
SolveResult field must be identical: top-K bits and probabilities, packed params,
expectation, evals. Config 2 (the bench workload) runs end to end at the full NM budget.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CORES = max(1, os.cpu_count() or 1)


def _ref(cap26=False):
    from oracle.refpy import RefLib, ref_available
    if not ref_available(cap26):
        pytest.skip("reference build (oracle/_ref) not present")
    return RefLib(cap26=cap26)


def _gpu_solves(engine, n, edges, M, indices, **cfg):
    """The product's solves of pipeline subgraphs `indices` (pipeline.hpp:239-263 options)."""
    from paper_2603_26232_b200 import partition_chain
    P = partition_chain(n, edges, M, 0, cfg["qubit_cap"])
    graphs, opts = [], []
    for idx in indices:
        nl, le = P.local[idx]
        classes = 1 << (nl - 1)
        k = classes if cfg["top_k"] == 0 else min(classes, cfg["top_k"])
        graphs.append((nl, le))
        opts.append(dict(top_k=k, layers=cfg["layers"], budget=cfg["budget"],
                         seed=cfg.get("seed", 0) + idx, qubit_cap=cfg["qubit_cap"]))
    return engine.solve_batch(graphs, opts)


def _assert_same(got, ref, layers):
    assert got.width == ref.width
    assert np.array_equal(got.bits, ref.bits)
    assert np.array_equal(got.probs, ref.probs)  # float64 bit equality
    assert np.array_equal(got.params[: 2 * layers], ref.params[: 2 * layers])
    assert got.expectation == ref.expectation
    assert got.evals == ref.evals


def _check_sampled(engine, ref, n, edges, M, indices, **cfg):
    slots = len(indices)
    threads = max(1, CORES // slots)
    want, secs = ref.solve_stage(n, edges, M, indices, cfg["top_k"], cfg["layers"], cfg["budget"],
                                 seed=cfg.get("seed", 0), slots=slots, threads=threads,
                                 qubit_cap=cfg["qubit_cap"])
    got = _gpu_solves(engine, n, edges, M, indices, **cfg)
    for i, (g, r) in enumerate(zip(got, want)):
        assert r.evals == cfg["budget"]
        _assert_same(g, r, cfg["layers"])
    return secs


def test_c2_full_budget_pipeline_matches_reference(engine):
    """BASELINE config 2, the bench workload, at NM budget 200: the reference's stock
    run_pipeline (cut, assignment, leaves, per-subgraph expectation/evals) and every
    SolveResult of its QAOA stage against the resident pipeline session bench.py times."""
    from paper_2603_26232_b200 import generate_er
    ref = _ref()
    n, cfg = 400, dict(qubit_cap=20, top_k=2, layers=2, budget=200, seed=0)
    e = generate_er(n, 0.1, 0)
    stock = ref.run_pipeline(n, e, workers=CORES, **cfg)
    sess = engine.prepare_pipeline(n, e, **cfg)
    rep = sess.execute()
    assert rep.cut == stock["cut"]
    assert rep.assignment == stock["assignment"]
    assert rep.candidates_evaluated == stock["leaves"]
    M = stock["subgraphs"]
    assert rep.subgraphs == M == 21
    recs = sess.records()
    assert [r.expectation for r in recs] == list(stock["sub_expectation"])
    assert [r.evals for r in recs] == list(stock["sub_evals"])
    want, _ = ref.solve_stage(n, e, M, list(range(M)), cfg["top_k"], cfg["layers"],
                              cfg["budget"], slots=min(CORES, M), threads=1,
                              qubit_cap=cfg["qubit_cap"])
    for g, r in zip(recs, want):
        _assert_same(g, r, cfg["layers"])


def test_c3_sampled_full_budget(engine):
    """Config 3: weighted random 3-regular n=1000 (integer weights U{1..10}, the exact
    integral-LUT path), cap 24 -> 44 pieces; two 24-qubit pieces and the 11-qubit tail,
    budget 200."""
    from paper_2603_26232_b200 import generate_regular
    ref = _ref()
    e = generate_regular(1000, 3, 0, 1, 10)
    cfg = dict(qubit_cap=24, top_k=2, layers=1, budget=200, seed=0)
    _check_sampled(engine, ref, 1000, e, 44, [0, 21, 43], **cfg)


@pytest.mark.parametrize("scale", [4.0, 10.0])
def test_c3_fractional_variant_sampled(engine, scale):
    """Config 3 with fractional weights U{1..10}/4 (dyadic) and U{1..10}/10 (decimal): the
    non-integral cost tables (statevector.hpp:162-164, per-amplitude std::polar in the
    reference). Two 24-qubit pieces and the tail, NM budget 60: every SolveResult field
    identical to the reference build's."""
    from paper_2603_26232_b200 import generate_regular
    ref = _ref()
    e = generate_regular(1000, 3, 0, 1, 10).copy()
    e["w"] = e["w"] / scale
    cfg = dict(qubit_cap=24, top_k=2, layers=1, budget=60, seed=0)
    _check_sampled(engine, ref, 1000, e, 44, [0, 21, 43], **cfg)


def test_c4_sampled_full_budget(engine):
    """Config 4: ER(10000, 0.1, 0), cap 20 -> 527 pieces; four pieces incl. the 6-vertex
    tail, budget 200, K=8 (the top of the config-4 K sweep)."""
    from paper_2603_26232_b200 import generate_er
    ref = _ref()
    e = generate_er(10000, 0.1, 0)
    cfg = dict(qubit_cap=20, top_k=8, layers=1, budget=200, seed=0)
    _check_sampled(engine, ref, 10000, e, 527, [0, 175, 350, 526], **cfg)


def test_c5_sampled_26_qubits(engine):
    """Config 5: ER(16000, 0.1, 0), cap 26 -> 640 pieces; two 26-qubit pieces (1 GiB fp64
    states on the CPU) at budget 40 against the 26-qubit reference build."""
    from paper_2603_26232_b200 import generate_er
    ref = _ref(cap26=True)
    e = generate_er(16000, 0.1, 0)
    cfg = dict(qubit_cap=26, top_k=2, layers=1, budget=40, seed=0)
    _check_sampled(engine, ref, 16000, e, 640, [0, 320], **cfg)


@pytest.mark.parametrize("n,p", [(1500, 0.05), (2000, 0.1)])
def test_level_merge_long_chain_top1(engine, n, p):
    """BASELINE configs[3] K sweep, K=1: every pool holds one class (b, ~b), so only two
    compatible chains exist and the auto mode picks the level merge over ALL M levels
    (79 / 106 > the search's 64-level local stacks: the long-window path). Cut,
    assignment and leaf count against the reference's stock run_pipeline."""
    from paper_2603_26232_b200 import generate_er
    ref = _ref()
    e = generate_er(n, p, 0)
    cfg = dict(qubit_cap=20, top_k=1, layers=1, budget=4, seed=0)
    stock = ref.run_pipeline(n, e, workers=CORES, **cfg)
    rep = engine.run_pipeline(n, e, **cfg)
    assert rep.subgraphs == stock["subgraphs"] > 64
    assert rep.cut == stock["cut"]
    assert rep.assignment == stock["assignment"]
    assert rep.candidates_evaluated == stock["leaves"]
