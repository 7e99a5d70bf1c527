"""GPU parity: statevector.hpp / qaoa.hpp hot path through the C-ABI vs the oracle.

Bit-exact (==) on the integral-weight path: amplitudes, expectation, probabilities,
top-K bits; mirrors test_statevector.cpp / test_qaoa.cpp and acceptance crit 6.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rand_state(q, seed):
    rng = np.random.default_rng(seed)
    v = rng.normal(size=(1 << q)) + 1j * rng.normal(size=(1 << q))
    return (v / np.sqrt(np.sum(np.abs(v) ** 2))).astype(np.complex128)


def bits_equal(a, b):
    return np.array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64)) or \
        np.array_equal(np.asarray(a), np.asarray(b))


@pytest.mark.parametrize("q,p_edge,seed", [(2, 1.0, 0), (5, 0.5, 3), (10, 0.3, 1), (13, 0.3, 2),
                                           (14, 0.3, 4), (16, 0.2, 5), (20, 0.1, 6)])
@pytest.mark.parametrize("layers", [1, 2, 3])
def test_run_ansatz_bit_exact(engine, oracle, q, p_edge, seed, layers):
    e = oracle.generate_er(q, p_edge, seed)
    rng = np.random.default_rng(seed + 100 * layers)
    g = rng.uniform(0, np.pi, layers)
    b = rng.uniform(0, np.pi, layers)
    a_ref, ex_ref = oracle.run_ansatz(q, e, g, b)
    a_gpu, ex_gpu = engine.run_ansatz(q, e, g, b)
    assert np.array_equal(a_gpu, a_ref)
    assert ex_gpu == ex_ref


def test_ramp_skips_are_exact(engine, oracle):
    # p=1 ramp: beta = 0 (mixer skipped); gamma = 0 (phase skipped)
    e = oracle.generate_er(12, 0.4, 9)
    for g, b in [([np.pi / 2], [0.0]), ([0.0], [0.7]), ([0.0], [0.0])]:
        a_ref, ex_ref = oracle.run_ansatz(12, e, g, b)
        a_gpu, ex_gpu = engine.run_ansatz(12, e, g, b)
        assert np.array_equal(a_gpu, a_ref)
        assert ex_gpu == ex_ref


@pytest.mark.parametrize("q", [1, 3, 8, 12, 13, 15])
def test_layers_on_arbitrary_states(engine, oracle, q):
    e = oracle.generate_er(q, 0.5, q) if q > 1 else np.zeros(0, oracle_edge_dtype())
    s = rand_state(q, 11 + q)
    assert np.array_equal(engine.apply_mixer_layer(s, 0.77), oracle.apply_mixer_layer(s, 0.77))
    assert np.array_equal(engine.apply_cost_layer(s, q, e, 1.3),
                          oracle.apply_cost_layer(s, q, e, 1.3))
    assert engine.expectation(s, q, e) == oracle.expectation(s, q, e)
    assert engine.norm_sq(s) == oracle.norm_sq(s)


def oracle_edge_dtype():
    from oracle.refpy import EDGE_DTYPE
    return EDGE_DTYPE


def test_identities(engine):
    e = [(0, 1), (1, 2), (0, 2)]
    s = rand_state(3, 1)
    assert np.array_equal(engine.apply_cost_layer(s, 3, e, 0.0), s)  # statevector.hpp:149
    assert np.array_equal(engine.apply_mixer_layer(s, 0.0), s)       # statevector.hpp:193
    one = engine.apply_mixer_layer(np.array([1, 0], np.complex128), np.pi / 2)
    assert abs(one[0]) < 1e-12 and abs(one[1] - (-1j)) < 1e-12      # test_statevector.cpp:137
    plus = engine.plus_state(2)
    out = engine.apply_cost_layer(plus, 2, [(0, 1)], np.pi)          # test_statevector.cpp:95
    assert np.allclose(out.real, [0.5, -0.5, -0.5, 0.5], atol=1e-12)


def test_plus_state(engine, oracle):
    for q in (1, 3, 12, 14):
        assert np.array_equal(engine.plus_state(q, 24), oracle.plus_state(q, 24))


@pytest.mark.parametrize("q,k,fold", [(2, 2, True), (2, 4, False), (5, 16, True), (9, 4, True),
                                      (12, 7, False), (14, 8, True), (16, 1500, True),
                                      # register top-K boundary (K <= 32) vs the sort paths
                                      (11, 17, False), (18, 32, True), (18, 33, True)])
def test_top_candidates_random(engine, oracle, q, k, fold):
    s = rand_state(q, q * 7 + k)
    b0, p0 = oracle.top_candidates(s, k, fold)
    b1, p1 = engine.top_candidates(s, k, fold)
    assert np.array_equal(b1, b0)
    assert np.array_equal(p1, p0)


def test_top_candidates_tie_order(engine):
    # test_qaoa.cpp:116-139: folded classes and lexicographic tie order 0,3,2,1
    s = np.sqrt(np.array([0.4, 0.1, 0.1, 0.4])).astype(np.complex128)
    b, p = engine.top_candidates(s, 2, True)
    assert list(b) == [0, 2] and abs(p[0] - 0.8) < 1e-12 and abs(p[1] - 0.2) < 1e-12
    b, _ = engine.top_candidates(s, 4, False)
    assert list(b) == [0, 3, 2, 1]


def test_top_candidates_plateaus(engine, oracle):
    # QAOA states of sparse graphs have huge plateaus of exactly equal probabilities
    e = oracle.generate_er(10, 0.1, 0)
    a, _ = oracle.run_ansatz(10, e, [1.1], [0.4])
    for k in (1, 2, 4, 17, 32, 37, 512):
        b0, p0 = oracle.top_candidates(a, k, True)
        b1, p1 = engine.top_candidates(a, k, True)
        assert np.array_equal(b1, b0) and np.array_equal(p1, p0)


def test_eval_batch_matches_oracle(engine, oracle):
    graphs = [(q, oracle.generate_er(q, 0.3, q)) for q in (4, 9, 14, 15)]
    rng = np.random.default_rng(5)
    idx = np.array([0, 1, 2, 3, 2, 1, 0, 3], np.int32)
    params = rng.uniform(0, np.pi, (len(idx), 4))
    out = engine.eval_batch(graphs, 2, idx, params)
    for k, i in enumerate(idx):
        n, e = graphs[i]
        _, ex = oracle.run_ansatz(n, e, params[k, :2], params[k, 2:], want_amps=False)
        assert out[k] == ex


def test_errors_map_to_reference_types(engine):
    from paper_2603_26232_b200 import ConfigError, ResourceError
    with pytest.raises(ConfigError):
        engine.top_candidates(rand_state(3, 0), 5, True)  # > 4 folded classes
    with pytest.raises(ConfigError):
        engine.solve_subgraph(0, [])
    with pytest.raises(ResourceError):
        engine.solve_subgraph(21, [(0, 20)])  # default cap 20 (test_qaoa.cpp:243-254)
    with pytest.raises(ConfigError):
        engine.run_ansatz(3, [(0, 0)], [0.1], [0.1])  # self-loop


@pytest.mark.parametrize("n", [3, 40000])  # bitset path (n <= ~32k) and hash-set path
def test_duplicate_edges_rejected_like_add_edge(engine, n):
    """graph.hpp:37-50: a repeated pair (either orientation) is a config_error."""
    from paper_2603_26232_b200 import ConfigError
    dup = [(0, 1, 1.0), (1, 2, 1.0), (1, 0, 1.0)]
    with pytest.raises(ConfigError):
        if n <= 24:
            engine.cost_table(n, dup)
        else:  # the pipeline validates the whole graph before partitioning
            engine.run_pipeline(n, dup, qubit_cap=20, top_k=1, layers=1, budget=1)
    if n == 3:
        out, integral, mx = engine.cost_table(n, [(0, 1, 1.0), (1, 2, 1.0), (0, 2, 1.0)])
        assert integral and mx == 2.0


def _frac_graph(oracle, q, kind, seed):
    rng = np.random.default_rng(seed)
    e = oracle.generate_er(q, 0.3, seed).copy()
    if kind == "real":
        e["w"] = rng.uniform(0.1, 1.1, len(e))
    elif kind == "quarter":  # dyadic: every cut value exact, few distinct
        e["w"] = rng.integers(1, 11, len(e)) / 4.0
    elif kind == "tenth":  # decimal: edge-order rounding, a few thousand distinct values
        e["w"] = rng.integers(1, 11, len(e)) / 10.0
    else:  # "heavy": integral but total > 65535 (statevector.hpp:89, the values path)
        e["w"] = rng.integers(1000, 9000, len(e)).astype(np.float64)
    return e


def _ansatz_both(engine, oracle, q, e, layers, seed):
    rng = np.random.default_rng(seed + 7)
    g = rng.uniform(0.2, np.pi, layers)
    b = rng.uniform(0.2, np.pi, layers)
    a0, x0 = oracle.run_ansatz(q, e, g, b, threads=max(1, min(32, __import__("os").cpu_count() or 1)))
    a1, x1 = engine.run_ansatz(q, e, g, b)
    got = engine.eval_batch([(q, e)], layers, np.zeros(1, np.int32), np.concatenate([g, b])[None, :])
    return a0, x0, a1, x1, got[0]


@pytest.mark.parametrize("q,layers,kind", [(10, 1, "real"), (14, 2, "real"), (17, 2, "real"),
                                           (20, 2, "quarter"), (20, 1, "tenth"), (22, 1, "quarter"),
                                           (24, 1, "tenth"), (18, 2, "heavy")])
def test_fractional_weights_bit_exact(engine, oracle, q, layers, kind):
    """Non-integral tables take statevector.hpp:162-164: amps[z] *= std::polar(1, -gamma *
    val[z]) with glibc's sin/cos. The engine finds the table's distinct values on the device,
    the host evaluates std::polar for each (the reference's own operation and libm), and the
    passes apply them through the LUT path; the expectation reads the fp64 values. Every
    table with <= 65,535 distinct values is bit-exact: all tables up to 17 qubits, dyadic
    and decimal weights, integral tables whose total exceeds 65,535."""
    e = _frac_graph(oracle, q, kind, q)
    a0, x0, a1, x1, xe = _ansatz_both(engine, oracle, q, e, layers, q)
    assert np.array_equal(a1, a0)
    assert x1 == x0 and xe == x0


@pytest.mark.parametrize("q,layers", [(20, 2), (22, 1)])
def test_fractional_weights_within_tolerance(engine, oracle, q, layers):
    """Random real weights on 20+ qubits give more than 65,535 distinct cut values: the
    device evaluates sin/cos itself (glibc's are not correctly rounded in ~0.13% of
    arguments), held to the north-star fp64 tolerance (1e-10 relative)."""
    e = _frac_graph(oracle, q, "real", q)
    a0, x0, a1, x1, xe = _ansatz_both(engine, oracle, q, e, layers, q)
    assert abs(x1 - x0) <= 1e-10 * abs(x0)
    assert np.max(np.abs(a1 - a0)) <= 1e-10 * np.max(np.abs(a0))
    assert abs(xe - x0) <= 1e-10 * abs(x0)


@pytest.mark.parametrize("q", [14, 20])
def test_identity_layers_in_multipass_chains(engine, oracle, q):
    """gamma == 0 (no phase, statevector.hpp:149) and beta == 0 (identity mixer, :193) in
    a middle layer: the streaming passes skip those tiles (the refill path without work)."""
    e = oracle.generate_er(q, 0.3, q + 1)
    for g, b in [([0.7, 0.0, 1.1], [0.3, 0.0, 0.9]), ([0.0, 0.5], [0.0, 0.4])]:
        a0, x0 = oracle.run_ansatz(q, e, g, b)
        a1, x1 = engine.run_ansatz(q, e, g, b)
        assert np.array_equal(a1, a0) and x1 == x0


@pytest.mark.parametrize("env", [{"QCG_PASS_B": "tma"},
                                 {"QCG_PASS_B": "tma", "QCG_B5_STORE": "stg"},
                                 {"QCG_PASS_B": "v4"},
                                 {"QCG_GRAPH": "0", "QCG_PASS_A": "v4"},
                                 {"QCG_PASS_B": "tma", "QCG_B5_EARLY": "1"},
                                 {"QCG_PASS_B": "tma", "QCG_B5_EARLY": "0"}],
                         ids=["tma-tensor-store", "tma-register-store", "v4", "direct-launch-v4-pass-a",
                              "tma-early-refill", "tma-no-early-refill"])
def test_pass_b_kernel_variants(env):
    """Every pass B kernel (qc_pass.cu: TMA boxes with tensor or register stores, v4
    per-thread gathers), and the chain without CUDA-graph capture and with the v4 pass A,
    bit-exact at all geometry classes (tests/gpu_pass_variants.py)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, os.path.join(here, "gpu_pass_variants.py")],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout[-2000:] + r.stderr[-2000:]


def test_split_launches():
    """Passes split into several persistent launches (slot offsets in the tensor maps):
    tests/gpu_many_slots.py with one chunk and the TMA pass B forced."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    env = {**os.environ, "QCG_CHUNKS": "1", "QCG_PASS_B": "tma"}
    r = subprocess.run([sys.executable, os.path.join(here, "gpu_many_slots.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout[-2000:] + r.stderr[-2000:]


def test_graph_replay_across_graphs_and_shapes(engine, oracle):
    """Chunk steps replay captured CUDA graphs keyed by shape and buffers; the graphs
    evaluated travel in the staging copy. Alternate different graphs of the same shape
    and a different shape on one engine: every result must match the oracle bit for bit."""
    rng = np.random.default_rng(7)
    ga = oracle.generate_er(16, 0.3, 1)
    gb = oracle.generate_er(16, 0.5, 2)
    gc = oracle.generate_er(18, 0.3, 3)
    for q, e in [(16, ga), (16, gb), (18, gc), (16, ga), (16, gb), (18, gc)]:
        prm = rng.uniform(0.1, 3.0, size=(3, 4))
        got = engine.eval_batch([(q, e)], 2, np.zeros(3, np.int32), prm)
        for k in range(3):
            x0 = oracle.run_ansatz(q, e, prm[k, :2], prm[k, 2:], want_amps=False)[1]
            assert got[k] == x0, (q, k, got[k], x0)


# ---- CostTable (statevector.hpp:75-111), direct ---------------------------------------
@pytest.mark.parametrize("case", ["er20", "weighted_int18", "over_65535", "fractional16"])
def test_cost_table_matches_reference(engine, oracle, case):
    """The device cut table (k_levels) against the reference's CostTable on the same graph:
    the integral uint16 path (q=20 ER; integer weights), the total-weight > 65535 fallback
    to the double table (statevector.hpp:84-89; test_statevector.cpp:72-80), and
    fractional weights summed in edge-list order (statevector.hpp:101-110). Bit-exact."""
    rng = np.random.default_rng(20)
    if case == "er20":
        n, e = 20, oracle.generate_er(20, 0.3, 2)
    elif case == "weighted_int18":
        n = 18
        e = [(u, v, float(rng.integers(1, 50))) for u in range(n) for v in range(u + 1, n)
             if rng.random() < 0.3]
    elif case == "over_65535":
        n = 16
        e = [(u, v, float(rng.integers(900, 1400))) for u in range(n) for v in range(u + 1, n)]
        assert sum(w for _, _, w in e) > 65535
    else:
        n = 16
        e = [(u, v, 0.1 + rng.random()) for u in range(n) for v in range(u + 1, n)
             if rng.random() < 0.4]
    want, wint, wmax = oracle.cost_table(n, e)
    got, gint, gmax = engine.cost_table(n, e)
    assert gint == wint == (case in ("er20", "weighted_int18"))
    assert gmax == wmax
    assert np.array_equal(got, want)


def _blocked_sum_ref(f):
    """statevector.hpp:48-65 blocked_sum: sequential sums over 4096-blocks, then the block
    partials in order (np.add.accumulate is strictly left to right in float64)."""
    parts = [np.add.accumulate(np.concatenate(([0.0], f[i:i + 4096])))[-1] for i in range(0, len(f), 4096)]
    return np.add.accumulate(np.concatenate(([0.0], parts)))[-1]


@pytest.mark.parametrize("q,kind", [(13, "ties"), (14, "range"), (15, "crossings"), (16, "mixed"),
                                    (14, "zeros")])
def test_blocked_sum_adversarial(engine, q, kind):
    """The segmented exact block sum (k_blocksum_seg) against the sequential reference on
    inputs built to break its fast path: exact ties at acc's half-ulp (1 + 2^-53 rounds to
    even), a 2^-60..2^10 dynamic range, values that cross a binade every few terms, runs of
    zeros and subnormal-adjacent magnitudes. |a|^2 = a.x^2 + a.y^2 is formed exactly as the
    kernel forms it, then summed in the reference's order."""
    rng = np.random.default_rng(q)
    n = 1 << q
    if kind == "ties":  # each block: 1.0, then 2^-53 (ties at acc's half-ulp) and 5 * 2^-54
        re = np.full(n, 2.0 ** -27)
        im = np.where(rng.random(n) < 0.6, 2.0 ** -27, 2.0 ** -26)
        re[::4096] = 1.0
        im[::4096] = 0.0
    elif kind == "range":
        re = np.ldexp(rng.random(n) + 0.5, rng.integers(-30, 5, n))
        im = np.ldexp(rng.random(n) + 0.5, rng.integers(-30, 5, n))
    elif kind == "crossings":  # geometric growth: the running sum doubles every few terms
        k = np.arange(n) % 4096
        re = np.sqrt(np.ldexp(1.0, (k // 3) % 40 - 20)) * (1 + rng.random(n) * 1e-3)
        im = np.zeros(n)
    elif kind == "zeros":
        re = rng.standard_normal(n)
        im = rng.standard_normal(n)
        re[rng.random(n) < 0.7] = 0.0
        im[re == 0.0] = 0.0
        re[:5000] = 0.0
        im[:5000] = 0.0
    else:
        re = rng.standard_normal(n) * np.ldexp(1.0, rng.integers(-8, 8, n))
        im = rng.standard_normal(n)
        im[rng.random(n) < 0.1] = 0.0
    a = (re + 1j * im).astype(np.complex128)
    f = a.real * a.real + a.imag * a.imag  # two rounded products, one rounded add
    got = engine.norm_sq(a)
    want = _blocked_sum_ref(f)
    assert got == want, (kind, got, want)


@pytest.mark.parametrize("q,kind", [(24, "ties"), (24, "range"), (25, "crossings"), (24, "smooth")])
def test_partial_sum_adversarial(engine, q, kind):
    """The in-order sum over the block partials (statevector.hpp:61-62; 4096 partials at
    q=24, 8192 at q=25 = two 4096-chunks carried) runs the segmented exact sum. Each block
    holds one nonzero amplitude at its first index, so its partial is exactly that f value
    and the partial sequence is chosen freely: ties at acc's half-ulp, a wide dynamic range,
    binade crossings every few partials, and smooth data (the fast path)."""
    rng = np.random.default_rng(q + len(kind))
    n, nbl = 1 << q, 1 << (q - 12)
    if kind == "ties":
        x = np.full(nbl, 2.0 ** -27)
        y = np.where(rng.random(nbl) < 0.6, 2.0 ** -27, 2.0 ** -26)
        x[::512] = 1.0
        y[::512] = 0.0
    elif kind == "range":
        x = np.ldexp(rng.random(nbl) + 0.5, rng.integers(-40, 10, nbl))
        y = np.ldexp(rng.random(nbl) + 0.5, rng.integers(-40, 10, nbl))
    elif kind == "crossings":
        k = np.arange(nbl)
        x = np.sqrt(np.ldexp(1.0, (k // 2) % 50 - 25)) * (1 + rng.random(nbl) * 1e-3)
        y = np.zeros(nbl)
    else:
        x = 1e-3 * (1 + rng.random(nbl))
        y = 1e-3 * rng.random(nbl)
    a = np.zeros(n, np.complex128)
    a[:: 4096] = x + 1j * y
    v = x * x + y * y
    want = np.add.accumulate(np.concatenate(([0.0], v)))[-1]
    got = engine.norm_sq(a)
    assert got == want, (kind, got, want)
