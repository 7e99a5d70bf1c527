"""TEST INFRASTRUCTURE ONLY — regenerate tests/golden/ from the reference itself.

Runs the unmodified reference (oracle/_ref/libqcut_ref.so, built by `make -C oracle ref`
from /root/reference/proj/include) and records golden vectors for the hot path:

* config 1 (ER(100,0.1,0), cap 10, p=1, K=4): pipeline cut + assignment, and every
  subgraph's SolveResult;
* run_ansatz amplitudes (sha256 of the raw fp64 bytes) + expectation bits at q=2..20;
* full Nelder-Mead (x, f) trajectories (qaoa.hpp:85-117) for several (graph, p, seed);
* top-K on QAOA plateau states, folded and unfolded;
* level / chained merge results on seeded pools (unit and fractional weights).

Usage:  python oracle/gen_golden.py   (writes tests/golden/golden.json + traces.npz)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.refpy import RefLib, edges_array  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def hx(x: float) -> str:
    return float(x).hex()


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def random_pool(first, last, k, rng):
    pool = []
    for a, b in zip(first, last):
        w = int(b - a + 1)
        reps = set()
        while len(reps) < min(k, 1 << (w - 1)):
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
    return edges_array([(u, v, float(0.1 + rng.uniform())) for u in range(n)
                        for v in range(u + 1, n) if rng.uniform() < p])


def main():
    ref = RefLib()
    os.makedirs(OUT, exist_ok=True)
    gold = {"generator": "oracle/gen_golden.py (reference: oracle/_ref/libqcut_ref.so)"}
    traces = {}

    # ---- config 1 --------------------------------------------------------------------
    e = ref.generate_er(100, 0.1, 0)
    rep = ref.run_pipeline(100, e, qubit_cap=10, top_k=4, layers=1, budget=200, seed=0, workers=1)
    first, last, local_m, inter = ref.partition(100, e, 11, 0, 10)
    subs = []
    for i in range(11):
        a, b = int(first[i]), int(last[i])
        sel = (e["u"] >= a) & (e["v"] <= b)
        le = e[sel].copy()
        le["u"] -= a
        le["v"] -= a
        s = ref.solve_subgraph(b - a + 1, le, top_k=4, layers=1, budget=200, seed=i, fold=True,
                               qubit_cap=10)
        subs.append(dict(n=b - a + 1, m=int(len(le)), expectation=hx(s.expectation),
                         params=[hx(x) for x in s.params[:2]], bits=[int(x) for x in s.bits],
                         probs=[hx(x) for x in s.probs], evals=s.evals))
    gold["config1"] = dict(edges=int(len(e)), edges_sha=sha(e), cut=rep["cut"],
                           assignment=rep["assignment"], leaves=int(rep["leaves"]),
                           inter_edges=int(inter), first=[int(x) for x in first],
                           last=[int(x) for x in last], subgraphs=subs)

    # ---- amplitudes -------------------------------------------------------------------
    amp = []
    for q, pe, seed, p in [(2, 1.0, 0, 1), (5, 0.5, 3, 2), (10, 0.3, 1, 3), (13, 0.3, 2, 2),
                           (14, 0.3, 4, 1), (16, 0.2, 5, 2), (20, 0.1, 6, 1)]:
        ge = ref.generate_er(q, pe, seed)
        rng = np.random.default_rng(seed + 1000 * p)
        g = rng.uniform(0, np.pi, p)
        b = rng.uniform(0, np.pi, p)
        a, ex = ref.run_ansatz(q, ge, g, b)
        amp.append(dict(q=q, p_edge=pe, seed=seed, layers=p, gammas=[hx(x) for x in g],
                        betas=[hx(x) for x in b], amps_sha=sha(a), expectation=hx(ex),
                        norm=hx(ref.norm_sq(a))))
    gold["ansatz"] = amp

    # ---- NM trajectories -------------------------------------------------------------
    tr = []
    for k, (n, pe, p, budget, seed) in enumerate([(2, 1.0, 1, 200, 0), (6, 0.5, 2, 120, 7),
                                                  (10, 0.3, 1, 200, 3), (10, 0.3, 3, 200, 4),
                                                  (12, 0.5, 3, 150, 0)]):
        ge = ref.generate_er(n, pe, seed)
        o = ref.optimize(n, ge, p, budget, seed, trace=True)
        traces[f"x{k}"] = o["trace_x"]
        traces[f"f{k}"] = o["trace_f"]
        tr.append(dict(n=n, p_edge=pe, layers=p, budget=budget, seed=seed, key=k,
                       params=[hx(x) for x in o["params"]], expectation=hx(o["expectation"]),
                       evals=o["evals"]))
    gold["optimize"] = tr

    # ---- top-K on plateau states -----------------------------------------------------
    tk = []
    ge = ref.generate_er(10, 0.1, 0)
    a, _ = ref.run_ansatz(10, ge, [1.1], [0.4])
    for k, fold in [(1, True), (4, True), (37, True), (512, True), (8, False), (1024, False)]:
        bits, probs = ref.top_candidates(a, k, fold)
        tk.append(dict(k=k, fold=fold, bits=[int(x) for x in bits], probs_sha=sha(probs)))
    gold["topk"] = dict(graph=dict(n=10, p=0.1, seed=0), gamma=hx(1.1), beta=hx(0.4), cases=tk)

    # ---- merges ----------------------------------------------------------------------
    mg = []
    rng = np.random.default_rng(7)
    for name, n, edges, M, k in [("er13", 13, ref.generate_er(13, 0.4, 3), 3, 3),
                                 ("er21", 21, ref.generate_er(21, 0.3, 9), 5, 2),
                                 ("w14", 14, weighted(14, 0.5, 4), 4, 2),
                                 ("er400", 400, ref.generate_er(400, 0.1, 0), 21, 2)]:
        first, last, _, _ = ref.partition(n, edges, M)
        pool = random_pool(first, last, k, rng)
        case = dict(name=name, n=n, M=M, edges_sha=sha(edges), pool=pool)
        if name in ("er13", "w14", "er21"):
            for inc in (False, True):
                r = ref.level_merge(n, edges, M, pool, incremental=inc)
                case[f"level_inc{int(inc)}"] = dict(value=hx(r.value),
                                                     assignment="".join(map(str, r.assignment)),
                                                     leaves=int(r.leaves))
        r = ref.chained_merge(n, edges, M, pool)
        case["chained"] = dict(value=hx(r.value), assignment="".join(map(str, r.assignment)),
                               leaves=int(r.leaves))
        if name == "w14":
            case["edges"] = [[int(x["u"]), int(x["v"]), hx(x["w"])] for x in edges]
        mg.append(case)
    gold["merge"] = mg

    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(gold, f, indent=1)
    np.savez_compressed(os.path.join(OUT, "traces.npz"), **traces)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
