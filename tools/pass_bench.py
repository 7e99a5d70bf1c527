#!/usr/bin/env python3
"""Microbenchmark of the statevector pass kernels: one launch chain over S slots of
q-qubit subgraphs (ER(q, p_edge)), p layers, timed per kernel with CUDA events on the
engine stream (qc_engine_profile). Prints per-kernel us/launch and algorithmic GB/s.

  python tools/pass_bench.py --q 20 --slots 21 --layers 2 --reps 20
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_26232_b200 import Engine, generate_er  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--q", type=int, default=20)
    ap.add_argument("--slots", type=int, default=21)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--p-edge", type=float, default=0.1)
    ap.add_argument("--no-phase", action="store_true", help="gamma = 0: pass A without the phase")
    ap.add_argument("--precision", type=int, default=64, choices=(64, 32))
    ap.add_argument("--per-launch", action="store_true",
                    help="also report pass_low us per rep (spread of a sporadic slow run)")
    ap.add_argument("--lib", default="", help="load this libqcgpu build instead (A/B runs)")
    a = ap.parse_args()
    if a.lib:
        import paper_2603_26232_b200 as pkg
        pkg._LIB = pkg.load_library(a.lib)
    eng = Engine(0)
    if a.precision == 32:
        eng.set_precision(32)
    graphs = [(a.q, generate_er(a.q, max(a.p_edge, 0.2), 100 + i)) for i in range(a.slots)]
    rng = np.random.default_rng(0)
    idx = np.arange(a.slots, dtype=np.int32)
    prm = rng.uniform(0.1, 3.0, size=(a.slots, 2 * a.layers))
    if a.no_phase:
        prm[:, :a.layers] = 0.0
    ref = eng.eval_batch(graphs, a.layers, idx, prm)  # warm-up (+ first-touch)
    per = []
    if a.per_launch:
        for _ in range(a.reps):
            eng.profile(True)
            eng.eval_batch(graphs, a.layers, idx, prm)
            v = eng.profile_read()["pass_low"]
            per.append(round(1e3 * v["ms"] / max(v["launches"], 1), 1))
    eng.profile(True)
    for _ in range(a.reps):
        out = eng.eval_batch(graphs, a.layers, idx, prm)
        assert os.environ.get("QCG_PA_DBG") or a.precision == 32 or np.array_equal(out, ref)
    prof = eng.profile_read()
    res = {}
    for k, v in prof.items():
        if v["launches"]:
            us = 1e3 * v["ms"] / v["launches"]
            res[k] = dict(launches=v["launches"], us=round(us, 2),
                          GBs=round(v["bytes"] / (v["ms"] * 1e-3) / 1e9, 1))
    print(json.dumps(dict(q=a.q, slots=a.slots, layers=a.layers,
                          impl=os.environ.get("QCG_PASS", "4"), kernels=res,
                          pass_low_launch_us=per or None)))


if __name__ == "__main__":
    main()
