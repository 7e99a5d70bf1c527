#!/usr/bin/env python3
"""One pipeline solve of a bench workload with the bench's roofline-step launch shape
(QCG_CHUNKS=1: every pass launch covers all slots), at a small NM budget (the per-launch
shape does not depend on the budget). Prints the engine's algorithmic bytes per launch
per kernel kind (CUDA-event profile of every launch). Run under ncu by
tools/ncu_traffic.py, which pairs these with ncu's DRAM bytes of the same kernels."""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("QCG_CHUNKS", "1")

import bench  # noqa: E402  (workload table and generators)
from paper_2603_26232_b200 import Engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--precision", type=int, default=64, choices=(64, 32))
    ap.add_argument("--budget", type=int, default=6)
    a = ap.parse_args()
    w = dict(bench.WORKLOADS[a.workload])
    eng = Engine(0)
    eng.set_precision(a.precision)
    edges = bench.workload_graph(w)
    cfg = dict(qubit_cap=w["qubit_cap"], top_k=w["top_k"], layers=w["layers"], budget=a.budget,
               seed=0)
    eng.profile(1)
    eng.run_pipeline(w["n"], edges, **cfg)
    prof = eng.profile_read()
    eng.profile(False)
    out = {k: {"launches": v["launches"], "alg_bytes_per_launch": v["bytes"] / v["launches"],
               "us_per_launch": 1e3 * v["ms"] / v["launches"]}
           for k, v in prof.items() if v["launches"]}
    print("PROBE " + json.dumps({"workload": a.workload, "precision": a.precision, "kinds": out}))


if __name__ == "__main__":
    main()
