#!/usr/bin/env python3
"""Host-side split of the lockstep optimiser's per-chunk-step preparation (results + NM
tell, staging build, launch) for one resident solve of a bench workload."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2603_26232_b200 import Engine  # noqa: E402

w = dict(bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
eng = Engine(0)
edges = bench.workload_graph(w)
sess = eng.prepare_pipeline(w["n"], edges, qubit_cap=w["qubit_cap"], top_k=w["top_k"],
                            layers=w["layers"], budget=w["budget"], seed=0)
sess.execute()
eng.host_stats(reset=True)
for _ in range(3):
    sess.execute()
h = eng.host_stats(reset=True)
steps = h["chunk_steps"]
print(json.dumps({k: (v / steps * 1e6 if k.endswith("_s") else v) for k, v in h.items()}))
