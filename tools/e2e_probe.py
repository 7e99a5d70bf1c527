"""Wall time of consecutive qc_run_pipeline calls (C2 workload) with the stage split."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_26232_b200 import Engine, generate_er
eng = Engine(0)
edges = generate_er(400, 0.1, 0)
cfg = dict(qubit_cap=20, top_k=2, layers=2, budget=200, seed=0)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 10):
    t = time.perf_counter()
    r = eng.run_pipeline(400, edges, **cfg)
    w = time.perf_counter() - t
    print(f"{i}: wall {w*1e3:.1f} ms  partition {r.partition_s*1e3:.2f} qaoa {r.qaoa_s*1e3:.1f} merge {r.merge_s*1e3:.2f} host {eng.host_stats(reset=True)}", flush=True)
