"""C5 probe: ER(16000, 0.1, seed 0) split into 26-qubit subgraphs (640 pieces), p=1, top-K 2,
windowed merge -- through qc_run_pipeline on one GPU at a reduced NM budget, to size the
full-budget run. usage: python tools/c5_probe.py [budget]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_26232_b200 import Engine, generate_er
budget = int(sys.argv[1]) if len(sys.argv) > 1 else 4
t = time.perf_counter()
edges = generate_er(16000, 0.1, 0)
print(f"generate: {len(edges)} edges in {time.perf_counter() - t:.1f} s", flush=True)
eng = Engine(0)
cfg = dict(qubit_cap=26, top_k=2, layers=1, budget=budget, seed=0)
for rep in range(2):
    t = time.perf_counter()
    r = eng.run_pipeline(16000, edges, **cfg)
    w = time.perf_counter() - t
    print(f"budget {budget}: wall {w:.2f} s  partition {r.partition_s:.3f} qaoa {r.qaoa_s:.2f} "
          f"merge {r.merge_s:.3f}  subgraphs {r.subgraphs} evals {r.evals} cut {r.cut} "
          f"evals/s {r.evals / r.qaoa_s:.0f}", flush=True)
