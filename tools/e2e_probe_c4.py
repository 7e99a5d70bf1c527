"""C4 end to end (qc_run_pipeline, host buffers) vs resident (qc_pipeline_execute): wall time
per call with the stage split and the engine's host counters, to locate the e2e overhead."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_26232_b200 import Engine, generate_er
eng = Engine(0)
edges = generate_er(10000, 0.1, 0)
cfg = dict(qubit_cap=20, top_k=2, layers=1, budget=int(sys.argv[1]) if len(sys.argv) > 1 else 200, seed=0)
sess = eng.prepare_pipeline(10000, edges, **cfg)
for i in range(3):
    eng.host_stats(reset=True)
    t = time.perf_counter(); r = sess.execute(); w = time.perf_counter() - t
    print(f"resident {i}: wall {w*1e3:.1f} ms qaoa {r.qaoa_s*1e3:.1f} merge {r.merge_s*1e3:.2f} host {eng.host_stats(reset=True)}", flush=True)
    t = time.perf_counter(); r = eng.run_pipeline(10000, edges, **cfg); w = time.perf_counter() - t
    print(f"e2e      {i}: wall {w*1e3:.1f} ms partition {r.partition_s*1e3:.2f} qaoa {r.qaoa_s*1e3:.1f} merge {r.merge_s*1e3:.2f} host {eng.host_stats(reset=True)}", flush=True)
