import sys, os
sys.path.insert(0, os.getcwd())
from paper_2603_26232_b200 import Engine, generate_er
eng = Engine(0)
for n, cap, L, K, b in [(400, 20, 1, 1, 20), (1000, 20, 1, 1, 10), (2000, 20, 1, 1, 5), (10000, 20, 1, 1, 5), (10000, 20, 1, 2, 5)]:
    e = generate_er(n, 0.1, 0)
    r = eng.run_pipeline(n, e, qubit_cap=cap, top_k=K, layers=L, budget=b, seed=0)
    print(n, K, r.cut, r.windowed, flush=True)
