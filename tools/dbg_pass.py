import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_26232_b200 import Engine, generate_er
from oracle.refpy import OracleLib
orc = OracleLib(); eng = Engine(0)
for q in [int(x) for x in sys.argv[1].split(",")]:
    for layers in (1, 2):
        e = generate_er(q, 0.3, q)
        rng = np.random.default_rng(q)
        g = rng.uniform(0.1, np.pi, layers); b = rng.uniform(0.1, np.pi, layers)
        a0, x0 = orc.run_ansatz(q, e, g, b)
        a1, x1 = eng.run_ansatz(q, e, g, b)
        a2, x2 = eng.run_ansatz(q, e, g, b)
        bad = np.nonzero(a1 != a0)[0]
        print(q, layers, "x_ok", x0 == x1, "det", np.array_equal(a1, a2), "nbad", len(bad),
              "first", bad[:8].tolist(), "maxdiff", float(np.max(np.abs(a1 - a0))), flush=True)
if len(sys.argv) > 2:
    q = int(sys.argv[2]); S = int(sys.argv[3]); layers = 2
    graphs = [(q, generate_er(q, 0.2, 100 + i)) for i in range(S)]
    rng = np.random.default_rng(0)
    prm = rng.uniform(0.1, 3.0, size=(S, 2 * layers))
    idx = np.arange(S, dtype=np.int32)
    o1 = eng.eval_batch(graphs, layers, idx, prm)
    o2 = eng.eval_batch(graphs, layers, idx, prm)
    ref = [orc.run_ansatz(q, graphs[i][1], prm[i, :layers], prm[i, layers:])[1] for i in range(min(S, 4))]
    print("batch", q, S, "det", np.array_equal(o1, o2), "ref_ok", [o1[i] == ref[i] for i in range(len(ref))],
          (o1 - o2)[:6].tolist())
