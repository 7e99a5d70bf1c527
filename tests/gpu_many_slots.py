"""Helper for test_gpu_statevector.py::test_split_launches (run in a subprocess with
QCG_CHUNKS=1 and QCG_PASS_B=tma): 3200 evaluations of one 14-qubit graph in a single chunk,
more slots than one persistent launch caches descriptors for (21 x 148), so every pass is
split into several launches whose TMA tensor maps start at a slot offset. Sampled points
are compared bit-exactly with the oracle. Prints OK."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.refpy import checker  # noqa: E402
from paper_2603_26232_b200 import Engine  # noqa: E402


def main():
    orc = checker()  # the reference build (oracle/_ref) when present
    eng = Engine(0)
    q, p, n = 14, 2, 3200
    e = orc.generate_er(q, 0.3, 5)
    rng = np.random.default_rng(11)
    prm = rng.uniform(0.1, 3.0, size=(n, 2 * p))
    got = eng.eval_batch([(q, e)], p, np.zeros(n, np.int32), prm)
    for k in list(range(0, 8)) + list(range(3100, 3200, 13)) + [n - 1]:
        x0 = orc.run_ansatz(q, e, prm[k, :p], prm[k, p:], want_amps=False)[1]
        assert got[k] == x0, (k, got[k], x0)
    print("OK")


if __name__ == "__main__":
    main()
