"""Helper for test_gpu_statevector.py::test_pass_b_kernel_variants (run in a subprocess so
the QCG_PASS_B / QCG_B5_STORE kernel selection, read once per process, can be forced).

Checks the engine against the oracle, bit-exact, at subgraph sizes covering every pass B
geometry class: mirror passes with 1..8 targets (q = 14..21) and the 9-target pass
followed by a mirror pass (q = 22); states (F_STATE_OUT) and expectations alone
(eval_batch: the f pass without the state write); and the fp32 mode's expectations
(within 1e-4, RX and Walsh-Hadamard mixers). Prints OK.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.refpy import checker  # noqa: E402
from paper_2603_26232_b200 import Engine  # noqa: E402


def main():
    orc = checker()  # the reference build (oracle/_ref) when present
    orc.set_qubit_cap(26)
    eng = Engine(0)
    threads = max(1, min(32, os.cpu_count() or 1))
    for q in (14, 16, 19, 20, 21, 22):
        e = orc.generate_er(q, 0.2, 100 + q)
        rng = np.random.default_rng(q)
        g = rng.uniform(0.1, 3.0, 2)
        b = rng.uniform(0.1, 3.0, 2)
        a0, x0 = orc.run_ansatz(q, e, g, b, threads=threads)
        a1, x1 = eng.run_ansatz(q, e, g, b)
        assert np.array_equal(a1, a0), f"q={q}: amplitudes differ"
        assert x1 == x0, f"q={q}: expectation {x1!r} != {x0!r}"
        got = eng.eval_batch([(q, e)], 2, np.zeros(1, np.int32), np.concatenate([g, b])[None, :])
        assert got[0] == x0, f"q={q}: eval_batch {got[0]!r} != {x0!r}"
    # optional fp32 mode (F_FP32): same pass structure on float2 states, within 1e-4
    # (both mixer forms: RX butterflies and the Walsh-Hadamard variant)
    f32 = Engine(0)
    f32.set_precision(32)
    wht = Engine(0)
    wht.set_precision(32)
    wht.set_mixer("wht")
    for q in (14, 16, 19, 20, 22, 24):
        e = orc.generate_er(q, 0.2, 100 + q)
        rng = np.random.default_rng(q)
        prm = np.concatenate([rng.uniform(0.1, 3.0, 2), rng.uniform(0.1, 3.0, 2)])
        x0 = orc.run_ansatz(q, e, prm[:2], prm[2:], threads=threads, want_amps=False)[1]
        for name, en in (("rx", f32), ("wht", wht)):
            got = en.eval_batch([(q, e)], 2, np.zeros(1, np.int32), prm[None, :])
            assert abs(got[0] - x0) <= 1e-4 * abs(x0), f"fp32 {name} q={q}: {got[0]!r} vs {x0!r}"
    print("OK")


if __name__ == "__main__":
    main()
