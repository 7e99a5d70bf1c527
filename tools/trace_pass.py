#!/usr/bin/env python3
"""Phase timeline of the TMA pass A tile loop (k_pass_a5), from clock64 stamps taken by
each consumer group's lane 0 in CTAs 0-3 (build/libqcgpu_trace.so = the library built
with -DQCG_TRACE: `make -C paper_2603_26232_b200/csrc trace`).

Events per tile: 0 loop top, 1 after the pending refill, 2 data ready (tag + mbarrier),
3 round 0 done, 4 round 1 done, 5 round-2 loads done (after two group barriers),
6 round 2 computed + staged, 7 after the fence + group barrier (bulk store issued next).

  QCG_CHUNKS=1 python tools/trace_pass.py --q 20 --slots 21 --layers 1
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_26232_b200 as pkg  # noqa: E402

CTAS, TILES, EV = 4, 40, 8
NAMES = ["refill", "wait", "r0", "r1", "r2_ld", "r2_mix", "fence_sync"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--q", type=int, default=20)
    ap.add_argument("--slots", type=int, default=21)
    ap.add_argument("--layers", type=int, default=1)
    ap.add_argument("--dump", default="")
    ap.add_argument("--profile", action="store_true")
    a = ap.parse_args()
    lib = pkg.load_library(os.path.join(ROOT, "build", "libqcgpu_trace.so"))
    pkg._LIB = lib
    eng = pkg.Engine(0)
    graphs = [(a.q, pkg.generate_er(a.q, 0.2, 100 + i)) for i in range(a.slots)]
    rng = np.random.default_rng(0)
    idx = np.arange(a.slots, dtype=np.int32)
    prm = rng.uniform(0.1, 3.0, size=(a.slots, 2 * a.layers))
    eng.eval_batch(graphs, a.layers, idx, prm)
    if a.profile:  # CUDA-event time of the same launches, for the launch overhead
        eng.profile(1)
    buf = np.zeros(CTAS * 2 * TILES * EV, np.int64)
    eng.eval_batch(graphs, a.layers, idx, prm)
    lib.qc_trace_read(buf.ctypes.data_as(C.POINTER(C.c_longlong)), C.c_int(buf.size))
    ctab = np.zeros(1024 * 4, np.uint64)
    lib.qc_trace_read_ctas(ctab.ctypes.data_as(C.POINTER(C.c_ulonglong)), C.c_int(ctab.size))
    ctab = ctab.reshape(1024, 4).astype(np.int64)
    ctab = ctab[ctab[:, 0] > 0]
    if a.profile:
        pr = eng.profile_read()
        eng.profile(False)
    t = buf.reshape(CTAS, 2, TILES, EV)
    out = {"q": a.q, "slots": a.slots, "layers": a.layers, "ctas": []}
    for c in range(CTAS):
        t0 = t[c][t[c] > 0].min()
        cta = {}
        for g in range(2):
            rows = [r for r in t[c, g] if r[0] > 0 and r[7] > 0]
            d = np.array([np.diff(r) for r in rows], dtype=float)
            cta[f"g{g}"] = {"tiles": len(rows),
                            "mean_clk": dict(zip(NAMES, np.round(d.mean(0), 0).tolist())) if len(rows) else {},
                            "first_top": int(rows[0][0] - t0) if rows else None,
                            "last_end": int(rows[-1][7] - t0) if rows else None}
        out["ctas"].append(cta)
    if a.profile:
        out["event_us"] = {k: round(1e3 * v["ms"] / v["launches"], 2) for k, v in pr.items() if v["launches"]}
    if len(ctab):
        t0 = ctab[:, 0].min()
        ends = np.maximum(ctab[:, 2], ctab[:, 3]) - t0
        out["launch_ns"] = {
            "ctas": int(len(ctab)),
            "entry_spread": int(ctab[:, 0].max() - t0),
            "prologue_mean": float(np.mean(ctab[:, 1] - ctab[:, 0])),
            "end_min": int(ends.min()), "end_median": float(np.median(ends)), "end_max": int(ends.max()),
            "group_end_gap_mean": float(np.mean(np.abs(ctab[:, 2] - ctab[:, 3]))),
        }
    print(json.dumps(out))
    if a.dump:
        np.save(a.dump, t)


if __name__ == "__main__":
    main()
