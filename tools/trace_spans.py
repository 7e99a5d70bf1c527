#!/usr/bin/env python3
"""GPU timeline of one bench step from kernel spans (globaltimer at each CTA group's entry
and exit; build/libqcgpu_trace.so, `make -C paper_2603_26232_b200/csrc trace`).

Runs the bench workload's resident pipeline session (prepare once, one warm-up execute,
one traced execute: the timed region's chunking, streams and CUDA graphs), then reports
per-SM busy fraction over the step, per-kernel-kind busy time, and idle gaps.

  python tools/trace_spans.py --workload c2 [--dump gpurun_out/spans_c2.npy]
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
import bench  # noqa: E402
import paper_2603_26232_b200 as pkg  # noqa: E402

KINDS = {1: "pass_a5", 2: "pass_a", 3: "pass_b", 4: "pass_b5", 5: "blocksum", 6: "onchip"}
REC = np.dtype([("kind", "<u4"), ("block", "<u4"), ("smg", "<u4"), ("pad", "<u4"),
                ("t0", "<u8"), ("t1", "<u8")])


def read(lib):
    out = []
    for fn in ("qc_span_read_pass", "qc_span_read_kernels"):
        buf = np.zeros(1 << 20, REC)
        n = C.c_int(0)
        rc = getattr(lib, fn)(buf.ctypes.data_as(C.c_void_p), C.c_int(buf.size), C.byref(n))
        assert rc == 0
        out.append(buf[: n.value])
    return np.concatenate(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2", choices=sorted(bench.WORKLOADS))
    ap.add_argument("--budget", type=int, default=0, help="override the NM budget (0: workload's)")
    ap.add_argument("--dump", default="")
    a = ap.parse_args()
    lib = pkg.load_library(os.path.join(ROOT, "build", "libqcgpu_trace.so"))
    pkg._LIB = lib
    w = dict(bench.WORKLOADS[a.workload])
    eng = pkg.Engine(0)
    edges = bench.workload_graph(w)
    cfg = dict(qubit_cap=w["qubit_cap"], top_k=w["top_k"], layers=w["layers"],
               budget=a.budget or w["budget"], seed=0)
    sess = eng.prepare_pipeline(w["n"], edges, **cfg)
    sess.execute()
    read(lib)
    rep = sess.execute()
    sp = read(lib)
    t0 = int(sp["t0"].min())
    t1 = int(sp["t1"].max())
    span = t1 - t0
    sm = sp["smg"] & 0xFFFF
    res = {"workload": a.workload, "cut": rep.cut, "qaoa_s": rep.qaoa_s, "records": int(len(sp)),
           "gpu_span_ms": span / 1e6}
    # per-SM busy (union of intervals)
    busy = []
    for s in np.unique(sm):
        iv = sp[sm == s]
        order = np.argsort(iv["t0"])
        st, en = iv["t0"][order].astype(np.int64), iv["t1"][order].astype(np.int64)
        tot, cur_s, cur_e = 0, st[0], en[0]
        for x, y in zip(st[1:], en[1:]):
            if x > cur_e:
                tot += cur_e - cur_s
                cur_s, cur_e = x, y
            else:
                cur_e = max(cur_e, y)
        tot += cur_e - cur_s
        busy.append(tot / span)
    res["sm_busy_mean"] = float(np.mean(busy))
    res["sm_busy_min"] = float(np.min(busy))
    kinds = {}
    for k, name in KINDS.items():
        m = sp["kind"] == k
        if m.any():
            d = (sp["t1"][m] - sp["t0"][m]).astype(np.float64)
            kinds[name] = {"spans": int(m.sum()), "busy_ms_per_sm": float(d.sum() / 1e6 / len(busy) / 2
                                                                        if k <= 4 else d.sum() / 1e6 / len(busy)),
                           "mean_span_us": float(d.mean() / 1e3)}
    res["kinds"] = kinds
    print(json.dumps(res))
    if a.dump:
        np.save(a.dump, sp)


if __name__ == "__main__":
    main()
