#!/usr/bin/env python3
"""ncu DRAM traffic per launch of the engine kernels, per bench workload, for
bench.py's roofline.traffic (profiles/ncu_traffic.json, keys "<workload>/<f64|f32>/<kind>").

For each workload: `ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,
gpu__time_duration.sum --clock-control none` over tools/traffic_probe.py (one solve with
the bench's roofline-step launch shape), every launch of the pass / block-sum kernels.
Per kernel kind: mean DRAM bytes per launch, and the ratio to the algorithmic bytes the
engine counts for the same launches (bench.py reports traffic = ratio x its own
algorithmic bytes per launch, so a workload's line carries its own measured ratio).

  python tools/ncu_traffic.py c1 c2 c3 c4 c5 [--precision 32] [--merge profiles/ncu_traffic.json]
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KIND = [("k_pass_a", "pass_low"), ("k_pass_b", "pass_high"), ("k_blocksum", "blocksum"),
        ("k_fsum_f32", "blocksum"), ("k_onchip", "onchip")]


def kind_of(name: str):
    for pat, k in KIND:
        if pat in name:
            return k
    return None


def run(workload: str, precision: int, budget: int, max_launches: int):
    cmd = ["ncu", "--csv", "--clock-control", "none", "--launch-count", str(max_launches),
           "--kernel-name", "regex:k_pass_a|k_pass_b|k_blocksum|k_fsum_f32|k_onchip",
           "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           sys.executable, os.path.join(ROOT, "tools", "traffic_probe.py"), "--workload", workload,
           "--precision", str(precision), "--budget", str(budget)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=3000)
    probe = None
    lines = []
    for ln in r.stdout.splitlines():
        if ln.startswith("PROBE "):
            probe = json.loads(ln[6:])
        elif ln.startswith('"'):
            lines.append(ln)
    if probe is None:
        raise RuntimeError(f"{workload}: probe failed\n{r.stdout[-2000:]}\n{r.stderr[-2000:]}")
    per = {}
    for row in csv.DictReader(io.StringIO("\n".join(lines))):
        k = kind_of(row.get("Kernel Name", ""))
        if k is None:
            continue
        key = (row["ID"], k)
        d = per.setdefault(key, {})
        val = float(row["Metric Value"].replace(",", ""))
        unit = row.get("Metric Unit", "")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
                 "GB": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9,
                 "us": 1e-6, "ms": 1e-3}.get(unit, 1)
        d[row["Metric Name"]] = val * scale
    agg = {}
    for (_, k), d in per.items():
        a = agg.setdefault(k, {"launches": 0, "dram": 0.0, "sec": 0.0})
        a["launches"] += 1
        a["dram"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
        a["sec"] += d.get("gpu__time_duration.sum", 0.0)
    out = {}
    tag = "f64" if precision == 64 else "f32"
    for k, a in agg.items():
        pk = probe["kinds"].get(k)
        dpl = a["dram"] / a["launches"]
        ent = {"dram_bytes_per_launch": dpl, "launches_captured": a["launches"],
               "ncu_us_per_launch": 1e6 * a["sec"] / a["launches"],
               "source": f"tools/ncu_traffic.py: ncu DRAM read+write of every {k} launch of one "
                         f"{workload} solve (budget {budget}, QCG_CHUNKS=1: the bench roofline "
                         f"step's launch shape), first {max_launches} engine launches"}
        if pk:
            ent["alg_bytes_per_launch"] = pk["alg_bytes_per_launch"]
            ent["traffic_over_algorithmic"] = dpl / pk["alg_bytes_per_launch"] if pk["alg_bytes_per_launch"] else None
        out[f"{workload}/{tag}/{k}"] = ent
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workloads", nargs="+")
    ap.add_argument("--precision", type=int, default=64)
    ap.add_argument("--budget", type=int, default=6)
    ap.add_argument("--max-launches", type=int, default=120)
    ap.add_argument("--merge", default="")
    a = ap.parse_args()
    res = {}
    if a.merge and os.path.exists(a.merge):
        with open(a.merge) as f:
            res = json.load(f)
    for wl in a.workloads:
        res.update(run(wl, a.precision, a.budget, a.max_launches))
        print(json.dumps({k: v for k, v in res.items() if k.startswith(wl + "/")}), flush=True)
    if a.merge:
        with open(a.merge, "w") as f:
            json.dump(res, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
