#!/usr/bin/env python3
"""Benchmark: end-to-end Max-Cut solve time & subgraph-QAOA evals/s on B200.

One bench "step" = one full solve of the workload through the hot path: the batched
QAOA stage (lockstep Nelder-Mead over all subgraphs, `budget` objective evaluations
each, final circuit + top-K) and the candidate merge, i.e. pipeline.hpp:219-334.

  value  — evals/s with the inputs resident in HBM (qc_pipeline_prepare once, then
           qc_pipeline_execute per step): M * budget / device time per step.
  e2e    — the same metric through the reference-facing C-ABI call with HOST buffers
           (qc_run_pipeline: graph edges in, cut + assignment out; partition, table
           upload, per-step parameter uploads and result reads inside the timed region).

Default workload (BASELINE configs[1], one B200): ER(n=400, p=0.1, seed 0) split with
qubit_cap 20 into 21 chained 20-qubit subgraphs, QAOA depth p=2, top-K 2, budget 200,
level merge (2*2^21 = 4,194,304 leaves). N>1 (torchrun, one rank per GPU over NCCL):
the subgraphs are sharded in contiguous blocks, solve records are all-gathered over
NVLink (the only collective) and rank 0 merges.

`--impl reference` times the reference's own CPU implementation (oracle/_ref, the
unmodified qcut headers; the C restatement if that build is absent) on this host's
cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PROFILE_STRIDE = 16  # per-kernel CUDA events on one launch in 16 (sampled, live)
METRIC = "end-to-end Max-Cut solve time & subgraph-QAOA evals/s at 1/2/4/8 B200"
# FP64 ceiling for the no-FMA butterfly stream, measured on B200 with tools/ubench_fp64.cu
# (8 DMUL + 4 DADD per pair, all SMs): profiles/r1_ubench_fp64.txt
FP64_PEAK_TOPS = 18.44
UNIT = "evals/s"

WORKLOADS = {
    # BASELINE configs[1]: 400-vertex ER (the paper's 1,600x comparison size), 20-qubit
    # subgraphs, p=1-2, one B200
    "c2": dict(n=400, p_edge=0.1, seed=0, qubit_cap=20, layers=2, top_k=2, budget=200,
               label="C2: ER(n=400,p=0.1,seed=0), cap 20 -> 21 x 20-qubit subgraphs, QAOA p=2, "
                     "top-K 2, NM budget 200, level merge (4,194,304 leaves)"),
    "c1": dict(n=100, p_edge=0.1, seed=0, qubit_cap=10, layers=1, top_k=4, budget=200,
               label="C1: ER(n=100,p=0.1,seed=0), cap 10 -> 11 x 10-qubit subgraphs, p=1, "
                     "top-K 4, level merge (8,388,608 leaves)"),
    "c3": dict(n=1000, regular=3, wlo=1, whi=10, seed=0, qubit_cap=24, layers=1, top_k=2,
               budget=200,
               label="C3: weighted random 3-regular (n=1000, integer weights U{1..10}, seed 0), "
                     "cap 24 -> 44 subgraphs (43 x 24 + 1 x 11 qubits), p=1, top-K 2"),
    "c4": dict(n=10000, p_edge=0.1, seed=0, qubit_cap=20, layers=1, top_k=2, budget=200,
               label="C4: ER(n=10000,p=0.1,seed=0), cap 20 -> 527 x 20-qubit subgraphs, p=1, "
                     "top-K 2, windowed merge"),
    "c5": dict(n=16000, p_edge=0.1, seed=0, qubit_cap=26, layers=1, top_k=2, budget=200,
               label="C5: ER(n=16000,p=0.1,seed=0), cap 26 -> 640 x 26-qubit subgraphs, p=1, "
                     "top-K 2, windowed merge"),
}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def workload_graph(w, reference=False):
    """The workload's synthetic graph. The product arm uses the product's host generators
    (qc_generate_er = graph.hpp:146-160; qc_generate_regular for config 3); the reference
    arm uses the reference's own generator (oracle/_ref) — the graphs are identical
    (tests/test_cpu_abi.py)."""
    if reference:
        from oracle.refpy import OracleLib, RefLib, ref_available
        lib = RefLib() if ref_available() else OracleLib()
        if "regular" in w:
            return OracleLib().generate_regular(w["n"], w["regular"], w["seed"], w["wlo"], w["whi"])
        return lib.generate_er(w["n"], w["p_edge"], w["seed"])
    from paper_2603_26232_b200 import generate_er, generate_regular
    if "regular" in w:
        return generate_regular(w["n"], w["regular"], w["seed"], w["wlo"], w["whi"])
    return generate_er(w["n"], w["p_edge"], w["seed"])


class ClockSampler:
    """SM/memory clocks, power, temperature and throttle reasons sampled every 100 ms during the timed region, in-process
    through NVML (the same counters nvidia-smi reports; a polling nvidia-smi process was
    observed to stall the driver and inflate individual steps by 35-65 ms)."""

    REASONS = {  # nvmlClocksEventReason* bits
        "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4,
    }

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self.mem, self.power, self.temp = [], [], []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.thread = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def loop():
                while not self._stop.is_set():
                    try:
                        self.samples.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                        self.mem.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM)))
                        self.power.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0)
                        self.temp.append(float(pynvml.nvmlDeviceGetTemperature(h, pynvml.NVML_TEMPERATURE_GPU)))
                        bits = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for nm, b in self.REASONS.items():
                            if bits & b:
                                self.reasons.add(nm)
                    except Exception:
                        pass
                    self._stop.wait(0.1)
            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None

    def stop(self):
        if self.thread is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        self._stop.set()
        self.thread.join(timeout=2)
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_min_mhz": min(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "samples": len(self.samples),
                "mem_mhz": [min(self.mem), max(self.mem)] if self.mem else None,
                "power_w_max": max(self.power) if self.power else None,
                "temp_c_max": max(self.temp) if self.temp else None,
                "reasons": sorted(self.reasons), "source": "NVML (in-process, 100 ms)"}


# --------------------------------------------------------------------------------------
# CPU baseline / reference arm
# --------------------------------------------------------------------------------------
def reference_sample(w, edges, budgets=(4, 12)):
    """Time the reference pipeline (partition -> QAOA stage -> merge, all host threads) at
    two small NM budgets and extrapolate the QAOA stage linearly to the full budget
    (fixed per-subgraph costs — cost table, final circuit, top-K — are the intercept).
    Returns (evals/s, description, kind, cores, seconds spent)."""
    from oracle.refpy import OracleLib, RefLib, ref_available
    kind = "reference" if ref_available() else "port"
    lib = RefLib() if kind == "reference" else OracleLib()
    cores = os.cpu_count() or 1
    t0 = time.time()
    runs = []
    for b in budgets:
        r = lib.run_pipeline(w["n"], edges, qubit_cap=w["qubit_cap"], top_k=w["top_k"],
                             layers=w["layers"], budget=b, seed=0, workers=cores)
        runs.append(r)
    (b1, r1), (b2, r2) = zip(budgets, runs)
    slope = max((r2["qaoa_s"] - r1["qaoa_s"]) / (b2 - b1), 0.0)
    fixed = max(r1["qaoa_s"] - slope * b1, 0.0)
    qaoa_full = fixed + slope * w["budget"]
    merge_s = min(r1["merge_s"], r2["merge_s"])
    total = r1["partition_s"] + qaoa_full + merge_s
    M = r1["subgraphs"]
    value = M * w["budget"] / total
    desc = (f"{'oracle/_ref (unmodified qcut headers)' if kind == 'reference' else 'oracle C port'}"
            f" run_pipeline with workers={cores} at NM budgets {b1} and {b2}; QAOA stage "
            f"extrapolated linearly to budget {w['budget']} ({qaoa_full:.2f} s), merge "
            f"{merge_s:.2f} s measured, total {total:.2f} s per solve of {M} subgraphs")
    return value, desc, kind, cores, time.time() - t0, total


def run_reference_arm(args, w):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    edges = workload_graph(w, reference=True)
    for _ in range(args.warmup):
        reference_sample(w, edges)
    vals, totals = [], []
    desc = kind = cores = None
    for _ in range(args.steps):
        v, desc, kind, cores, _, total = reference_sample(w, edges)
        vals.append(v)
        totals.append(total)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": statistics.median(totals) * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w["label"], "n": w["n"], "p_edge": w.get("p_edge"),
                   "qubit_cap": w["qubit_cap"], "layers": w["layers"], "top_k": w["top_k"],
                   "budget": w["budget"], "parallelism": f"cpu x{cores} threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------------------
def steady_state(eng, w, kernel, slots=(10, 40), reps=8):
    """The dominant pass kernel at two batch sizes of the workload's subgraph shape (one
    chunk, one stream, every launch timed by CUDA events): time per launch = fixed +
    slots x slope, so the steady-state bandwidth is bytes-per-slot / slope. Separates the
    per-launch fixed cost (launch, ring fill, drain) from the streaming efficiency."""
    from paper_2603_26232_b200 import generate_er
    q, p = w["qubit_cap"], w["layers"]
    e = generate_er(q, 0.2, 1)
    rng = np.random.default_rng(0)
    prev = os.environ.get("QCG_CHUNKS")
    os.environ["QCG_CHUNKS"] = "1"
    pts = []
    try:
        for n in slots:
            prm = rng.uniform(0.1, 3.0, size=(n, 2 * p))
            idx = np.zeros(n, np.int32)
            eng.eval_batch([(q, e)], p, idx, prm)  # warm (buffers, graph capture)
            eng.profile(1)
            for _ in range(reps):
                eng.eval_batch([(q, e)], p, idx, prm)
            v = eng.profile_read()[kernel]
            eng.profile(False)
            if not v["launches"]:
                return None
            pts.append((n, v["ms"] * 1e3 / v["launches"], v["bytes"] / v["launches"]))
    finally:
        if prev is None:
            os.environ.pop("QCG_CHUNKS", None)
        else:
            os.environ["QCG_CHUNKS"] = prev
    (n1, t1, b1), (n2, t2, b2) = pts
    slope = (t2 - t1) / (n2 - n1)                  # us per slot
    per_slot = b2 / n2                             # algorithmic bytes per slot and launch
    return {"kernel": kernel, "subgraph_qubits": q, "slots": [n1, n2],
            "us_per_launch": [round(t1, 2), round(t2, 2)], "us_per_slot": round(slope, 3),
            "fixed_us_per_launch": round(t1 - n1 * slope, 2),
            "achieved": per_slot / (slope * 1e-6) / 1e9 if slope > 0 else None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--precision", type=int, default=64, choices=[64, 32],
                    help="64: exact fp64 (the parity path, default); 32: optional fp32 mode (1e-4)")
    ap.add_argument("--report", default="",
                    help="also write the run as an ExperimentReport JSON v1 (report.hpp) with a "
                         "'gpu' section to this path")
    ap.add_argument("--profile-stride", type=int, default=PROFILE_STRIDE,
                    help="CUDA-event sampling of 1 launch in N during the timed region (0: off)")
    args = ap.parse_args()
    w = dict(WORKLOADS[args.workload])
    if args.impl == "reference":
        return run_reference_arm(args, w)

    import torch
    import torch.distributed as dist
    from paper_2603_26232_b200 import Engine

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # QCG_BENCH_BACKEND=gloo exercises the multi-rank path on a box with fewer GPUs than
    # ranks (ranks share devices, records gathered through host memory); default NCCL.
    backend = os.environ.get("QCG_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    coll_dev = torch.device("cuda", local) if backend == "nccl" else torch.device("cpu")
    eng = Engine(local)
    eng.set_precision(args.precision)
    stream = torch.cuda.ExternalStream(eng.stream_handle(), device=local)
    edges = workload_graph(w)
    cfg = dict(qubit_cap=w["qubit_cap"], top_k=w["top_k"], layers=w["layers"],
               budget=w["budget"], seed=0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")  # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- single GPU: resident session (value) -------------------------------------
    if world == 1:
        sess = eng.prepare_pipeline(w["n"], edges, **cfg)
        M = None

        def step_value():
            return sess.execute()
    else:
        from paper_2603_26232_b200.distributed import solve_sharded
        M = eng.subgraph_count(w["n"], edges, **cfg)

        def step_value():
            # shard the QAOA stage, one NCCL all-gather of solve records, merge on rank 0
            return solve_sharded(eng, w["n"], edges, rank, world, device=coll_dev, **cfg)

    def timed(fn, steps, prof=False):
        """per-step device time via CUDA events on the engine stream, L2 flushed between."""
        times, last = [], None
        launches0 = eng.launches
        if prof and args.profile_stride > 0:
            eng.profile(args.profile_stride)
        for _ in range(steps):
            flush.zero_()
            barrier()
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            last = fn()
            ev1.record(stream)
            barrier()
            times.append(ev0.elapsed_time(ev1) / 1e3)
        launches = eng.launches - launches0
        profile = eng.profile_read() if prof and args.profile_stride > 0 else {}
        if prof:
            eng.profile(False)
        return times, last, launches, profile

    for _ in range(args.warmup):
        step_value()
        barrier()
    clocks = ClockSampler(local)
    eng.host_stats(reset=True)
    tv0 = eng.transfers()
    clocks.start()
    t_val, rep, launches, profile = timed(step_value, args.steps, prof=True)
    tv1 = eng.transfers()
    clk = clocks.stop()
    host = eng.host_stats(reset=True)

    # max over ranks
    tot = torch.tensor([sum(t_val)], dtype=torch.float64, device=coll_dev)
    lt = torch.tensor([launches], dtype=torch.float64, device=coll_dev)
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
        dist.all_reduce(lt, op=dist.ReduceOp.SUM)
    sec_per_step = tot.item() / args.steps
    n_sub = rep.subgraphs if rank == 0 and rep is not None else (M or 0)
    evals_per_step = (rep.evals if rank == 0 and rep is not None else 0)

    # ---- e2e through the C-ABI with host buffers (N=1; N>1 reuses the sharded path)
    e2e = None
    if world == 1:
        h0, d0 = eng.transfers()

        def step_e2e():
            return eng.run_pipeline(w["n"], edges, **cfg)
        for _ in range(args.warmup):
            step_e2e()
        barrier()
        h0, d0 = eng.transfers()
        t_e2e, rep_e2e, _, _ = timed(step_e2e, args.steps)
        h1, d1 = eng.transfers()
        assert rep_e2e.cut == rep.cut and rep_e2e.assignment == rep.assignment
        e2e = {"value": rep_e2e.evals / (sum(t_e2e) / args.steps), "unit": UNIT,
               "h2d_bytes_per_step": (h1 - h0) // args.steps,
               "d2h_bytes_per_step": (d1 - d0) // args.steps,
               "ms_per_step": sum(t_e2e) / args.steps * 1e3,
               "step_ms": [round(t * 1e3, 2) for t in t_e2e],
               "stage_s": {"partition": rep_e2e.partition_s, "qaoa": rep_e2e.qaoa_s,
                           "merge": rep_e2e.merge_s}}
    # ---- roofline for the dominant kernel --------------------------------------------
    # The timed region runs chunks on concurrent streams, so per-launch event durations
    # there are stretched by sharing the GPU. The kernel roofline is therefore taken from
    # one extra, single-stream step in which EVERY launch is bracketed by CUDA events on
    # its own stream; the timed-region (sampled) figures are reported beside it.
    iso_prev = os.environ.get("QCG_CHUNKS")
    os.environ["QCG_CHUNKS"] = "1"
    eng.profile(1)
    step_value()  # every rank: the multi-GPU step contains the record all-gather
    barrier()
    profile_iso = eng.profile_read()
    eng.profile(False)
    if iso_prev is None:
        os.environ.pop("QCG_CHUNKS", None)
    else:
        os.environ["QCG_CHUNKS"] = iso_prev
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    if e2e is None:
        # multi-GPU: the timed step is already the C-ABI call with host buffers on every
        # rank (graph edges in, records out through the host for the gather, merge on rank 0)
        e2e = {"value": evals_per_step / sec_per_step, "unit": UNIT,
               "h2d_bytes_per_step": (tv1[0] - tv0[0]) // args.steps,
               "d2h_bytes_per_step": (tv1[1] - tv0[1]) // args.steps,
               "note": "rank 0's copies; the sharded step runs through qc_shard_solve / "
                       "qc_merge_records with host buffers on every rank"}

    peak, peak_kind = load_peaks()
    dom = max(profile_iso, key=lambda k: profile_iso[k]["ms"])
    d = profile_iso[dom]
    iso_ms = sum(v["ms"] for v in profile_iso.values())
    iso_bytes = sum(v["bytes"] for v in profile_iso.values())
    achieved = d["bytes"] / (d["ms"] / 1e3) / 1e9 if d["ms"] > 0 else 0.0
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(dom)
            traffic = tr.get("dram_bytes_per_launch") if tr else None
    except Exception:
        pass
    fp64_peak = FP64_PEAK_TOPS
    fp64_ach = d.get("fp64_ops", 0.0) / (d["ms"] / 1e3) / 1e12 if d["ms"] > 0 else 0.0
    ss = None
    if world == 1 and dom in ("pass_low", "pass_high"):
        try:
            ss = steady_state(eng, w, dom)
            if ss and ss.get("achieved"):
                ss["frac"] = ss["achieved"] / peak
        except Exception as ex:  # diagnostic only: never fail the bench on it
            ss = {"error": str(ex)[:200]}
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind ==
                "measured" else "fallback (B200_PROFILING.md)",
                "algorithmic_bytes_per_launch": d["bytes"] / max(d["launches"], 1),
                "avg_launch_ms": d["ms"] / max(d["launches"], 1),
                "measured": "every launch of one single-stream step, CUDA events on its stream",
                "launches": d["launches"],
                "share_of_step": d["ms"] / iso_ms if iso_ms else None,
                # streaming efficiency without the per-launch fixed cost (see steady_state)
                "steady_state": ss,
                # the fp64 parity path forbids FMA: every butterfly is 8 DMUL + 4 DADD, so
                # the FP64 pipe is the second ceiling (co-bound for the 12-target pass A)
                "fp64": {"achieved_tops": fp64_ach, "peak_tops": fp64_peak,
                         "frac": fp64_ach / fp64_peak,
                         "ops_per_launch": d.get("fp64_ops", 0.0) / max(d["launches"], 1),
                         "peak_source": "measured: tools/ubench_fp64.cu mixer_pair pattern "
                                        "(profiles/r1_ubench_fp64.txt)"},
                "kernels": {k: {"launches": v["launches"], "ms": round(v["ms"], 3),
                                "GB/s": round(v["bytes"] / (v["ms"] / 1e3) / 1e9, 1)
                                if v["ms"] > 0 else 0.0,
                                "fp64_Tops": round(v.get("fp64_ops", 0.0) / (v["ms"] / 1e3) / 1e12, 2)
                                if v["ms"] > 0 else 0.0}
                            for k, v in profile_iso.items() if v["launches"]},
                # all engine kernels' algorithmic bytes of one step / timed step time
                "step_aggregate_GBs": iso_bytes / sec_per_step / 1e9,
                "step_aggregate_frac": iso_bytes / sec_per_step / 1e9 / peak,
                "timed_region_sampled": {
                    "stride": args.profile_stride, "streams": 2,
                    "kernels": {k: {"launches": v["launches"], "ms": round(v["ms"], 3),
                                    "GB/s": round(v["bytes"] / (v["ms"] / 1e3) / 1e9, 1)
                                    if v["ms"] > 0 else 0.0}
                                for k, v in profile.items() if v["launches"]}}}

    line = {
        "metric": METRIC, "value": evals_per_step / sec_per_step, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec_per_step * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64" if args.precision == 64 else "f32",
        "data": "synthetic (graph.hpp:146 ER generator restated in qc_generate_er)",
        "config": {"workload": w["label"], "n": w["n"], "p_edge": w.get("p_edge"),
                   "qubit_cap": w["qubit_cap"], "subgraphs": n_sub, "layers": w["layers"],
                   "top_k": w["top_k"], "budget": w["budget"], "parallelism": f"shard{world}",
                   "l2": "working set (21 half-states x 8 MiB + f buffers) > 126 MB L2; "
                         "L2 flushed (256 MB write) between timed steps"},
        "solve_time_s": sec_per_step, "cut": rep.cut, "evals_per_step": evals_per_step,
        "step_ms": [round(t * 1e3, 2) for t in t_val],
        "host_s_per_step": {k: (v / args.steps if k != "chunk_steps" else v // args.steps)
                            for k, v in host.items()},
        "stage_s": {"partition": rep.partition_s, "qaoa": rep.qaoa_s, "merge": rep.merge_s},
        "e2e": e2e, "gpu_launches": int(lt.item()), "clocks": clk, "roofline": roofline,
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            v, desc, kind, cores, _, total = reference_sample(w, workload_graph(w, reference=True))
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                                    "sample": desc}
        except Exception as ex:  # report, never fail the bench line
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(),
                                    "kind": "unavailable", "sample": str(ex)}
    print(json.dumps(line), flush=True)
    if args.report and rep is not None:
        from paper_2603_26232_b200.report import emit_report, experiment_report
        doc = experiment_report(
            rep, n=w["n"], edges=len(edges), cfg=dict(cfg, shard_count=world), generated=True,
            p=w.get("p_edge", 0.0), graph_seed=w["seed"],
            gpu={"device": torch.cuda.get_device_name(local), "n_gpus": world,
                 "precision": f"fp{args.precision}", "evals_per_s": line["value"],
                 "e2e_evals_per_s": e2e["value"], "ms_per_step": line["ms_per_step"],
                 "roofline": {"kernel": roofline["kernel"], "hbm_frac": roofline["frac"],
                              "fp64_frac": roofline["fp64"]["frac"]},
                 "clocks": clk})
        with open(args.report, "w") as f:
            f.write(emit_report(doc))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
