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
def host_info():
    """CPU model, logical cores and memory of this host (the reference arm's hardware)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    mem = None
    try:
        with open("/proc/meminfo") as f:
            mem = round(int(f.readline().split()[1]) / 2**20, 1)
    except (OSError, ValueError, IndexError):
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "mem_gib": mem}


def subgraph_count(w):
    """partition.hpp:163-167 derive_subgraph_count (the chain split both arms use)."""
    n, cap = w["n"], w["qubit_cap"]
    return 1 if n <= cap else (n - 1 + cap - 2) // (cap - 1)


def config_dict(w, world):
    """The workload description; identical in both arms (same keys, same values)."""
    return {"workload": w["label"], "n": w["n"], "p_edge": w.get("p_edge"),
            "graph": "weighted random 3-regular" if "regular" in w else "Erdos-Renyi",
            "qubit_cap": w["qubit_cap"], "subgraphs": subgraph_count(w), "layers": w["layers"],
            "top_k": w["top_k"], "budget": w["budget"], "seed": w["seed"],
            "parallelism": f"shard{world}"}


# Workloads whose full reference solve fits a bench run (C1 ~0.2 s, C2 ~27 s on 16 host
# threads). The others take minutes to hours on the CPU (C3 ~8 min, C4 ~2 h, C5 ~days),
# so their reference numbers come from a bounded sample of the same QAOA stage.
FULL_REFERENCE = ("c1", "c2")
# sampled reference: NM budget per sampled solve (the ramp eval + the first simplex points)
SAMPLE_BUDGET = {"c3": 4, "c4": 40, "c5": 2}


def ref_lib(w):
    from oracle.refpy import OracleLib, RefLib, ref_available
    cap26 = w["qubit_cap"] > 24
    if ref_available(cap26):
        return RefLib(cap26=cap26), "reference"
    lib = OracleLib()
    lib.set_qubit_cap(26 if cap26 else 24)
    return lib, "port"


def reference_full(w, edges, cores):
    """One full solve of the workload by the reference's stock run_pipeline
    (pipeline.hpp:391: partition -> QAOA stage -> merge; workers = all host threads)."""
    lib, kind = ref_lib(w)
    r = lib.run_pipeline(w["n"], edges, qubit_cap=w["qubit_cap"], top_k=w["top_k"],
                         layers=w["layers"], budget=w["budget"], seed=w["seed"], workers=cores)
    value = r["subgraphs"] * w["budget"] / r["total_s"]
    return value, r, kind


def sample_indices(M, S):
    return sorted(set(int(round(x)) for x in np.linspace(0, M - 1, S)))


def reference_sampled(w, edges, cores, indices=None):
    """A bounded sample of the reference QAOA stage: S = min(cores, M) subgraphs spread over
    the chain solved concurrently exactly as pipeline.hpp:223-280 schedules one round
    (slots = min(workers, M) std::threads, threads_per = workers / slots OpenMP threads each,
    seed = base + idx), at a reduced NM budget b. The stage at the full budget B is then
    ceil(M/S) such rounds of B/b times the sampled round (the fixed per-solve costs —
    cost table, final circuit, top-K — are counted B/b times, which overstates the CPU
    time by at most a few percent; the merge is not included)."""
    lib, kind = ref_lib(w)
    M = subgraph_count(w)
    S = min(cores, M)
    idx = indices if indices is not None else sample_indices(M, S)
    b = SAMPLE_BUDGET[w["key"]]
    threads = max(1, cores // min(S, M))
    out, secs = lib.solve_stage(w["n"], edges, M, idx, w["top_k"], w["layers"], b,
                                seed=w["seed"], slots=len(idx), threads=threads,
                                qubit_cap=w["qubit_cap"])
    rounds = -(-M // S)
    stage_s = rounds * secs * (w["budget"] / b)
    value = M * w["budget"] / stage_s
    desc = (f"{'oracle/_ref (unmodified qcut headers)' if kind == 'reference' else 'oracle C port'}:"
            f" {len(idx)} of {M} subgraphs (indices {idx[0]}..{idx[-1]}) solved concurrently "
            f"({threads} OpenMP thread(s) each, pipeline.hpp:223-280 round) at NM budget {b} in "
            f"{secs:.2f} s; QAOA stage at budget {w['budget']} = {rounds} rounds x "
            f"{w['budget'] // b if w['budget'] % b == 0 else w['budget'] / b} x sample = "
            f"{stage_s:.1f} s (extrapolated; merge excluded)")
    return value, desc, kind, out, idx, b, secs


def cpu_eval_microbench(cores, qs=(10, 16, 20, 24, 26)):
    """BASELINE.md section 3 step 3 / SURVEY 8(d): seconds per objective evaluation of
    the reference (run_ansatz + expectation, qaoa.hpp:89-91) at p=1 on ER(q, 0.5) subgraphs,
    1 and all host threads."""
    from oracle.refpy import RefLib, ref_available
    if not ref_available(True):
        return None
    lib = RefLib(cap26=True)
    out = []
    for q in qs:
        e = lib.generate_er(q, 0.5, q)
        for th in sorted({1, cores}):
            reps = 3 if q <= 20 else 1
            sec, _ = lib.eval_timing(q, e, [0.4], [0.9], threads=th, reps=reps)
            out.append({"q": q, "threads": th, "s_per_eval": sec,
                        "amp_layers_per_s": (1 << q) / sec})
    return out


def run_reference_arm(args, w):
    """The reference's own CPU implementation on this host, all host threads: C1/C2 are
    full-budget solves by the stock run_pipeline, timed per step; C3-C5 are the sampled
    stage of reference_sampled. A wall-clock guard keeps the run inside the driver's
    step limit: steps stop early (and "steps" says how many ran) past --ref-time-limit."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cores = os.cpu_count() or 1
    edges = workload_graph(w, reference=True)
    full = w["key"] in FULL_REFERENCE
    t_start = time.time()

    def step():
        if full:
            v, r, kind = reference_full(w, edges, cores)
            return v, r["total_s"], kind, (f"stock run_pipeline (pipeline.hpp:391) at the full NM "
                                            f"budget {w['budget']}, workers={cores}: partition "
                                            f"{r['partition_s']:.3f} s + QAOA {r['qaoa_s']:.2f} s + "
                                            f"merge {r['merge_s']:.2f} s, cut {r['cut']:.0f}"), r
        v, desc, kind, _, _, _, _ = reference_sampled(w, edges, cores)
        return v, subgraph_count(w) * w["budget"] / v, kind, desc, None

    warm_done = 0
    for _ in range(args.warmup):
        if time.time() - t_start > args.ref_time_limit / 3:
            break
        step()
        warm_done += 1
    vals, totals, desc, kind, last = [], [], None, None, None
    for _ in range(args.steps):
        el = time.time() - t_start
        per = (el / max(1, warm_done + len(vals)))
        if vals and el + per > args.ref_time_limit:
            break
        v, total, kind, desc, last = step()
        vals.append(v)
        totals.append(total)
    value = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": len(vals), "warmup": warm_done,
        "steps_requested": args.steps, "warmup_requested": args.warmup,
        "ms_per_step": statistics.median(totals) * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(w, args.gpus),
        "measured": "full solve per step" if full else "sampled stage, extrapolated",
        "extrapolated": not full,
        "step_s": [round(t, 3) for t in totals],
        "wall_s": round(time.time() - t_start, 1),
        "host": host_info(),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind,
                         "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if last is not None:
        line["result"] = {"cut": last["cut"], "candidates_evaluated": last["leaves"],
                          "assignment_sha1": __import__("hashlib").sha1(
                              last["assignment"].encode()).hexdigest()}
    print(json.dumps(line), flush=True)
    return 0


def parity_full(w, edges, cores, rep, records):
    """cpu_baseline for C1/C2 plus the parity block: the reference's stock run_pipeline at
    the full budget (timed -> cpu_baseline) and every SolveResult of its QAOA stage
    (ref_solve_stage) against the GPU's timed run (the cut, assignment, leaves of the last
    timed step; the SolveResults of the resident session, qc_pipeline_records)."""
    value, r, kind = reference_full(w, edges, cores)
    lib, _ = ref_lib(w)
    M = r["subgraphs"]
    want, _ = lib.solve_stage(w["n"], edges, M, list(range(M)), w["top_k"], w["layers"],
                              w["budget"], seed=w["seed"], slots=min(cores, M), threads=1,
                              qubit_cap=w["qubit_cap"])
    L = w["layers"]
    same = [bool(g.width == o.width and np.array_equal(g.bits, o.bits) and
                 np.array_equal(g.probs, o.probs) and np.array_equal(g.params[:2 * L], o.params[:2 * L])
                 and g.expectation == o.expectation and g.evals == o.evals)
            for g, o in zip(records, want)]
    parity = {
        "checker": "oracle/_ref stock run_pipeline + ref_solve_stage" if kind == "reference"
        else "oracle C port",
        "budget": w["budget"], "subgraphs": M,
        "cut": [rep.cut, r["cut"]], "cut_equal": rep.cut == r["cut"],
        "assignment_equal": rep.assignment == r["assignment"],
        "candidates_evaluated_equal": rep.candidates_evaluated == r["leaves"],
        "expectations_equal": [x.expectation for x in records] == list(r["sub_expectation"]),
        "evals_equal": [x.evals for x in records] == list(r["sub_evals"]),
        "solve_results_equal": sum(same), "solve_results_compared": len(same),
    }
    parity["all_equal"] = bool(parity["cut_equal"] and parity["assignment_equal"] and
                               parity["candidates_evaluated_equal"] and parity["expectations_equal"]
                               and parity["evals_equal"] and all(same) and len(same) == M)
    desc = (f"{'oracle/_ref (unmodified qcut headers)' if kind == 'reference' else 'oracle C port'}"
            f" stock run_pipeline, one full solve at NM budget {w['budget']}, workers={cores}: "
            f"partition {r['partition_s']:.3f} s + QAOA {r['qaoa_s']:.2f} s + merge "
            f"{r['merge_s']:.2f} s = {r['total_s']:.2f} s")
    return {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": desc}, parity


def parity_sampled(eng, w, edges, cores):
    """cpu_baseline for C3-C5 (reference_sampled) plus the parity block: the same sampled
    subgraphs solved by the product at the sample budget, every SolveResult identical."""
    from paper_2603_26232_b200 import partition_chain
    value, desc, kind, want, idx, b, _ = reference_sampled(w, edges, cores)
    P = partition_chain(w["n"], edges, subgraph_count(w), 0, w["qubit_cap"])
    graphs, opts = [], []
    for i in idx:
        nl, le = P.local[i]
        k = min(1 << (nl - 1), w["top_k"]) if w["top_k"] else 1 << (nl - 1)
        graphs.append((nl, le))
        opts.append(dict(top_k=k, layers=w["layers"], budget=b, seed=w["seed"] + i,
                         qubit_cap=w["qubit_cap"]))
    got = eng.solve_batch(graphs, opts)
    L = w["layers"]
    same = [bool(g.width == o.width and np.array_equal(g.bits, o.bits) and
                 np.array_equal(g.probs, o.probs) and np.array_equal(g.params[:2 * L], o.params[:2 * L])
                 and g.expectation == o.expectation and g.evals == o.evals)
            for g, o in zip(got, want)]
    parity = {"checker": "oracle/_ref ref_solve_stage" if kind == "reference" else "oracle C port",
              "sampled_subgraphs": idx, "budget": b, "solve_results_equal": sum(same),
              "solve_results_compared": len(same), "all_equal": all(same) and len(same) == len(idx),
              "note": "full-budget sampled solves of this workload: tests/test_gpu_configs.py"}
    return {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": desc}, parity


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
    ap.add_argument("--mixer", default="rx", choices=["rx", "wht"],
                    help="fp32 mode's mixer form: rx (mixer_pair rotations, default) or wht "
                         "(Walsh-Hadamard: H diag H with add/sub butterflies; --precision 32)")
    ap.add_argument("--report", default="",
                    help="also write the run as an ExperimentReport JSON v1 (report.hpp) with a "
                         "'gpu' section to this path")
    ap.add_argument("--profile-stride", type=int, default=PROFILE_STRIDE,
                    help="CUDA-event sampling of 1 launch in N during the timed region (0: off)")
    ap.add_argument("--ref-time-limit", type=float, default=1500.0,
                    help="reference arm: stop starting steps past this many seconds")
    ap.add_argument("--no-cpu-microbench", action="store_true",
                    help="skip the per-eval CPU microbenchmark of the cpu_baseline leg")
    args = ap.parse_args()
    w = dict(WORKLOADS[args.workload])
    w["key"] = args.workload
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
    if args.mixer != "rx":
        eng.set_mixer(args.mixer)
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
    sess = None
    if world == 1:
        sess = eng.prepare_pipeline(w["n"], edges, **cfg)
        M = None

        def step_value():
            return sess.execute()
    else:
        from paper_2603_26232_b200.distributed import ShardedSession
        M = eng.subgraph_count(w["n"], edges, **cfg)
        # resident like N=1: partition + this rank's cut tables once (qc_pipeline_prepare with
        # shard_count = world), then per step: this rank's block of the QAOA stage, one NCCL
        # all-gather of the solve records, merge on rank 0 with the session's partition
        shard = ShardedSession(eng, w["n"], edges, rank, world, device=coll_dev, **cfg)

        def step_value():
            return shard.step()

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
    # the timed region runs exactly as production does (CUDA-graph replay of every chunk
    # step; no profiling events)
    t_val, rep, launches, _ = timed(step_value, args.steps)
    tv1 = eng.transfers()
    clk = clocks.stop()
    host = eng.host_stats(reset=True)
    # the same K steps again with one launch in --profile-stride bracketed by CUDA events on
    # its stream (direct launches: events are not captured into the replayed graphs)
    _, _, _, profile = timed(step_value, args.steps, prof=True)

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
    fp_tag = "f64" if args.precision == 64 else "f32"
    traffic, traffic_src = None, None
    try:  # ncu DRAM bytes of THIS workload's dominant kernel (tools/ncu_traffic.py)
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f).get(f"{w['key']}/{fp_tag}/{dom}")
        if tr and tr.get("traffic_over_algorithmic") and d["launches"]:
            # ncu's DRAM/algorithmic ratio for the same kernel at this workload's launch
            # shape, times this step's algorithmic bytes per launch
            traffic = tr["traffic_over_algorithmic"] * d["bytes"] / d["launches"]
            traffic_src = (f"{tr.get('source')}; DRAM/algorithmic = "
                           f"{tr['traffic_over_algorithmic']:.3f} x this step's algorithmic "
                           f"bytes per launch")
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
    kernels = {k: {"launches": v["launches"], "ms": round(v["ms"], 3),
                   "GB/s": round(v["bytes"] / (v["ms"] / 1e3) / 1e9, 1) if v["ms"] > 0 else 0.0,
                   "fp64_Tops": round(v.get("fp64_ops", 0.0) / (v["ms"] / 1e3) / 1e12, 2)
                   if v["ms"] > 0 else 0.0}
               for k, v in profile_iso.items() if v["launches"]}
    common = {"kernel": dom, "avg_launch_ms": d["ms"] / max(d["launches"], 1),
              "measured": "every launch of one single-stream step, CUDA events on its stream",
              "launches": d["launches"], "share_of_step": d["ms"] / iso_ms if iso_ms else None,
              "kernels": kernels,
              "step_aggregate_GBs": iso_bytes / sec_per_step / 1e9,
              "step_aggregate_frac": iso_bytes / sec_per_step / 1e9 / peak,
              "timed_region_sampled": {
                  "stride": args.profile_stride, "streams": 2,
                  "note": "a second pass of the K timed steps with sampled per-launch events "
                          "(concurrent chunks stretch each launch's event span)",
                  "kernels": {k: {"launches": v["launches"], "ms": round(v["ms"], 3),
                                  "GB/s": round(v["bytes"] / (v["ms"] / 1e3) / 1e9, 1)
                                  if v["ms"] > 0 else 0.0}
                              for k, v in profile.items() if v["launches"]}}}
    if dom == "onchip":
        # whole subgraph state in one CTA's shared memory for every layer: no HBM stream,
        # the ceiling is the FP64 pipe (explicit DMUL/DADD, no FMA) — and dependent latency
        roofline = {"bound": "fp64", "achieved": fp64_ach, "peak": fp64_peak, "unit": "Tops/s",
                    "frac": fp64_ach / fp64_peak, "traffic": traffic,
                    "peak_source": "measured: tools/ubench_fp64.cu mixer_pair pattern "
                                   "(profiles/r1_ubench_fp64.txt)",
                    "algorithmic_fp64_ops_per_launch": d.get("fp64_ops", 0.0) / max(d["launches"], 1),
                    "note": "on-chip kernel (Q <= 12): HBM is not touched between layers, so an HBM "
                            "fraction is meaningless; FP64 issue and latency bound it", **common}
    else:
        roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                    "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)" if peak_kind ==
                    "measured" else "fallback (B200_PROFILING.md)",
                    "algorithmic_bytes_per_launch": d["bytes"] / max(d["launches"], 1),
                    # streaming efficiency without the per-launch fixed cost (see steady_state)
                    "steady_state": ss,
                    # the fp64 parity path forbids FMA: every butterfly is 8 DMUL + 4 DADD, so
                    # the FP64 pipe is the second ceiling (co-bound for the 12-target pass A)
                    "fp64": {"achieved_tops": fp64_ach, "peak_tops": fp64_peak,
                             "frac": fp64_ach / fp64_peak,
                             "ops_per_launch": d.get("fp64_ops", 0.0) / max(d["launches"], 1),
                             "peak_source": "measured: tools/ubench_fp64.cu mixer_pair pattern "
                                            "(profiles/r1_ubench_fp64.txt)"},
                    **common}
    q = w["qubit_cap"]
    amp_b = 16 if args.precision == 64 else 8
    ws = subgraph_count(w) * (1 << (q - 1)) * (amp_b + amp_b // 2)
    l2 = (f"per-step working set {ws / 2**20:.0f} MiB (states + f of {subgraph_count(w)} "
          f"half-states of {q} qubits) {'>' if ws > 126 * 2**20 else '<'} 126 MB L2; "
          f"L2 flushed (256 MB write) before every timed step")
    if dom == "onchip":
        l2 = (f"on-chip kernel: each {q}-qubit state lives in shared memory for the whole eval; "
              f"inputs ({ws / 2**10:.0f} KiB) come from L2; L2 flushed (256 MB write) before "
              f"every timed step")

    line = {
        "metric": METRIC, "value": evals_per_step / sec_per_step, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec_per_step * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64" if args.precision == 64 else "f32",
        "data": "synthetic (graph.hpp:146 ER generator restated in qc_generate_er)",
        "config": config_dict(w, world), "l2": l2, "mixer": args.mixer,
        "solve_time_s": sec_per_step, "cut": rep.cut, "evals_per_step": evals_per_step,
        "step_ms": [round(t * 1e3, 2) for t in t_val],
        "host_s_per_step": {k: (v / args.steps if k != "chunk_steps" else v // args.steps)
                            for k, v in host.items()},
        "stage_s": {"partition": rep.partition_s, "qaoa": rep.qaoa_s, "merge": rep.merge_s},
        "e2e": e2e, "gpu_launches": int(lt.item()), "clocks": clk, "roofline": roofline,
    }
    if world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        try:
            ref_edges = workload_graph(w, reference=True)
            if w["key"] in FULL_REFERENCE:
                cb, parity = parity_full(w, ref_edges, cores, rep, sess.records())
            else:
                cb, parity = parity_sampled(eng, w, ref_edges, cores)
            line["cpu_baseline"], line["parity"] = cb, parity
        except Exception as ex:  # report, never fail the bench line
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": cores,
                                    "kind": "unavailable", "sample": repr(ex)[:300]}
        line["cpu_baseline"]["host"] = host_info()
        if not args.no_cpu_microbench and w["key"] == "c2":
            try:
                line["cpu_baseline"]["per_eval"] = cpu_eval_microbench(cores)
            except Exception as ex:
                line["cpu_baseline"]["per_eval"] = repr(ex)[:200]
    print(json.dumps(line), flush=True)
    if args.report and rep is not None:
        from paper_2603_26232_b200.report import emit_report, experiment_report
        doc = experiment_report(
            rep, n=w["n"], edges=len(edges), cfg=dict(cfg, shard_count=world), generated=True,
            p=w.get("p_edge", 0.0), graph_seed=w["seed"],
            gpu={"device": torch.cuda.get_device_name(local), "n_gpus": world,
                 "precision": f"fp{args.precision}", "evals_per_s": line["value"],
                 "e2e_evals_per_s": e2e["value"], "ms_per_step": line["ms_per_step"],
                 "roofline": {"kernel": roofline["kernel"], "bound": roofline["bound"],
                              "frac": roofline["frac"],
                              "fp64_frac": roofline.get("fp64", roofline)["frac"]},
                 "clocks": clk})
        with open(args.report, "w") as f:
            f.write(emit_report(doc))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
