"""ExperimentReport JSON v1 + sweep CSV for GPU runs (report.hpp:16-331).

The same document the reference's CLI writes (`to_json`, report.hpp:110-194), built from a
GPU pipeline run, plus one extra top-level object "gpu" (device, shards, evals/s,
amp-layers/s, precision, roofline, per-GPU times) that the reference's `parse_report`
ignores. The round trip through the reference's own parser and its `csv_row` is checked in
tests/test_cpu_report.py.
"""
from __future__ import annotations

import json
import math
import os
from typing import Any

SCHEMA_VERSION = 1

_PARTITION = {0: "balanced", 1: "paper-exact"}


def format_weight(w: float) -> str:
    """graph.hpp:174-179 detail::format_weight = std::to_chars(double): the shortest
    round-trip digits, fixed or scientific notation whichever is shorter (fixed on ties)."""
    w = float(w)
    if math.isnan(w) or math.isinf(w):
        return {True: "inf", False: "-inf"}[w > 0] if math.isinf(w) else "nan"
    if w == 0.0:
        return "-0" if math.copysign(1.0, w) < 0 else "0"
    r = repr(w)  # shortest round-trip digits
    sign = "-" if w < 0 else ""
    mant, _, exp = r.lstrip("-").partition("e")
    digits = mant.replace(".", "")
    point = mant.index(".") if "." in mant else len(mant)
    e10 = (int(exp) if exp else 0) + point - 1  # decimal exponent of the first digit
    stripped = digits.lstrip("0")
    e10 -= len(digits) - len(stripped)
    digits = stripped.rstrip("0") or "0"
    # fixed
    if e10 >= 0:
        ip = digits[: e10 + 1].ljust(e10 + 1, "0")
        fp = digits[e10 + 1:]
        fixed = ip + ("." + fp if fp else "")
    else:
        fixed = "0." + "0" * (-e10 - 1) + digits
    # scientific (exponent with sign and at least two digits)
    sci = digits[0] + ("." + digits[1:] if len(digits) > 1 else "") + \
        "e" + ("-" if e10 < 0 else "+") + f"{abs(e10):02d}"
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def experiment_report(run, *, n: int, edges: int, cfg: dict, generated: bool = True,
                      p: float = 0.0, graph_seed: int = 0, graph_file: str = "",
                      subgraphs: list[dict] | None = None, status: str = "ok",
                      error_stage: str = "", error_message: str = "",
                      gpu: dict | None = None) -> dict:
    """report.hpp:110-194 to_json for a GPU run.

    run: paper_2603_26232_b200.RunReport (cut, assignment, evals, subgraphs, windowed,
    candidates_evaluated, partition_s/qaoa_s/merge_s/total_s); cfg: the run_config keywords
    (Engine.run_config names). The schedule section reports the lockstep batch: one round in
    which every subgraph is in flight (rounds=1, slots=max_concurrent=M).
    """
    M = int(run.subgraphs) if run is not None else int(cfg.get("subgraphs", 0))
    d: dict[str, Any] = {"schema_version": SCHEMA_VERSION, "status": status}
    graph: dict[str, Any] = {"n": int(n), "edges": int(edges), "generated": bool(generated)}
    if generated:
        graph["p"] = float(p)
        graph["seed"] = int(graph_seed)
    else:
        graph["file"] = graph_file
    d["graph"] = graph
    merge_mode = {1: "level", 2: "windowed"}.get(int(cfg.get("merge_mode", 0)))
    if merge_mode is None:
        merge_mode = "windowed" if (run is not None and run.windowed) else "level"
    d["config"] = {
        "qubit_cap": int(cfg.get("qubit_cap", 20)),
        "subgraphs": M,
        "solvers": int(cfg.get("shard_count", 1)),
        "workers": int(cfg.get("workers", 1)),
        "top_k": int(cfg.get("top_k", 2)),
        "start_level": int(cfg.get("start_level", 1)),
        "layers": int(cfg.get("layers", 3)),
        "budget": int(cfg.get("budget", 200)),
        "seed": int(cfg.get("seed", 0)),
        "alpha": float(cfg.get("alpha", 0.0)),
        "fold": bool(cfg.get("fold", True)),
        "halve_symmetry": bool(cfg.get("halve_symmetry", False)),
        "partition_mode": _PARTITION.get(int(cfg.get("partition_mode", 0)), "balanced"),
        "merge_eval": "incremental" if cfg.get("merge_incremental", 1) else "full",
        "merge_mode": merge_mode,
        "baseline": str(cfg.get("baseline", "value")),
        "path_budget": float(cfg.get("path_budget", 1e9)),
        "nm_tolerance": float(cfg.get("nm_tolerance", 1e-5)),
        "local_restarts": int(cfg.get("local_restarts", 0)),
    }
    if run is not None:
        d["schedule"] = {"rounds": 1, "slots": M, "max_concurrent": M}
    if subgraphs:
        d["subgraphs"] = [{"index": int(s["index"]), "size": int(s["size"]),
                           "retained": int(s["retained"]), "expectation": float(s["expectation"]),
                           "evals": int(s["evals"]), "seconds": float(s.get("seconds", 0.0))}
                          for s in subgraphs]
    if run is not None and status == "ok":
        d["merge"] = {"best_value": float(run.cut), "assignment": run.assignment,
                      "candidates_evaluated": int(run.candidates_evaluated),
                      "validated": True}  # the device re-scores the winner (merge.hpp:327,408)
    t = {"partition_s": 0.0, "qaoa_s": 0.0, "merge_s": 0.0, "baseline_s": 0.0, "total_s": 0.0}
    if run is not None:
        t.update(partition_s=float(run.partition_s), qaoa_s=float(run.qaoa_s),
                 merge_s=float(run.merge_s),
                 total_s=float(run.partition_s + run.qaoa_s + run.merge_s))
    d["times"] = t
    d["environment"] = {"hardware_threads": os.cpu_count() or 1, "openmp": False,
                        "compiler": "nvcc 12.9 sm_100a + g++ (libqcgpu.so)"}
    if status == "error":
        d["error"] = {"stage": error_stage, "message": error_message}
    if gpu:
        d["gpu"] = gpu
    return d


def emit_report(d: dict) -> str:
    """report.hpp:196 emit_report: indented JSON and a trailing newline."""
    return json.dumps(d, indent=2) + "\n"


_REQUIRED = {
    "graph": ("n", "edges", "generated"),
    "config": ("qubit_cap", "subgraphs", "solvers", "workers", "top_k", "start_level", "layers",
               "budget", "seed", "alpha", "fold", "halve_symmetry", "partition_mode",
               "merge_eval", "merge_mode", "baseline", "path_budget", "nm_tolerance",
               "local_restarts"),
    "times": ("partition_s", "qaoa_s", "merge_s", "baseline_s", "total_s"),
}


def parse_report(text: str) -> dict:
    """report.hpp:200-309 parse_report: the same required fields, IoError otherwise."""
    from . import IoError
    try:
        d = json.loads(text)
    except ValueError as ex:
        raise IoError(f"report is not valid JSON: {ex}") from None
    try:
        if d["schema_version"] != SCHEMA_VERSION:
            raise IoError(f"unsupported report schema_version {d['schema_version']}")
        d["status"]
        for sec, keys in _REQUIRED.items():
            for k in keys:
                d[sec][k]
        d["graph"]["p" if d["graph"]["generated"] else "file"]
        if d["status"] == "error":
            d["error"]["stage"], d["error"]["message"]
    except (KeyError, TypeError) as ex:
        raise IoError(f"report is missing required fields: {ex}") from None
    return d


def csv_header() -> str:
    """report.hpp:311-313."""
    return "n,p,seed,M,K,L,cut,ar,ef,pei,partition_s,qaoa_s,merge_s,baseline_s,total_s"


def csv_row(d: dict) -> str:
    """report.hpp:316-331 (graphs loaded from files leave p and seed empty)."""
    g, c, t = d["graph"], d["config"], d["times"]
    num = format_weight
    cells = [str(g["n"]), num(g["p"]) if g["generated"] else "",
             str(g["seed"]) if g["generated"] else "", str(c["subgraphs"]), str(c["top_k"]),
             str(c["start_level"]), num(d["merge"]["best_value"]) if "merge" in d else ""]
    m = d.get("metrics")
    cells += [num(m["ar"]) if m else "", num(m["ef"]) if m else "", num(m["pei"]) if m else ""]
    cells += [num(t["partition_s"]), num(t["qaoa_s"]), num(t["merge_s"]), num(t["baseline_s"]),
              num(t["total_s"])]
    return ",".join(cells)
