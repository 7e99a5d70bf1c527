"""Parameter-grid sweep on the GPU, mirroring the reference CLI's `sweep` command
(qcut_main.cpp:213-290): a JSON grid object of scalar run settings plus list axes, one
ER(n, p, seed) instance per point, one `csv_header()` line then one `csv_row()` per point
(report.hpp:311-331), axes nested n > p > seed > top_k > merge_level. Alongside the CSV,
an optional JSON-lines sidecar carries the GPU fields per point (evals/s, stage times).

    python -m paper_2603_26232_b200.sweep grid.json out.csv [--jsonl out.jsonl] [--repeat 2]

Grid keys (qcut_main.cpp:232-258): scalars qubits, solvers (ignored: one engine), subgraphs,
layers, budget, alpha, workers (ignored), fold, halve_symmetry, path_budget, partition
("balanced" | "paper-exact"); axes n [20], p [0.5], seed [0], top_k [2], merge_level [1]
(a scalar is a one-element axis). Unlike the reference (nlohmann with comments
allowed) the grid must be plain JSON. The "baseline" metrics (AR/EF/PEI) are out of scope:
their CSV cells stay empty, as in a reference run without a baseline.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from typing import Any, Callable, Iterable

from . import ConfigError, IoError

_SCALARS = {"qubits": ("qubit_cap", int), "subgraphs": ("subgraphs", int),
            "layers": ("layers", int), "budget": ("budget", int), "alpha": ("alpha", float),
            "fold": ("fold", bool), "halve_symmetry": ("halve_symmetry", bool),
            "path_budget": ("path_budget", float), "solvers": (None, int),
            "workers": (None, int)}
_AXES = (("n", [20], int), ("p", [0.5], float), ("seed", [0], int), ("top_k", None, int),
         ("merge_level", None, int))


def parse_grid(grid: Any, base: dict | None = None) -> tuple[dict, list[dict]]:
    """qcut_main.cpp:222-270: (run settings, [points]). ConfigError on bad types or an
    empty axis, IoError if the grid is not a JSON object."""
    if not isinstance(grid, dict):
        raise IoError("grid file must hold a JSON object")
    cfg = dict(base or {})
    cfg.setdefault("top_k", 2)
    cfg.setdefault("start_level", 1)
    for key, (name, typ) in _SCALARS.items():
        if key in grid:
            v = grid[key]
            if isinstance(v, list) or (typ is not bool and isinstance(v, bool)) or \
                    (typ is bool and not isinstance(v, bool)) or \
                    (typ in (int, float) and not isinstance(v, (int, float))) or \
                    (typ is int and isinstance(v, float) and not v.is_integer()):
                raise ConfigError(f"grid scalar has the wrong type: {key}")
            if name:
                cfg[name] = typ(v)
    if "partition" in grid:
        mode = grid["partition"]
        if mode not in ("balanced", "paper-exact"):
            raise ConfigError("grid 'partition' must be balanced or paper-exact")
        cfg["partition_mode"] = 0 if mode == "balanced" else 1
    axes = []
    for key, fallback, typ in _AXES:
        if fallback is None:
            fallback = [cfg["top_k"] if key == "top_k" else cfg["start_level"]]
        v = grid.get(key, fallback)
        if not isinstance(v, list):
            v = [v]
        if not v:
            raise ConfigError(f"grid axis '{key}' is empty")
        for x in v:
            if isinstance(x, bool) or not isinstance(x, (int, float)) or \
                    (typ is int and isinstance(x, float) and not x.is_integer()):
                raise ConfigError(f"grid axis has the wrong type: {key}")
        axes.append([typ(x) for x in v])
    points = [dict(n=n, p=p, seed=s, top_k=k, start_level=lv)
              for n in axes[0] for p in axes[1] for s in axes[2] for k in axes[3] for lv in axes[4]]
    return cfg, points


def run_sweep(grid: Any, out, engine=None, jsonl=None, repeat: int = 1,
              runner: Callable[[dict, dict], tuple] | None = None) -> int:
    """Write the sweep CSV to `out` (a text stream). runner(cfg, point) -> (RunReport,
    edge count) defaults to the GPU pipeline (qc_run_pipeline); with repeat > 1 the last
    run is reported (the first pays table builds and first-touch)."""
    from .report import csv_header, csv_row, experiment_report
    cfg, points = parse_grid(grid)
    if runner is None:
        from . import Engine, generate_er
        eng = engine or Engine(0)

        def runner(run_cfg, pt):
            edges = generate_er(pt["n"], pt["p"], pt["seed"])
            rep = None
            for _ in range(max(1, repeat)):
                rep = eng.run_pipeline(pt["n"], edges, **run_cfg)
            return rep, len(edges)
    out.write(csv_header() + "\n")
    out.flush()
    for pt in points:
        run_cfg = dict(cfg, top_k=pt["top_k"], start_level=pt["start_level"])
        t0 = time.perf_counter()
        rep, m = runner(run_cfg, pt)
        wall = time.perf_counter() - t0
        doc = experiment_report(rep, n=pt["n"], edges=m, cfg=run_cfg, p=pt["p"],
                                graph_seed=pt["seed"])
        out.write(csv_row(doc) + "\n")
        out.flush()
        if jsonl is not None:
            qaoa = float(rep.qaoa_s)
            jsonl.write(json.dumps({"n": pt["n"], "p": pt["p"], "seed": pt["seed"],
                                    "top_k": pt["top_k"], "merge_level": pt["start_level"],
                                    "qubit_cap": run_cfg.get("qubit_cap", 20),
                                    "layers": run_cfg.get("layers", 3), "edges": m,
                                    "subgraphs": int(rep.subgraphs), "cut": float(rep.cut),
                                    "evals": int(rep.evals), "windowed": bool(rep.windowed),
                                    "total_s": float(rep.total_s), "qaoa_s": qaoa,
                                    "merge_s": float(rep.merge_s),
                                    "evals_per_s": rep.evals / qaoa if qaoa > 0 else None,
                                    "wall_s_incl_generation": wall}) + "\n")
            jsonl.flush()
    return len(points)


def main(argv: Iterable[str] | None = None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("grid")
    ap.add_argument("out", nargs="?", default="-")
    ap.add_argument("--jsonl", default=None)
    ap.add_argument("--repeat", type=int, default=2)
    a = ap.parse_args(list(argv) if argv is not None else None)
    try:
        with open(a.grid) as f:
            grid = json.load(f)
    except OSError as ex:
        raise IoError(f"cannot open grid file: {a.grid}") from ex
    except ValueError as ex:
        raise IoError(f"grid file is not valid JSON: {ex}") from ex
    out = sys.stdout if a.out == "-" else open(a.out, "w")
    side = open(a.jsonl, "w") if a.jsonl else None
    try:
        run_sweep(grid, out, jsonl=side, repeat=a.repeat)
    finally:
        if out is not sys.stdout:
            out.close()
        if side:
            side.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
