"""Sweep grid (paper_2603_26232_b200/sweep.py) vs the reference CLI's cmd_sweep
(qcut_main.cpp:213-290): defaults, axis order, error types, CSV layout. No GPU: the
pipeline is replaced by a stub runner."""
import io

import pytest

from paper_2603_26232_b200 import ConfigError, IoError, RunReport
from paper_2603_26232_b200.report import csv_header
from paper_2603_26232_b200.sweep import parse_grid, run_sweep


def test_defaults_match_cmd_sweep():
    cfg, pts = parse_grid({})
    assert pts == [dict(n=20, p=0.5, seed=0, top_k=2, start_level=1)]  # :256-260
    assert cfg["top_k"] == 2 and cfg["start_level"] == 1


def test_scalars_and_axis_nesting_order():
    cfg, pts = parse_grid({"qubits": 16, "layers": 2, "budget": 50, "partition": "paper-exact",
                           "n": [400, 800], "p": [0.1, 0.3], "seed": 7, "top_k": [2, 4]})
    assert cfg["qubit_cap"] == 16 and cfg["layers"] == 2 and cfg["budget"] == 50
    assert cfg["partition_mode"] == 1
    assert len(pts) == 8
    # n outermost, then p, seed, top_k, merge_level (qcut_main.cpp:270-274)
    assert [(x["n"], x["p"], x["top_k"]) for x in pts[:4]] == \
        [(400, 0.1, 2), (400, 0.1, 4), (400, 0.3, 2), (400, 0.3, 4)]
    assert all(x["seed"] == 7 and x["start_level"] == 1 for x in pts)


@pytest.mark.parametrize("grid,err", [
    ([1, 2], IoError),                       # not an object
    ({"p": []}, ConfigError),                # empty axis
    ({"n": ["a"]}, ConfigError),             # axis type
    ({"qubits": "20"}, ConfigError),         # scalar type
    ({"fold": 1}, ConfigError),              # bool scalar
    ({"partition": "greedy"}, ConfigError),  # partition mode
])
def test_grid_errors(grid, err):
    with pytest.raises(err):
        parse_grid(grid)


def test_csv_header_then_one_row_per_point():
    seen = []

    def runner(cfg, pt):
        seen.append((pt["n"], pt["p"], cfg["top_k"]))
        rep = RunReport(cut=float(pt["n"]), candidates_evaluated=4, partition_s=0.001,
                        qaoa_s=0.01, merge_s=0.002, total_s=0.013, subgraphs=2, windowed=False,
                        evals=400, assignment="0" * pt["n"])
        return rep, 3 * pt["n"]
    out, side = io.StringIO(), io.StringIO()
    n = run_sweep({"n": [10, 12], "p": 0.3, "top_k": [1, 3], "qubits": 10}, out, jsonl=side,
                  runner=runner)
    lines = out.getvalue().splitlines()
    assert n == 4 and len(lines) == 5 and lines[0] == csv_header()
    assert seen == [(10, 0.3, 1), (10, 0.3, 3), (12, 0.3, 1), (12, 0.3, 3)]
    cells = lines[1].split(",")
    assert cells[:7] == ["10", "0.3", "0", "2", "1", "1", "10"]  # n,p,seed,M,K,L,cut
    assert cells[7:10] == ["", "", ""]                           # no baseline metrics
    assert len(side.getvalue().splitlines()) == 4
