"""ExperimentReport JSON v1 / CSV (report.hpp) written by the product for GPU runs.

Checked against the reference's own parse_report / emit_report / csv_row (oracle/_ref/
report_rt, compiled from report.hpp where /root/reference exists): the document parses
unchanged, every reference field survives the round trip, and the CSV row is identical.
"""
import json
import math
import os
import subprocess

import pytest

from paper_2603_26232_b200 import IoError, RunReport
from paper_2603_26232_b200.report import (csv_header, csv_row, emit_report, experiment_report,
                                          format_weight, parse_report)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RT = os.path.join(ROOT, "oracle", "_ref", "report_rt")


def sample(status="ok", generated=True):
    run = RunReport(cut=4258.0, candidates_evaluated=4194304, partition_s=2.8e-05,
                    qaoa_s=0.0758, merge_s=0.00103, total_s=0.0768, subgraphs=21,
                    windowed=False, evals=4200, assignment="01" * 200)
    cfg = dict(qubit_cap=20, top_k=2, layers=2, budget=200, seed=0, nm_tolerance=1e-5)
    gpu = {"device": "NVIDIA B200", "n_gpus": 1, "precision": "fp64", "evals_per_s": 55301.9,
           "roofline": {"kernel": "pass_low", "hbm_frac": 0.434, "fp64_frac": 0.457}}
    subs = [{"index": i, "size": 20, "retained": 2, "expectation": 10.5 + i / 7,
             "evals": 200, "seconds": 0.0} for i in range(3)]
    return experiment_report(run, n=400, edges=8021, cfg=cfg, generated=generated, p=0.1,
                             graph_seed=0, graph_file="g.txt", subgraphs=subs, status=status,
                             error_stage="merge" if status == "error" else "",
                             error_message="boom" if status == "error" else "", gpu=gpu)


def test_python_round_trip_and_required_fields():
    d = sample()
    back = parse_report(emit_report(d))
    assert back == json.loads(emit_report(d))
    assert back["gpu"]["precision"] == "fp64"
    bad = json.loads(emit_report(d))
    del bad["times"]["qaoa_s"]
    with pytest.raises(IoError):
        parse_report(json.dumps(bad))
    with pytest.raises(IoError):
        parse_report("{not json")


@pytest.mark.parametrize("w,s", [(296.0, "296"), (0.1, "0.1"), (1e-05, "1e-05"),
                                  (100000.0, "1e+05"), (123456.0, "123456"), (0.0758, "0.0758"),
                                  (2.8e-05, "2.8e-05"), (1.5, "1.5"), (-3.25, "-3.25"),
                                  (1e22, "1e+22"), (4194304.0, "4194304")])
def test_format_weight_matches_to_chars(w, s):
    assert format_weight(w) == s


@pytest.mark.skipif(not os.path.exists(RT), reason="reference report.hpp driver not built")
@pytest.mark.parametrize("status,generated", [("ok", True), ("ok", False), ("error", True)])
def test_reference_parser_reads_product_reports(status, generated):
    d = sample(status, generated)
    out = subprocess.run([RT], input=emit_report(d), capture_output=True, text=True, check=True)
    body, csv_line, hdr_line = out.stdout.rsplit("\n", 3)[0], *out.stdout.rsplit("\n", 3)[1:3]
    ref = json.loads(body)
    for key, val in ref.items():  # every field the reference knows survives unchanged
        if isinstance(val, dict):
            for k, v in val.items():
                mine = d[key][k]
                assert (mine == v) or (isinstance(v, float) and math.isclose(mine, v, rel_tol=0,
                                                                            abs_tol=0)), (key, k)
        elif isinstance(val, list):
            assert val == d[key]
        else:
            assert d[key] == val
    assert csv_line == "CSV:" + csv_row(d)
    assert hdr_line == "HDR:" + csv_header()
    assert "gpu" not in ref  # the extra section is ignored by the reference
