"""Multi-GPU paths on one B200 (the only GPU count gpurun offers): the sharded QAOA stage
must give the single-GPU result bit for bit — cut, assignment, leaf count, evals.

* qc_run_pipeline_multi: one process, n engines (one host thread each), NCCL record gather
  (n=1 here: ncclCommInitAll on cuda:0) or, for engines sharing a device, host gather.
* qc_comm_create / qc_gather_topk: the per-rank NCCL gather entry point (nranks=1).
* torchrun, 2 ranks on cuda:0 with gloo: distributed.solve_sharded, the bench's N>1 step.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _same(a, b):
    assert a.cut == b.cut
    assert a.assignment == b.assignment
    assert a.candidates_evaluated == b.candidates_evaluated
    assert a.evals == b.evals and a.subgraphs == b.subgraphs


C1 = dict(qubit_cap=10, top_k=4, layers=1, budget=200, seed=0)


def test_pipeline_multi_host_gather_two_engines(engine):
    from paper_2603_26232_b200 import Engine, generate_er, run_pipeline_multi
    e = generate_er(100, 0.1, 0)
    single = engine.run_pipeline(100, e, **C1)
    assert single.cut == 296.0
    other = Engine(0)
    try:
        for k in (2, 3):
            _same(run_pipeline_multi([engine] + [other] * (k - 1), 100, e, **C1), single)
    finally:
        other.close()


def test_pipeline_multi_nccl_one_gpu(engine):
    from paper_2603_26232_b200 import Comm, generate_er, run_pipeline_multi
    e = generate_er(100, 0.1, 0)
    single = engine.run_pipeline(100, e, **C1)
    comms = Comm.create_all([engine])
    try:
        assert comms[0].rank() == (0, 1)
        _same(run_pipeline_multi([engine], 100, e, comms=comms, **C1), single)
    finally:
        for c in comms:
            c.close()


def test_gather_topk_nccl_rank(engine):
    """qc_comm_id -> qc_comm_create -> qc_gather_topk with the real record geometry."""
    from paper_2603_26232_b200 import Comm, generate_er, unpack_records
    e = generate_er(100, 0.1, 0)
    rb, M = engine.run_record_bytes(100, e, **C1)
    local = engine.shard_solve(100, e, 0, M, rb, **C1)
    comm = Comm.create(engine, 1, 0, Comm.unique_id())
    try:
        allrec = comm.gather_topk(local, M, M, rb)
    finally:
        comm.close()
    assert np.array_equal(allrec, local)
    recs = unpack_records(allrec, M, rb, 1)
    assert [len(r.bits) for r in recs] == [4] * M and all(r.evals == 200 for r in recs)
    assert list(recs[0].bits) == [72, 584, 328, 840]  # SURVEY Appendix E, subgraph 0
    rep = engine.merge_records(100, e, allrec, M, **C1)
    assert rep.cut == 296.0


def test_sharded_narrow_pieces_all_classes(engine):
    """pieces narrower than the cap (n=30, cap 20 -> widths 16, 15) with top_k=0
    (every class retained): records are sized from the partition, not the cap."""
    from paper_2603_26232_b200 import generate_er, run_pipeline_multi, Engine
    e = generate_er(30, 0.3, 4)
    cfg = dict(qubit_cap=20, top_k=0, layers=1, budget=20, seed=3)
    single = engine.run_pipeline(30, e, **cfg)
    other = Engine(0)
    try:
        _same(run_pipeline_multi([engine, other], 30, e, **cfg), single)
    finally:
        other.close()


@pytest.mark.parametrize("mode", ["oneshot", "session"])
@pytest.mark.parametrize("n,p,cfg", [
    (400, 0.1, dict(qubit_cap=20, top_k=2, layers=2, budget=8, seed=0)),   # config-2 shape
    (100, 0.1, C1),                                                          # config 1
])
def test_torchrun_two_ranks_gloo(engine, tmp_path, n, p, cfg, mode):
    from paper_2603_26232_b200 import generate_er
    out = tmp_path / "rank0.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000),
           os.path.join(ROOT, "tests", "gpu_sharded_run.py"), str(out), str(n), str(p),
           json.dumps(cfg), mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    got = json.loads(out.read_text())
    single = engine.run_pipeline(n, generate_er(n, p, 0), **cfg)
    assert got["cut"] == single.cut and got["assignment"] == single.assignment
    assert got["leaves"] == single.candidates_evaluated and got["evals"] == single.evals


def test_sharded_session_single_process(engine):
    """qc_pipeline_prepare with shard_count = 3 on one engine per shard: each session holds
    only its block's cut tables; concatenated records merged by one session equal the
    single-GPU pipeline (cut, assignment, leaves, evals), twice in a row."""
    from paper_2603_26232_b200 import generate_er
    e = generate_er(400, 0.1, 0)
    cfg = dict(qubit_cap=20, top_k=2, layers=2, budget=8, seed=0)
    single = engine.run_pipeline(400, e, **cfg)
    sessions = [engine.prepare_pipeline(400, e, shard_index=r, shard_count=3, **cfg) for r in range(3)]
    try:
        rb, M = sessions[0].geometry()
        assert M == 21
        for _ in range(2):
            recs = np.concatenate([s.execute_shard() for s in sessions])
            assert recs.size == rb * M
            _same(sessions[1].merge_records(recs), single)
    finally:
        for s in sessions:
            s.close()
