"""Launched by tests/test_gpu_multi.py under torchrun (world size 2 on ONE B200, gloo):
every rank solves its contiguous shard of the subgraphs on cuda:0 through the C-ABI, the
records are all-gathered (gloo through host memory: NCCL refuses two ranks on one device),
rank 0 merges and writes the RunReport as JSON. mode "oneshot": qc_shard_solve +
qc_merge_records per call; mode "session": the bench's N>1 step (ShardedSession:
qc_pipeline_prepare with shard_count = world once, then qc_pipeline_execute_shard +
qc_pipeline_merge_records), run twice to check it repeats."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch.distributed as dist

    from paper_2603_26232_b200 import Engine, generate_er
    from paper_2603_26232_b200.distributed import ShardedSession, solve_sharded

    out, n, p, cfg = sys.argv[1], int(sys.argv[2]), float(sys.argv[3]), json.loads(sys.argv[4])
    mode = sys.argv[5] if len(sys.argv) > 5 else "oneshot"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    eng = Engine(0)
    if mode == "session":
        sess = ShardedSession(eng, n, generate_er(n, p, 0), rank, world, **cfg)
        first = sess.step()
        rep = sess.step()
        if rank == 0:
            assert (first.cut, first.assignment) == (rep.cut, rep.assignment)
        sess.close()
    else:
        rep = solve_sharded(eng, n, generate_er(n, p, 0), rank, world, **cfg)
    if rank == 0:
        with open(out, "w") as f:
            json.dump(dict(cut=rep.cut, assignment=rep.assignment, leaves=rep.candidates_evaluated,
                           evals=rep.evals, subgraphs=rep.subgraphs), f)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
