"""Multi-GPU plumbing: subgraphs sharded across ranks, one gather of solve records.

The QAOA stage shards naturally (every subgraph solve is a pure function of its local
graph, options and seed + index, pipeline.hpp:239-263), so each rank solves a contiguous
block of subgraph indices on its own GPU with no data-path collective. The only exchange
is the gather of the fixed-size solve records (top-K candidates, params, expectation,
evals) to rank 0 for the merge — an all-gather over NCCL/NVLink (gloo on CPU in tests).
"""
from __future__ import annotations

import numpy as np


def shard_bounds(engine_or_lib, M: int, world: int):
    """[(begin, end)] per rank: contiguous balanced blocks (qc_shard_range)."""
    if hasattr(engine_or_lib, "shard_range"):
        return [engine_or_lib.shard_range(M, r, world) for r in range(world)]
    import ctypes as C
    out = []
    for r in range(world):
        b, e = C.c_int32(0), C.c_int32(0)
        rc = engine_or_lib.qc_shard_range(C.c_int(M), C.c_int(r), C.c_int(world), C.byref(b),
                                          C.byref(e))
        if rc != 0:
            raise ValueError("invalid shard request")
        out.append((b.value, e.value))
    return out


def gather_records(local: np.ndarray, bounds, record_bytes: int, rank: int, device=None):
    """All-gather every rank's records (uint8, count*record_bytes) with one collective.
    Returns the M records in subgraph order on every rank."""
    import torch
    import torch.distributed as dist
    world = len(bounds)
    maxcount = max(e - b for b, e in bounds)
    buf = torch.zeros(maxcount * record_bytes, dtype=torch.uint8, device=device)
    if local.size:
        buf[: local.size].copy_(torch.from_numpy(np.ascontiguousarray(local)).to(buf.device))
    out = torch.empty(world * maxcount * record_bytes, dtype=torch.uint8, device=device)
    dist.all_gather_into_tensor(out, buf)
    host = out.cpu().numpy().reshape(world, maxcount * record_bytes)
    return np.concatenate([host[r, : (e - b) * record_bytes] for r, (b, e) in enumerate(bounds)])


def solve_sharded(engine, n: int, edges, rank: int, world: int, device=None, **cfg):
    """One distributed solve: shard the QAOA stage, gather records, merge on rank 0.
    Returns the RunReport on rank 0, None elsewhere."""
    # record geometry from the same chain partition the C side packs with (widest piece,
    # not the qubit cap: the two differ whenever the pieces are narrower than the cap)
    rb, M = engine.run_record_bytes(n, edges, **cfg)
    bounds = shard_bounds(engine, M, world)
    begin, end = bounds[rank]
    rec = engine.shard_solve(n, edges, begin, end, rb, **cfg)
    allrec = gather_records(rec, bounds, rb, rank, device=device)
    if rank == 0:
        return engine.merge_records(n, edges, allrec, M, **cfg)
    return None


class ShardedSession:
    """Resident sharded solve (one process per GPU): the partition and this rank's device
    cut tables are built once (qc_pipeline_prepare with shard_count = world); each step()
    runs this rank's block of the QAOA stage, all-gathers the fixed-size records once and
    merges on rank 0 with the session's partition (qc_pipeline_merge_records) — no
    re-partition of the edge list per step. Returns the RunReport on rank 0, None elsewhere."""

    def __init__(self, engine, n: int, edges, rank: int, world: int, device=None, **cfg):
        self.rank, self.world, self.device = rank, world, device
        self.sess = engine.prepare_pipeline(n, edges, shard_index=rank, shard_count=world, **cfg)
        self.rb, self.M = self.sess.geometry()
        self.bounds = shard_bounds(engine, self.M, world)

    def step(self):
        rec = self.sess.execute_shard()
        allrec = gather_records(rec, self.bounds, self.rb, self.rank, device=self.device)
        if self.rank == 0:
            return self.sess.merge_records(allrec)
        return None

    def close(self):
        self.sess.close()
