"""CPU multi-process (gloo, world_size 2): the sharding + record gather plumbing of the
multi-GPU path (paper_2603_26232_b200/distributed.py). Each rank packs synthetic
fixed-size records for its contiguous shard; after the single all-gather every rank
must hold all M records in subgraph order."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, M, rb, q):
    import torch.distributed as dist

    from paper_2603_26232_b200 import load_library
    from paper_2603_26232_b200.distributed import gather_records, shard_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bounds = shard_bounds(load_library(), M, world)
        b, e = bounds[rank]
        # record i = bytes (i * 7 + k) % 251 — identifies its subgraph index
        local = np.concatenate([((np.arange(rb) + i * 7) % 251).astype(np.uint8)
                                for i in range(b, e)]) if e > b else np.zeros(0, np.uint8)
        allrec = gather_records(local, bounds, rb, rank)
        want = np.concatenate([((np.arange(rb) + i * 7) % 251).astype(np.uint8) for i in range(M)])
        q.put((rank, bool(np.array_equal(allrec, want)), bounds))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("M,world", [(21, 2), (5, 2), (1, 2)])
def test_gather_records_gloo(M, world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, 104, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res)
    bounds = res[0][2]
    assert bounds[0][0] == 0 and bounds[-1][1] == M
    assert all(bounds[i][1] == bounds[i + 1][0] for i in range(world - 1))


def test_shim_header_compiles():
    """include/qcut_gpu.hpp (the qcut::-style C++ drop-in) compiles and links against
    libqcgpu.so; running it needs a GPU (tests/test_gpu_cpp.py)."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = os.path.join(root, "build", "shim_config1")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    r = subprocess.run(["g++", "-std=c++20", "-O2", f"-I{root}/include",
                        f"{root}/tests/cpp/shim_config1.cpp", f"-L{root}/paper_2603_26232_b200",
                        "-lqcgpu", f"-Wl,-rpath,{root}/paper_2603_26232_b200", "-o", out],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
