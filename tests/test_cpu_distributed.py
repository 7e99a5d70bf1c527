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


def pack_record(rb, layers, width, bits, probs, params, expectation, evals):
    """The solve-record layout of include/qcgpu.h (what qc_shard_solve writes)."""
    body = rb - 24 - 16 * layers
    kcap = 0
    while 8 * ((kcap * 4 + 7) // 8) + 8 * kcap < body:
        kcap += 1
    r = np.zeros(rb, np.uint8)
    r[:16] = np.array([width, len(bits), evals, 1], np.int32).view(np.uint8)
    r[16:24] = np.array([expectation]).view(np.uint8)
    r[24:24 + 4 * len(bits)] = np.asarray(bits, np.uint32).view(np.uint8)
    po = 24 + 8 * ((kcap * 4 + 7) // 8)
    r[po:po + 8 * len(probs)] = np.asarray(probs, np.float64).view(np.uint8)
    ao = po + 8 * kcap
    r[ao:ao + 16 * layers] = np.asarray(params, np.float64).view(np.uint8)
    return r


def _record_of(i, width, kcap, layers):
    k = min(kcap, 1 + i % kcap)
    return dict(width=width, bits=[(i * 13 + j) % (1 << (width - 1)) * 2 for j in range(k)],
                probs=[1.0 / (i + j + 2) for j in range(k)],
                params=[i + 0.25 * l for l in range(2 * layers)], expectation=i + 0.5, evals=200 + i)


def _worker_real(rank, world, port, n, cfg, q):
    """qc_run_record_bytes + qc_shard_range of the real (n, cfg) run, records packed in the
    real layout, one gloo all-gather, unpacked by the product's unpack_records."""
    import torch.distributed as dist

    from paper_2603_26232_b200 import load_library, run_record_bytes, unpack_records
    from paper_2603_26232_b200.distributed import gather_records, shard_bounds

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        edges = np.zeros(0, dtype=[("u", "<u4"), ("v", "<u4"), ("w", "<f8")])  # geometry only
        rb, M = run_record_bytes(n, edges, **cfg)
        bounds = shard_bounds(load_library(), M, world)
        b, e = bounds[rank]
        L = cfg["layers"]
        widths = [cfg["qubit_cap"]] * M
        local = np.concatenate([pack_record(rb, L, **_record_of(i, widths[i], cfg["top_k"], L))
                                for i in range(b, e)]) if e > b else np.zeros(0, np.uint8)
        allrec = gather_records(local, bounds, rb, rank)
        recs = unpack_records(allrec, M, rb, L)
        ok = len(recs) == M
        for i, r in enumerate(recs):
            want = _record_of(i, widths[i], cfg["top_k"], L)
            ok &= (r.width == want["width"] and list(r.bits) == want["bits"] and
                   list(r.probs) == want["probs"] and list(r.params) == want["params"] and
                   r.expectation == want["expectation"] and r.evals == want["evals"])
        q.put((rank, bool(ok), M, rb, bounds))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,cap,top_k,layers,M_expected", [(10000, 20, 2, 1, 527),
                                                            (16000, 26, 2, 1, 640),
                                                            (10000, 20, 8, 2, 527)])
def test_real_record_geometry_gloo(n, cap, top_k, layers, M_expected):
    """BASELINE configs 4 and 5 (527 / 640 pieces): the real shard ranges and record
    geometry over two gloo ranks, every record back in subgraph order."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    cfg = dict(qubit_cap=cap, top_k=top_k, layers=layers, budget=200, seed=0)
    procs = [ctx.Process(target=_worker_real, args=(r, 2, port, n, cfg, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _, _, _ in res)
    M, rb = res[0][2], res[0][3]
    assert M == M_expected and rb == 24 + 8 * ((top_k * 4 + 7) // 8) + 8 * top_k + 16 * layers


def test_record_bytes_follow_partition_not_cap():
    """with pieces narrower than the cap and top_k = 0 the record must be sized
    for the widest piece's class count (n=30, cap 20 -> widths 16 and 15)."""
    from paper_2603_26232_b200 import load_library, run_record_bytes
    lib = load_library()
    import ctypes as C
    lib.qc_record_bytes.restype = C.c_int64
    e = np.zeros(0, dtype=[("u", "<u4"), ("v", "<u4"), ("w", "<f8")])
    rb, M = run_record_bytes(30, e, qubit_cap=20, top_k=0, layers=1)
    assert M == 2 and rb == lib.qc_record_bytes(1 << 15, 1)
    rb, M = run_record_bytes(30, e, qubit_cap=20, top_k=4, layers=3)
    assert rb == lib.qc_record_bytes(4, 3)


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
