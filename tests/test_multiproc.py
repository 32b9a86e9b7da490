"""World-size-2 CPU coverage of the N>1 path (gloo): query shards per rank,
no data-path collective, results gathered only for checking, timing reduced
as the max over ranks -- the same host logic bench.py runs under torchrun
with NCCL on B200s.  The per-rank search here is the CPU oracle (no GPU in
this container); the GPU engine's sharded equivalence is covered by
tests/test_gpu_parity.py::test_multi_device_fleet_invariance."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1512_02831_b200.dist import max_over_ranks, shard_range


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from oracle import oracle as O
    rng = np.random.default_rng(5)
    refs = rng.random((3000, 6), dtype=np.float32)
    queries = rng.random((1001, 6), dtype=np.float32)
    tree = O.build_tree(refs, 5)
    lo, hi = shard_range(queries.shape[0], rank, world)
    keys = O.knn_tree(tree, queries[lo:hi], 7)["keys"]
    t = max_over_ranks(float(rank + 1))
    # gather shards (checking only; the search itself exchanged nothing)
    sizes = [None] * world
    dist.all_gather_object(sizes, (lo, hi, keys.view(np.int64).tolist()))
    if rank == 0:
        full = np.zeros((queries.shape[0], 7), np.uint64)
        for lo_, hi_, k_ in sizes:
            full[lo_:hi_] = np.asarray(k_, np.int64).view(np.uint64).reshape(hi_ - lo_, 7)
        want = O.brute_keys(refs, queries, 7)
        out.put((bool(np.array_equal(full, want)), t))
    dist.destroy_process_group()


def test_shard_range_partitions():
    for m in (0, 1, 7, 1001):
        for w in (1, 2, 3, 8):
            rs = [shard_range(m, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == m
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
    with pytest.raises(ValueError):
        shard_range(5, 2, 2)


def test_two_rank_gloo_sharded_search():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    ok, tmax = q.get(timeout=5)
    assert ok
    assert tmax == 2.0
