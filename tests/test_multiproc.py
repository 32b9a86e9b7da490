"""World-size-2 CPU coverage of the N>1 path (gloo): bench.py's query shards per rank,
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
    """One rank of bench.py's multi-rank flow at a small size: the rank's
    workload (bench.rank_work / bench.workload), a per-rank search (the CPU
    oracle stands in for the B200 engine here), the per-rank parity check
    (bench.check_rows) and the only cross-rank traffic (bench.reduce_ranks,
    bench.job_value)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from oracle import oracle as O
    n, m = 4000, 1001
    res = {}
    for scaling in ("strong", "weak"):
        w = bench.rank_work(scaling, rank, world, n, m)
        refs, queries = bench.workload(w, n, m)
        otree = O.build_tree(refs, 5)
        keys = O.knn_tree(otree, queries, bench.K)["keys"]
        ok = bench.check_rows(otree, queries, keys.view(np.int64), 50, 1, True)
        red = bench.reduce_ranks(float(rank + 1), 0.5 * (rank + 1), ok)
        value = bench.job_value(w["total"], 3, [red["dev_ms_max"] / 1e3])
        parts = [None] * world
        dist.all_gather_object(parts, (w, queries.tolist(), keys.view(np.int64).tolist()))
        res[scaling] = (red, value, parts, refs)
    if rank == 0:
        out.put(res)
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


def test_two_rank_gloo_bench_flow():
    """bench.py's rank logic on two gloo ranks: strong scaling shards the
    config-2 queries exactly (the shards concatenate to the single-rank
    queries and their results to the single-rank results), weak scaling gives
    rank 1 config 3's chunk 1, timings reduce to the slowest rank and parity
    to the AND over ranks."""
    import bench
    from oracle import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    n, m = 4000, 1001
    refs_all, q_all = bench.mixture_rows(n, m, 0, m)
    want = O.knn_tree(O.build_tree(refs_all, 5), q_all, bench.K)["keys"]
    # strong: shards partition the queries; whole job = m queries per step
    red, value, parts, refs = res["strong"]
    assert np.array_equal(refs, refs_all)
    assert [p_[0]["lo"] for p_ in parts] == [0, 501] and parts[-1][0]["hi"] == m
    assert np.array_equal(np.concatenate([np.asarray(p_[1], np.float32) for p_ in parts]), q_all)
    got = np.concatenate([np.asarray(p_[2], np.int64).view(np.uint64) for p_ in parts])
    assert np.array_equal(got, want)
    assert red == {"dev_ms_max": 2.0, "e2e_s_max": 1.0, "parity_all": True}
    assert value == 3 * m / 2e-3
    # weak: rank 0 the config-2 queries, rank 1 config 3's chunk 1; total = 2m per step
    red, value, parts, _ = res["weak"]
    assert parts[0][0]["kind"] == "cfg2" and parts[1][0] == {"kind": "chunk", "chunk": 1, "size": m, "total": 2 * m}
    assert np.array_equal(np.asarray(parts[0][1], np.float32), q_all)
    assert np.array_equal(np.asarray(parts[1][1], np.float32), bench.query_chunk(1, m))
    assert value == 3 * 2 * m / 2e-3
