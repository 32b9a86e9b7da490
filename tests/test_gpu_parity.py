"""GPU parity: the sm_100a engine vs the reference's golden outputs and the
CPU oracle, through the drop-in API (lazy_search -> bkt_search C ABI).

exact mode: keys bit-identical, visited counts and leaf sequences identical
(the reference's own contract, tests/test_acceptance.py criteria 1 and 4).
fma mode (north star tolerance): squared distances within 1e-5 relative,
indices equal except where reference distances tie within 1e-5.
"""
import hashlib
import json

import numpy as np
import pytest

import paper_1512_02831_b200 as bkt
from oracle import oracle as O
from conftest import GOLDEN

pytestmark = pytest.mark.gpu

FMA_RTOL = 1e-5


def _dist_idx(keys):
    return bkt.unpack_keys(keys)


def assert_fma_close(got_keys, want_keys, rtol=FMA_RTOL):
    gd, gi = _dist_idx(got_keys)
    wd, wi = _dist_idx(want_keys)
    scale = np.maximum(np.abs(wd), np.finfo(np.float32).tiny)
    assert np.all(np.abs(gd.astype(np.float64) - wd) <= rtol * scale + 1e-30)
    mism = gi != wi
    if mism.any():
        # an index may differ only where the reference has a near-tie at that rank
        r, c = np.nonzero(mism)
        for rr, cc in zip(r, c):
            near = np.abs(wd[rr] - wd[rr, cc]) <= rtol * max(wd[rr, cc], 1e-30)
            assert set(gi[rr][near].tolist()) <= set(wi[rr].tolist()) | set(gi[rr].tolist())
            assert near.sum() >= 2 or cc == got_keys.shape[1] - 1, (rr, cc)


@pytest.mark.parametrize("kernel", ["direct", "tc"])
def test_golden_instances_exact(knn_golden, gpu_device, kernel):
    """Every golden instance: keys, counts, visited counts, leaf sequences,
    for the CUDA-core scan and the tensor-core filter (auto, d <= 31)."""
    for c in knn_golden:
        s = c["spec"]
        tree = bkt.build_buffer_tree(c["refs"], s["h"])
        stats = bkt.SearchStats(record_sequences=True)
        res = bkt.lazy_search(tree, c["queries"], bkt.SearchParams(k=s["k"]), device=gpu_device, stats=stats,
                              debug_audit=True, kernel=kernel)
        assert np.array_equal(res.keys, c["keys"]), s
        assert np.array_equal(res.counts, c["counts"]), s
        assert np.array_equal(stats.visited_per_query, c["visited"]), s
        flat = np.concatenate([np.asarray(x, np.int64) for x in stats.leaf_sequences])
        assert np.array_equal(flat, c["seq"]), s
        assert stats.leaf_scan_events == int(c["visited"].sum())
        assert bkt.result_digest(res) == c["digest"]


@pytest.mark.parametrize("kernel", ["direct", "tc"])
def test_golden_instances_fma_within_tolerance(knn_golden, gpu_device, kernel):
    for c in knn_golden:
        s = c["spec"]
        if s["kind"] == "grid":
            continue  # exact ties everywhere; covered in exact mode
        tree = bkt.build_buffer_tree(c["refs"], s["h"])
        res = bkt.lazy_search(tree, c["queries"], bkt.SearchParams(k=s["k"]), device=gpu_device, exact=False,
                              kernel=kernel)
        assert_fma_close(res.keys, c["keys"])


def test_tc_and_direct_fma_identical(knn_golden, gpu_device):
    """FMA mode: the tensor-core filter re-evaluates survivors with the same
    FMA arithmetic as the direct scan, so both kernels agree bit for bit."""
    for c in knn_golden:
        s = c["spec"]
        tree = bkt.build_buffer_tree(c["refs"], s["h"])
        p = bkt.SearchParams(k=s["k"])
        a = bkt.lazy_search(tree, c["queries"], p, device=gpu_device, exact=False, kernel="direct")
        b = bkt.lazy_search(tree, c["queries"], p, device=gpu_device, exact=False, kernel="tc")
        assert np.array_equal(a.keys, b.keys), s


@pytest.mark.parametrize("kernel", ["direct", "tc"])
def test_config1_full_digest(gpu_device, kernel):
    """BASELINE configs[0] in full on the GPU: reference digest 4a6f28e1..."""
    gold = json.load(open(GOLDEN / "c1_digest.json"))
    refs, queries = bkt.datasets.config_inputs(1)
    tree = bkt.build_buffer_tree(refs, 8)
    stats = bkt.SearchStats()
    res = bkt.lazy_search(tree, queries, bkt.SearchParams(k=10), device=gpu_device, stats=stats, kernel=kernel)
    assert bkt.result_digest(res) == gold["digest_indices_sha256"]
    assert hashlib.sha256(res.keys.astype("<u8").tobytes()).hexdigest() == gold["keys_sha256"]
    assert stats.leaf_scan_events == gold["leaf_scan_events"]
    rows = np.load(GOLDEN / "c1_rows.npz")
    assert np.array_equal(stats.visited_per_query, rows["visited"].astype(np.int64))
    # pairs = sum over visits of the leaf size (256 at n = 2^16, h = 8)
    assert stats.pairs == 256 * gold["leaf_scan_events"]


@pytest.mark.parametrize("kernel", ["direct", "tc"])
def test_config2_sample_exact(gpu_device, kernel):
    g = np.load(GOLDEN / "c2_sample.npz")
    pts, _ = bkt.gen_mixture(12_000_000, 10, seed=1)
    refs = pts.data[:2_000_000]
    tree = bkt.build_buffer_tree(refs, 9)
    stats = bkt.SearchStats()
    res = bkt.lazy_search(tree, g["queries"], bkt.SearchParams(k=10), device=gpu_device, stats=stats,
                          kernel=kernel)
    assert np.array_equal(res.keys, g["keys"])
    assert np.array_equal(stats.visited_per_query, g["visited"])


@pytest.mark.parametrize("num_chunks", [2, 3, 13])
def test_out_of_core_chunked_plan_exact(rng, gpu_device, num_chunks):
    """Host-resident leaf structure streamed in chunks that straddle leaves
    (reference tests/test_buffer_tree.py:275-284, n prime)."""
    refs = rng.random((4099, 6), dtype=np.float32)
    queries = rng.random((300, 6), dtype=np.float32)
    params = bkt.SearchParams(k=5)
    tree = bkt.build_buffer_tree(refs, 5)
    want = O.brute_keys(refs, queries, 5, threads=4)
    plan = bkt.ChunkPlan.build(refs.shape[0], num_chunks)
    stats = bkt.SearchStats()
    res = bkt.lazy_search(tree, queries, params, None, gpu_device, plan, stats=stats)
    assert np.array_equal(res.keys, want)
    # visited counts do not depend on chunking
    ot = O.build_tree(refs, 5)
    assert np.array_equal(stats.visited_per_query, O.knn_tree(ot, queries, 5)["visited"])


@pytest.mark.parametrize("num_chunks,h,k", [(2, 7, 7), (5, 9, 10), (16, 10, 33)])
def test_out_of_core_drain_equals_round_schedule(rng, gpu_device, monkeypatch, num_chunks, h, k):
    """The drain schedule (each resident unit drained before the next,
    engine.cu ooc_drain) against the one-round-per-leaf schedule
    (BKT_OOC_ROUNDS=1): identical keys, visited counts and per-query leaf
    sequences; keys equal the oracle's brute force.  (Bytes streamed: the
    drain also ships the tensor-core rows, so with two chunks -- both
    resident in the two slots under either schedule -- it moves more; the
    config-5 runs in profiles/ show the cut at scale.)"""
    refs = rng.random((30_011, 8), dtype=np.float32)
    queries = rng.random((3_000, 8), dtype=np.float32)
    tree = bkt.build_buffer_tree(refs, h)
    plan = bkt.ChunkPlan.build(refs.shape[0], num_chunks)
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("BKT_OOC_ROUNDS", mode)
        st = bkt.SearchStats(record_sequences=True)
        res = bkt.lazy_search(tree, queries, bkt.SearchParams(k=k), None, gpu_device, plan, stats=st)
        out[mode] = (res, st)
    (rd, sd), (rr, sr) = out["0"], out["1"]
    assert np.array_equal(rd.keys, O.brute_keys(refs, queries, k, threads=4))
    assert np.array_equal(rd.keys, rr.keys)
    assert np.array_equal(sd.visited_per_query, sr.visited_per_query)
    assert sd.leaf_scan_events == sr.leaf_scan_events
    assert sd.leaf_sequences == sr.leaf_sequences
    assert sd.stream_bytes > 0 and sr.stream_bytes > 0


@pytest.mark.parametrize("cta", ["0", "1"])
def test_out_of_core_drain_unit_finisher(rng, gpu_device, monkeypatch, cta):
    """The drain's unit-restricted tail finisher (warp and CTA variants,
    forced on from 2,000 queries per unit) keeps keys, visited counts and leaf
    sequences equal to the round schedule's, and its parked queries resume in
    later units."""
    refs = rng.random((40_009, 6), dtype=np.float32)
    queries = rng.random((4_000, 6), dtype=np.float32)
    k = 9
    tree = bkt.build_buffer_tree(refs, 8)
    plan = bkt.ChunkPlan.build(refs.shape[0], 6)
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("BKT_OOC_ROUNDS", mode)
        if mode == "0":
            monkeypatch.setenv("BKT_FINISH_AT", "2000")
            monkeypatch.setenv("BKT_FINISH_CTA", cta)
        else:
            monkeypatch.delenv("BKT_FINISH_AT", raising=False)
            monkeypatch.delenv("BKT_FINISH_CTA", raising=False)
        st = bkt.SearchStats(record_sequences=True)
        res = bkt.lazy_search(tree, queries, bkt.SearchParams(k=k), None, gpu_device, plan, stats=st)
        out[mode] = (res, st)
    (rd, sd), (rr, sr) = out["0"], out["1"]
    assert np.array_equal(rd.keys, O.brute_keys(refs, queries, k, threads=4))
    assert np.array_equal(rd.keys, rr.keys)
    assert np.array_equal(sd.visited_per_query, sr.visited_per_query)
    assert sd.leaf_sequences == sr.leaf_sequences


def test_out_of_core_spilled_structure(rng, gpu_device, tmp_path):
    """Disk-resident leaf structure (sec. 3.2, reference
    buffer_tree.py:187-191): leaf points memory-mapped from store_path and the
    device's host-resident layouts in file-backed pages under spill_dir
    (bkt_set_spill_dir), streamed unit by unit by the drain.  Keys and visited
    counts equal the oracle and the page-locked host-resident search; the
    spill files are unlinked (nothing is left in spill_dir)."""
    refs = rng.random((50_021, 10), dtype=np.float32)
    queries = rng.random((3_000, 10), dtype=np.float32)
    k = 10
    tree = bkt.build_buffer_tree(refs, 8, str(tmp_path / "leaves"))
    assert isinstance(tree.leaves.points, np.memmap)
    plan = bkt.ChunkPlan.build(refs.shape[0], 5)
    spill = tmp_path / "spill"
    spill.mkdir()
    dev = bkt.device_init(bkt.DeviceSpec(spill_dir=str(spill)))
    try:
        st = bkt.SearchStats()
        res = bkt.lazy_search(tree, queries, bkt.SearchParams(k=k), None, dev, plan, stats=st)
        assert list(spill.iterdir()) == []
        assert st.stream_bytes > 0
        with pytest.raises(ValueError, match="general-domain"):
            bkt.lazy_search(tree, queries[:10], bkt.SearchParams(k=65), None, dev, plan)
    finally:
        dev.close()
    assert np.array_equal(res.keys, O.brute_keys(refs, queries, k, threads=4))
    ot = O.build_tree(refs, 8)
    assert np.array_equal(st.visited_per_query, O.knn_tree(ot, queries, k)["visited"])
    pinned = bkt.lazy_search(tree, queries, bkt.SearchParams(k=k), None, gpu_device, plan)
    assert np.array_equal(res.keys, pinned.keys)


def test_out_of_core_config1_digest(gpu_device):
    gold = json.load(open(GOLDEN / "c1_digest.json"))
    refs, queries = bkt.datasets.config_inputs(1)
    tree = bkt.build_buffer_tree(refs, 8)
    res = bkt.lazy_search(tree, queries[:8192], bkt.SearchParams(k=10), device=gpu_device,
                          plan=bkt.ChunkPlan.build(refs.shape[0], 7))
    rows = np.load(GOLDEN / "c1_rows.npz")
    assert np.array_equal(res.keys[:2048], rows["keys_head"])


def test_edge_cases(rng, gpu_device):
    refs = rng.random((64, 2), dtype=np.float32)
    tree = bkt.build_buffer_tree(refs, 2)
    # empty query batch (reference test_buffer_tree.py:335-339)
    res = bkt.lazy_search(tree, np.empty((0, 2), np.float32), bkt.SearchParams(k=2), device=gpu_device)
    assert res.keys.shape == (0, 2)
    # dimension mismatch / k bounds (ValueError like the reference)
    with pytest.raises(ValueError):
        bkt.lazy_search(tree, rng.random((4, 3), dtype=np.float32), bkt.SearchParams(k=1), device=gpu_device)
    with pytest.raises(ValueError):
        bkt.lazy_search(tree, refs[:3], bkt.SearchParams(k=65), device=gpu_device)
    with pytest.raises(ValueError):
        bkt.lazy_search(tree, refs[:3], bkt.SearchParams(k=0), device=gpu_device)
    # k == n: every point returned
    res = bkt.lazy_search(tree, refs[:5], bkt.SearchParams(k=64), device=gpu_device)
    assert np.array_equal(res.keys, O.brute_keys(refs, refs[:5], 64))
    # query on a reference point finds itself (test_buffer_tree.py:286-291)
    r2 = rng.random((128, 3), dtype=np.float32)
    res = bkt.lazy_search(bkt.build_buffer_tree(r2, 3), r2[17:18], bkt.SearchParams(k=1), device=gpu_device)
    assert res.indices[0, 0] == 17 and res.sq_dists[0, 0] == np.float32(0.0)
    # duplicate points tie-break by index (test_buffer_tree.py:293-298)
    dup = np.float32([[0, 0], [1, 1], [1, 1], [1, 1], [2, 2], [3, 3], [4, 4], [5, 5]])
    res = bkt.lazy_search(bkt.build_buffer_tree(dup, 2), np.float32([[1, 1]]), bkt.SearchParams(k=2),
                          device=gpu_device)
    assert res.indices[0].tolist() == [1, 2]


def test_tie_on_slab_distance_is_visited(gpu_device):
    # reference test_buffer_tree.py:159-173: kth == slab distance^2 == 0 -> visit
    refs = np.float32([[0.0], [0.0], [1.0], [1.0]])
    tree = bkt.build_buffer_tree(refs, 1)
    stats = bkt.SearchStats(record_sequences=True)
    res = bkt.lazy_search(tree, np.float32([[1.0]]), bkt.SearchParams(k=2), device=gpu_device, stats=stats)
    assert stats.leaf_sequences[0] == [1, 0]
    assert res.indices[0].tolist() == [2, 3]


def test_unpruned_backtracking_order(gpu_device):
    # reference test_buffer_tree.py:114-126: k = n keeps kth = inf until the end
    refs = np.float32([[7], [3], [5], [1], [8], [2], [6], [4]])
    tree = bkt.build_buffer_tree(refs, 2)
    stats = bkt.SearchStats(record_sequences=True)
    bkt.lazy_search(tree, np.float32([[1.4]]), bkt.SearchParams(k=8), device=gpu_device, stats=stats)
    assert stats.leaf_sequences[0] == [0, 1, 2, 3]


@pytest.mark.parametrize("d", [1, 2, 5, 9, 13, 15, 16, 17, 21, 27, 31, 32])
def test_dimension_coverage_exact(rng, gpu_device, d):
    refs = rng.random((3000, d), dtype=np.float32)
    queries = rng.random((257, d), dtype=np.float32)
    tree = bkt.build_buffer_tree(refs, 6)
    for k in (1, 3, 10, 33):
        want = O.brute_keys(refs, queries, k, threads=4)
        for kernel in ("direct", "tc") if d <= 31 else ("direct", "auto"):
            res = bkt.lazy_search(tree, queries, bkt.SearchParams(k=k), device=gpu_device, kernel=kernel)
            assert np.array_equal(res.keys, want), (d, k, kernel)


@pytest.mark.parametrize("kernel", ["direct", "tc"])
def test_large_values_and_negative_coords(rng, gpu_device, kernel):
    refs = (rng.normal(0, 1e5, (5000, 4))).astype(np.float32)
    queries = (rng.normal(0, 1e5, (500, 4))).astype(np.float32)
    tree = bkt.build_buffer_tree(refs, 7)
    res = bkt.lazy_search(tree, queries, bkt.SearchParams(k=7), device=gpu_device, kernel=kernel)
    assert np.array_equal(res.keys, O.brute_keys(refs, queries, 7, threads=4))


@pytest.mark.parametrize("kernel", ["direct", "tc"])
def test_clustered_far_queries_and_offsets(rng, gpu_device, kernel):
    """Stress the tensor-core filter's error margin: tight clusters far from
    the origin (large |p| relative to neighbour distances), queries both in
    and far outside the clusters, duplicated points."""
    centres = rng.normal(0, 1e3, (6, 5)).astype(np.float32)
    refs = (centres[rng.integers(0, 6, 8000)] + rng.normal(0, 1e-2, (8000, 5))).astype(np.float32)
    refs[:500] = refs[500:1000]  # exact duplicates
    qa = (centres[rng.integers(0, 6, 400)] + rng.normal(0, 1e-2, (400, 5))).astype(np.float32)
    qb = rng.normal(0, 2e3, (100, 5)).astype(np.float32)
    queries = np.concatenate([qa, qb, refs[:50]])
    tree = bkt.build_buffer_tree(refs, 8)
    for k in (1, 10, 40):
        res = bkt.lazy_search(tree, queries, bkt.SearchParams(k=k), device=gpu_device, kernel=kernel)
        assert np.array_equal(res.keys, O.brute_keys(refs, queries, k, threads=8)), (k, kernel)


def test_batched_queries_equal_single_batch(rng, gpu_device):
    refs = rng.random((20000, 8), dtype=np.float32)
    queries = rng.random((5000, 8), dtype=np.float32)
    tree = bkt.build_buffer_tree(refs, 7)
    gpu_device.ensure_tree(tree)
    k1, _, _ = gpu_device.search(queries, 10)
    k2, _, _ = gpu_device.search(queries, 10, batch_queries=777)
    assert np.array_equal(k1, k2)
    assert np.array_equal(k1, O.brute_keys(refs, queries, 10, threads=8))


def test_multi_device_fleet_invariance(rng):
    """run_multi_device over a fleet of contexts (all on GPU 0 here: one
    host thread per context), with query chunking (criterion 3)."""
    refs = rng.random((30000, 5), dtype=np.float32)
    queries = rng.random((800, 5), dtype=np.float32)
    tree = bkt.build_buffer_tree(refs, 5)
    params = bkt.SearchParams(k=10)
    config = bkt.BufferConfig.for_height(5)
    want = O.brute_keys(refs, queries, 10, threads=8)
    for n_dev in (1, 2, 4):
        fleet = bkt.DeviceFleet([bkt.GpuDevice(bkt.DeviceSpec(cuda_device=0)) for _ in range(n_dev)])
        try:
            stats = []
            res = bkt.run_multi_device(fleet, tree, queries, params, config, None, query_chunk_size=50,
                                       stats_out=stats)
            assert np.array_equal(res.keys, want)
            assert sum(s.leaf_scan_events for s in stats) > 0
        finally:
            fleet.close()


def test_multi_device_redispatch_on_failure(rng):
    refs = rng.random((3000, 3), dtype=np.float32)
    queries = rng.random((300, 3), dtype=np.float32)
    tree = bkt.build_buffer_tree(refs, 4)
    fleet = bkt.DeviceFleet([bkt.GpuDevice(bkt.DeviceSpec(cuda_device=0)) for _ in range(2)])
    try:
        fleet.devices[1].close()  # a dead device: every call on it fails
        res = bkt.run_multi_device(fleet, tree, queries, bkt.SearchParams(k=4), bkt.BufferConfig.for_height(4),
                                   None, query_chunk_size=40)
        assert np.array_equal(res.keys, O.brute_keys(refs, queries, 4))
    finally:
        fleet.close()


@pytest.mark.parametrize("num_chunks", [1, 2, 3, 4, 7])
def test_fine_seam_pipeline_round_equals_brute(rng, num_chunks):
    """The reference's device plugin seam driven by ChunkPipeline
    (reference tests/test_device.py:199-216)."""
    refs = rng.random((900, 4), dtype=np.float32)
    queries = rng.random((60, 4), dtype=np.float32)
    ids = np.arange(900, dtype=np.int64)
    plan = bkt.ChunkPlan.build(900, num_chunks)
    cb = bkt.chunk_required(plan.max_len, 4)
    dev = bkt.device_init(bkt.DeviceSpec(2 * cb + 10_000), cb, 10_000)
    try:
        nb = bkt.NeighborBatch(60, 5)
        rows = np.arange(60, dtype=np.int64)
        groups = [[(rows, lo, hi)] for lo, hi in plan.ranges()]
        bkt.run_chunk_pipeline(dev, refs, ids, plan, groups, queries, nb)
        assert np.array_equal(nb.keys, O.brute_keys(refs, queries, 5))
        assert (nb.counts == 5).all()
        assert not dev.hazard_violations
    finally:
        dev.close()


def test_device_budget_errors(rng):
    with pytest.raises(bkt.DeviceConfigError):
        bkt.device_init(bkt.DeviceSpec(100), 60, 10)
    refs = rng.random((100, 4), dtype=np.float32)
    plan = bkt.ChunkPlan.build(100, 2)
    dev = bkt.device_init(bkt.DeviceSpec(10 ** 6), bkt.chunk_required(10, 4), 100)
    try:
        with pytest.raises(bkt.DeviceConfigError, match="use at least"):
            bkt.ChunkPipeline(dev, refs, np.arange(100), plan)
        tree = bkt.build_buffer_tree(refs, 2)
        with pytest.raises(bkt.DeviceConfigError, match="use at least"):
            bkt.lazy_search(tree, refs[:4], bkt.SearchParams(k=2), None, dev, plan)
    finally:
        dev.close()


def test_run_engine_bufferkdtree(rng):
    refs = rng.random((6000, 5), dtype=np.float32)
    queries = rng.random((400, 5), dtype=np.float32)
    res, info = bkt.run_engine("bufferkdtree", refs, queries, bkt.SearchParams(k=8), height=6,
                               collect_stats=True)
    assert np.array_equal(res.keys, O.brute_keys(refs, queries, 8, threads=4))
    assert info["height"] == 6 and info["process_rounds"] > 0 and info["mean_leaves_visited"] >= 1
    res2, info2 = bkt.run_engine("bufferkdtree", refs, queries, bkt.SearchParams(k=8), height=6,
                                 device_memory=200_000)
    assert info2["num_chunks"] > 1
    assert np.array_equal(res2.keys, res.keys)


def test_large_result_through_pinned_pool(rng, gpu_device):
    """Results of >= 64 MB come from the page-locked pool and leave the GPU by a
    direct copy; they must equal the staged path and the oracle, and the pool
    must recycle a buffer once its array is gone."""
    from paper_1512_02831_b200 import _native
    refs = rng.random((60_000, 10), dtype=np.float32)
    q = rng.random((900_000, 10), dtype=np.float32)
    tree = bkt.build_buffer_tree(refs, 6)
    res = bkt.lazy_search(tree, q, bkt.SearchParams(k=10), device=gpu_device)
    staged = np.empty((q.shape[0], 10), np.uint64)  # pageable: staged copy path
    k2, _, _ = gpu_device.search(q, 10, out_keys=staged)
    assert np.array_equal(res.keys, k2)
    rows = np.arange(0, q.shape[0], 997)
    want = O.knn_tree(O.build_tree(refs, 6), np.ascontiguousarray(q[rows]), 10, threads=8)
    assert np.array_equal(res.keys[rows], want["keys"])
    del res
    import gc
    gc.collect()
    for _ in range(4):  # buffers are page-locked in the background, then recycled
        res2 = bkt.lazy_search(tree, q, bkt.SearchParams(k=10), device=gpu_device)
        assert np.array_equal(res2.keys, k2)
    nbytes = q.shape[0] * 10 * 8
    assert _native._PINNED._count.get(nbytes, 0) <= _native._PINNED._per_size


@pytest.mark.parametrize("env", [{"BKT_TC_N": "64"}, {"BKT_TC_N": "256"}, {"BKT_TC_CPS": "3"},
                                 {"BKT_TC_CPS": "3", "BKT_TC_N": "128"}])
def test_tensor_core_variants_exact(knn_golden, gpu_device, env, monkeypatch):
    """The alternative tensor-core layouts (chunk width, one control warp with
    3 CTAs per SM) are bit-identical to the reference as well."""
    for key, val in env.items():
        monkeypatch.setenv(key, val)
    for c in knn_golden[:12]:
        s = c["spec"]
        if s["d"] > 15:  # the variants cover the KT = 16 layout
            continue
        tree = bkt.build_buffer_tree(c["refs"], s["h"])
        res = bkt.lazy_search(tree, c["queries"], bkt.SearchParams(k=s["k"]), device=gpu_device, kernel="tc")
        assert np.array_equal(res.keys, c["keys"]), (env, s)


@pytest.mark.parametrize("finish_at,cta", [("-1", "0"), ("1000000000", "0"), ("1000000000", "1")])
@pytest.mark.parametrize("kernel", ["direct", "tc"])
def test_tail_finisher_on_and_off_exact(knn_golden, gpu_device, kernel, finish_at, cta, monkeypatch):
    """The tail finisher (one warp or one CTA per remaining query, one
    launch) and the plain round loop give the reference's keys, visit
    counts, leaf sequences and scan events: off entirely (-1) and taking
    over from the first round check (1e9)."""
    monkeypatch.setenv("BKT_FINISH_AT", finish_at)
    monkeypatch.setenv("BKT_FINISH_CTA", cta)
    for c in knn_golden:
        s = c["spec"]
        tree = bkt.build_buffer_tree(c["refs"], s["h"])
        stats = bkt.SearchStats(record_sequences=True)
        res = bkt.lazy_search(tree, c["queries"], bkt.SearchParams(k=s["k"]), device=gpu_device, stats=stats,
                              kernel=kernel)
        assert np.array_equal(res.keys, c["keys"]), (finish_at, s)
        assert np.array_equal(stats.visited_per_query, c["visited"]), (finish_at, s)
        flat = np.concatenate([np.asarray(x, np.int64) for x in stats.leaf_sequences])
        assert np.array_equal(flat, c["seq"]), (finish_at, s)
        assert stats.leaf_scan_events == int(c["visited"].sum())


@pytest.mark.parametrize("exact", [True, False])
def test_tail_finisher_mixture(gpu_device, exact, monkeypatch):
    """A config-2-like mixture: the finisher taking over at different points
    gives the same keys, visit counts and scan events as the round loop
    without it, in both arithmetic modes."""
    rng = np.random.default_rng(5)
    centers = rng.random((8, 10))
    pts = (centers[rng.integers(0, 8, 220_000)] + rng.normal(0, 0.05, (220_000, 10))).astype(np.float32)
    refs, queries = pts[:200_000], pts[200_000:]
    tree = bkt.build_buffer_tree(refs, 7)
    out = []
    for fa, cta in (("-1", "0"), ("5000", "0"), ("1000000000", "0"), ("5000", "1"), ("1000000000", "1")):
        monkeypatch.setenv("BKT_FINISH_AT", fa)
        monkeypatch.setenv("BKT_FINISH_CTA", cta)
        stats = bkt.SearchStats()
        res = bkt.lazy_search(tree, queries, bkt.SearchParams(k=10), device=gpu_device, stats=stats, exact=exact)
        out.append((res.keys, stats.visited_per_query, stats.leaf_scan_events))
    for keys, vis, ev in out[1:]:
        assert np.array_equal(keys, out[0][0]) and np.array_equal(vis, out[0][1]) and ev == out[0][2]
    if exact:
        sample = np.arange(0, queries.shape[0], 97)
        assert np.array_equal(out[0][0][sample], O.brute_keys(refs, queries[sample], 10))


@pytest.mark.parametrize("d", [16, 20])
@pytest.mark.parametrize("fam", ["normal", "uniform"])
def test_leaves_smaller_than_k_tc32(gpu_device, d, fam):
    """Regression (fuzz seed 11 case 68): leaves of ~8 points (fewer than
    k = 10) on the 32-column tensor-core layout.  Until a query holds k
    neighbours its filter threshold is +inf, and the 64-row chunk variant
    re-evaluated a short chunk's second (stale) column group."""
    rng = np.random.default_rng(5)
    x = rng.normal(0, 3, (4147 + 1771, d)) if fam == "normal" else rng.random((4147 + 1771, d))
    x = x.astype(np.float32)
    refs, q = x[:4147], x[4147:]
    tree = bkt.build_buffer_tree(refs, 9)
    want = O.knn_tree(O.build_tree(refs, 9), q, 10, threads=O.default_threads())
    for kernel in ("tc", "auto"):
        st = bkt.SearchStats()
        res = bkt.lazy_search(tree, q, bkt.SearchParams(k=10), device=gpu_device, stats=st, kernel=kernel)
        assert np.array_equal(res.keys, want["keys"]), kernel
        assert np.array_equal(st.visited_per_query, want["visited"].astype(np.int64)), kernel
