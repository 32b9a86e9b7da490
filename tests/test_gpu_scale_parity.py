"""GPU parity at the BASELINE configurations' scale (the driver's -m gpu suite).

The golden/ fixtures pin small instances; these tests run the engine on
BASELINE-shaped inputs -- deep trees (h = 11, 14) over n >= 1M points, HBM-
and host-resident (4 chunks), k = 1 / 10 / 50 (config 5 shape); d = 15 / 27
at n = 2M (config 4); a config-3 stream chunk; uniform data at h = 11 -- and
compare >= 2,000 sampled rows' keys and visited-leaf counts bit-exactly
against the C oracle (oracle/bkt_oracle.c, the reference traversal of
buffer_tree.py:523-646 restated; pinned to the reference's goldens in
tests/test_oracle.py).  Each search runs a full batch (tens of thousands of
queries: many tiles per leaf, the tail finisher, the out-of-core chunk
rounds), and only the sampled rows are checked: rows are independent, so a
sample of a batch is checked against the oracle on exactly those queries.
"""
import numpy as np
import pytest

import paper_1512_02831_b200 as bkt
from oracle import oracle as O

pytestmark = pytest.mark.gpu

SAMPLE = 2000
_cache = {}


def _mixture(n, m, d):
    key = ("mix", n, m, d)
    if key not in _cache:
        pts, _ = bkt.gen_mixture(n + m, d, seed=1)
        _cache[key] = (np.ascontiguousarray(pts.data[:n]), np.ascontiguousarray(pts.data[n:]))
    return _cache[key]


def _tree(refs, h):
    key = ("tree", id(refs), h)
    if key not in _cache:
        _cache[key] = (bkt.build_buffer_tree(refs, h), O.build_tree(refs, h))
    return _cache[key]


def _check_sample(refs, queries, h, k, device, plan=None, kernel="auto", seed=0):
    tree, otree = _tree(refs, h)
    stats = bkt.SearchStats()
    res = bkt.lazy_search(tree, queries, bkt.SearchParams(k=k), None, device, plan, stats=stats, kernel=kernel)
    m = queries.shape[0]
    rows = np.sort(np.random.default_rng(seed).choice(m, size=min(SAMPLE, m), replace=False))
    want = O.knn_tree(otree, queries[rows], k, threads=O.default_threads())
    assert np.array_equal(res.keys[rows], want["keys"]), (h, k, kernel, plan)
    assert np.array_equal(stats.visited_per_query[rows], want["visited"].astype(np.int64)), (h, k, kernel)
    # every row finished with k real neighbours
    assert not np.any((res.keys & np.uint64(0xFFFFFFFF)) == np.uint64(0xFFFFFFFF))
    return res, stats


@pytest.mark.parametrize("h", [11, 14])
@pytest.mark.parametrize("k", [1, 10, 50])
@pytest.mark.parametrize("resident", ["hbm", "host4"])
def test_cfg5_shape_deep_trees(gpu_device, h, k, resident):
    """Config 5 shape at n = 1M: h = 11 (leaf 488) and h = 14 (leaf 61),
    HBM-resident (tensor-core filter) and host-resident in 4 chunks."""
    refs, queries = _mixture(1_000_000, 40_000, 10)
    plan = bkt.ChunkPlan.build(refs.shape[0], 4) if resident == "host4" else None
    _check_sample(refs, queries, h, k, gpu_device, plan=plan, seed=h * 100 + k)


@pytest.mark.parametrize("d", [15, 27])
def test_cfg4_shape_dims(gpu_device, d):
    """Config 4 shape: n = 2M mixture at d = 15 and 27, h = 9."""
    refs, queries = _mixture(2_000_000, 60_000, d)
    _check_sample(refs, queries, 9, 10, gpu_device, seed=d)


def test_cfg3_stream_chunk(gpu_device):
    """One config-3 query chunk (default_rng(1000 + c) recipe) against the
    config-2 references."""
    refs, _ = _mixture(2_000_000, 10_000_000, 10)
    q = bkt.datasets.gen_query_chunk(3, 1_000_000)
    _check_sample(refs, q, 9, 10, gpu_device, seed=3)


def test_uniform_headline_size_h11(gpu_device):
    """Uniform data at the headline size, deep tree: n = 2M, h = 11."""
    rng = np.random.default_rng(11)
    refs = rng.random((2_000_000, 10), dtype=np.float32)
    queries = rng.random((100_000, 10), dtype=np.float32)
    _check_sample(refs, queries, 11, 10, gpu_device, seed=11)


@pytest.mark.parametrize("kernel", ["direct", "tc"])
def test_cfg2_shape_both_kernels(gpu_device, kernel):
    """Config 2 shape (n = 2M, h = 9, k = 10) on a 200K-query batch, both scans."""
    refs, queries = _mixture(2_000_000, 10_000_000, 10)
    _check_sample(refs, queries[:200_000], 9, 10, gpu_device, kernel=kernel, seed=2)
