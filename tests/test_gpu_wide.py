"""GPU parity of the general-domain path (csrc/wide_search.cuh).

The reference accepts any k <= n (core.py:92-102), any height with 2^h <= n
(buffer_tree.py:159-163) and any d.  The round engine covers k <= 64, h <= 16
and d <= 32; everything else runs on the wide path (one CTA per query, the
whole traversal in one launch).  These tests hold it to the same bar as the
round engine: keys, visited counts, pairs and (where recorded) the leaf
sequences bit-identical to the C oracle (oracle/bkt_oracle.c), including the
reference's acceptance-style instances with k = 100 and d = 64.
"""
import numpy as np
import pytest

import paper_1512_02831_b200 as bkt
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _check(refs, queries, h, k, device, plan=None, exact=True, sequences=False):
    tree = bkt.build_buffer_tree(refs, h)
    otree = O.build_tree(refs, h)
    stats = bkt.SearchStats(record_sequences=sequences) if sequences else bkt.SearchStats()
    res = bkt.lazy_search(tree, queries, bkt.SearchParams(k=k), None, device, plan, stats=stats, exact=exact)
    maxv = int(tree.n_leaves) if sequences else 0
    want = O.knn_tree(otree, queries, k, threads=O.default_threads(), max_seq=maxv)
    if exact:
        assert np.array_equal(res.keys, want["keys"])
    else:
        gd, gi = bkt.unpack_keys(res.keys)
        wd, wi = bkt.unpack_keys(want["keys"])
        assert np.all(np.abs(gd.astype(np.float64) - wd) <= 1e-5 * np.maximum(wd, 1e-30))
    assert np.array_equal(stats.visited_per_query, want["visited"].astype(np.int64))
    assert stats.pairs == want["pairs"]
    assert stats.leaf_scan_events == int(want["visited"].sum())
    if sequences:
        for i in range(queries.shape[0]):
            v = int(want["visited"][i])
            assert list(stats.leaf_sequences[i]) == list(want["seq"][i, :v])
    return res, stats


def test_k100_d64_acceptance_shape(gpu_device):
    """k = 100, d = 64 (an acceptance-style instance outside the round engine)."""
    rng = np.random.default_rng(64)
    refs = rng.random((20_000, 64), dtype=np.float32)
    queries = rng.random((1_000, 64), dtype=np.float32)
    _check(refs, queries, 6, 100, gpu_device, sequences=True)


@pytest.mark.parametrize("k", [65, 100, 257])
def test_large_k_round_engine_tree(gpu_device, k):
    """k > 64 on a d = 10 tree that also has the tensor-core layout."""
    pts, _ = bkt.gen_mixture(60_000, 10, seed=5)
    refs, queries = np.ascontiguousarray(pts.data[:50_000]), np.ascontiguousarray(pts.data[50_000:])
    _check(refs, queries, 7, k, gpu_device)


def test_large_k_host_resident(gpu_device):
    """k = 100 on a host-resident (chunked) leaf structure: the wide kernel
    reads the mapped pinned copy in place."""
    rng = np.random.default_rng(3)
    refs = rng.random((30_000, 8), dtype=np.float32)
    queries = rng.random((2_000, 8), dtype=np.float32)
    plan = bkt.ChunkPlan.build(refs.shape[0], 3)
    _check(refs, queries, 6, 100, gpu_device, plan=plan)


def test_height_above_16(gpu_device):
    """h = 18 (2^18 leaves of 2 points): path state beyond 16 bits."""
    rng = np.random.default_rng(18)
    refs = rng.random((1 << 19, 3), dtype=np.float32)
    queries = rng.random((3_000, 3), dtype=np.float32)
    _check(refs, queries, 18, 4, gpu_device)


@pytest.mark.parametrize("d", [33, 100])
def test_dims_above_32(gpu_device, d):
    rng = np.random.default_rng(d)
    refs = rng.random((8_000, d), dtype=np.float32)
    queries = rng.random((500, d), dtype=np.float32)
    _check(refs, queries, 5, 10, gpu_device)


def test_k_equals_n(gpu_device):
    """k = n: every point is a neighbour (the row sorts the whole set)."""
    rng = np.random.default_rng(9)
    refs = rng.random((300, 5), dtype=np.float32)
    queries = rng.random((50, 5), dtype=np.float32)
    res, _ = _check(refs, queries, 3, 300, gpu_device)
    assert np.array_equal(np.sort(res.keys & np.uint64(0xFFFFFFFF), axis=1),
                          np.tile(np.arange(300, dtype=np.uint64), (50, 1)))


def test_huge_k_rows_in_global_memory(gpu_device):
    """k = 12,000: 2k keys per CTA exceed shared memory, rows live in HBM scratch."""
    rng = np.random.default_rng(12)
    refs = rng.random((40_000, 4), dtype=np.float32)
    queries = rng.random((64, 4), dtype=np.float32)
    _check(refs, queries, 4, 12_000, gpu_device)


def test_duplicates_and_ties_large_k(gpu_device):
    """Duplicated points (equal distances, ties broken by index) at k = 80."""
    rng = np.random.default_rng(4)
    base = rng.integers(0, 4, size=(2_000, 6)).astype(np.float32)
    refs = np.concatenate([base, base, base])
    queries = rng.integers(0, 4, size=(400, 6)).astype(np.float32)
    _check(refs, queries, 5, 80, gpu_device)


def test_fma_mode_large_k(gpu_device):
    rng = np.random.default_rng(6)
    refs = rng.random((20_000, 40), dtype=np.float32)
    queries = rng.random((300, 40), dtype=np.float32)
    _check(refs, queries, 5, 70, gpu_device, exact=False)
