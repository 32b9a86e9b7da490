"""Host-side logic of the drop-in (CPU only): native build vs the reference's
golden builds, the reference's index arithmetic KATs, result types, and the
C ABI surface of libbkt.so (loads and exports every symbol include/bkt.h
declares; no compute calls without a GPU)."""
import ctypes
import re

import numpy as np
import pytest
from hypothesis import given, strategies as st

import paper_1512_02831_b200 as bkt
from paper_1512_02831_b200 import _native
from conftest import GOLDEN, ROOT


def test_library_exports_every_header_symbol():
    header = (ROOT / "include" / "bkt.h").read_text()
    declared = set(re.findall(r"\b(bkt_[a-z0-9_]+)\s*\(", header))
    assert declared == set(_native.EXPORTS)
    lib = ctypes.CDLL(str(_native.LIB_PATH))
    for name in declared:
        assert hasattr(lib, name), name


def test_native_build_matches_reference_golden():
    b = np.load(GOLDEN / "build_kat.npz")
    for name in b["names"]:
        name = str(name)
        refs = b[name + "/refs"]
        tree = bkt.build_buffer_tree(refs, int(b[name + "/h"]))
        st = tree.leaves.leaf_starts
        members = np.concatenate([np.sort(tree.leaves.original_index[st[i]:st[i + 1]])
                                  for i in range(len(st) - 1)])
        assert np.array_equal(tree.top.split_values, b[name + "/split_values"]), name
        assert np.array_equal(tree.top.levels, b[name + "/levels"]), name
        assert np.array_equal(st, b[name + "/leaf_starts"]), name
        assert np.array_equal(members, b[name + "/members"]), name
        bkt.validate_structure(tree, refs)


def test_eight_point_line_by_hand():
    # reference tests/test_buffer_tree.py:52-61
    refs = np.float32([[7], [3], [5], [1], [8], [2], [6], [4]])
    tree = bkt.build_buffer_tree(refs, 2)
    assert tree.top.split_values.tolist() == [5.0, 3.0, 7.0]
    assert tree.top.levels.tolist() == [0, 1, 1]
    assert tree.leaves.leaf_starts.tolist() == [0, 2, 4, 6, 8]
    leaves = [sorted(np.asarray(tree.leaves.points)[slice(*tree.leaves.bounds(i)), 0]) for i in range(4)]
    assert leaves == [[1.0, 2.0], [3.0, 4.0], [5.0, 6.0], [7.0, 8.0]]
    bkt.validate_structure(tree, refs)


def test_native_build_large_matches_oracle(rng):
    from oracle import oracle as O
    refs = rng.random((200_003, 7), dtype=np.float32)
    tree = bkt.build_buffer_tree(refs, 11)
    ot = O.build_tree(refs, 11)
    assert np.array_equal(tree.top.split_values, ot.split_values)
    assert np.array_equal(tree.leaves.leaf_starts, ot.leaf_starts)
    st = tree.leaves.leaf_starts
    for i in range(0, 2048, 97):
        assert np.array_equal(np.sort(tree.leaves.original_index[st[i]:st[i + 1]]),
                              np.sort(ot.original_index[st[i]:st[i + 1]]))
    bkt.validate_structure(tree, refs)


def test_build_validation(rng):
    refs = rng.random((7, 2), dtype=np.float32)
    with pytest.raises(ValueError):
        bkt.build_buffer_tree(refs, 0)
    with pytest.raises(ValueError):
        bkt.build_buffer_tree(refs, 3)
    bkt.build_buffer_tree(refs, 2)
    bad = np.ones((4, 2), np.float32)
    bad[1, 1] = np.nan
    with pytest.raises(ValueError):
        bkt.build_buffer_tree(bad, 1)


def test_validate_catches_corruption(rng):
    refs = rng.random((64, 2), dtype=np.float32)
    tree = bkt.build_buffer_tree(refs, 3)
    tree.top.split_values[0] = np.float32(-1e9)
    with pytest.raises(ValueError):
        bkt.validate_structure(tree)


def test_store_path_memory_maps(rng, tmp_path):
    refs = rng.random((256, 3), dtype=np.float32)
    tree = bkt.build_buffer_tree(refs, 3, store_path=str(tmp_path / "leafpoints.npy"))
    assert isinstance(tree.leaves.points, np.memmap)
    bkt.validate_structure(tree, refs)


class TestBufferConfig:
    # reference tests/test_buffer_tree.py:25-48 and acceptance criterion 8
    def test_for_height_nine_defaults(self):
        cfg = bkt.BufferConfig.for_height(9)
        assert (cfg.buffer_capacity, cfg.fetch_count, cfg.half_full_threshold) == (32768, 327680, 16384)

    def test_overrides(self):
        cfg = bkt.BufferConfig.for_height(9, buffer_capacity=64, fetch_multiple=3, half_full_threshold=10)
        assert (cfg.buffer_capacity, cfg.fetch_count, cfg.half_full_threshold) == (64, 192, 10)

    def test_capacity_floor(self):
        assert bkt.BufferConfig.for_height(24).buffer_capacity == 1
        assert bkt.BufferConfig.for_height(30).half_full_threshold == 1

    def test_validation(self):
        for args in [(0, 1, 1), (4, 0, 2), (4, 1, 5)]:
            with pytest.raises(ValueError):
                bkt.BufferConfig(*args)


class TestChunkPlan:
    # reference tests/test_scheduler.py:22-119
    def test_ten_rows_three_chunks(self):
        plan = bkt.ChunkPlan.build(10, 3)
        assert plan.ranges() == [(0, 4), (4, 7), (7, 10)]
        assert plan.max_len == 4

    def test_overlapping(self):
        plan = bkt.ChunkPlan.build(10, 3)
        assert plan.overlapping(0, 10) == (0, 3)
        assert plan.overlapping(3, 5) == (0, 2)
        assert plan.overlapping(9, 10) == (2, 3)
        for lo, hi in [(3, 3), (5, 2), (-1, 4), (0, 11)]:
            with pytest.raises(ValueError):
                plan.overlapping(lo, hi)

    def test_build_validation(self):
        with pytest.raises(ValueError):
            bkt.ChunkPlan.build(0, 1)
        with pytest.raises(ValueError, match=r"\[1, 10\]"):
            bkt.ChunkPlan.build(10, 11)

    def test_assign_hand_example(self):
        plan = bkt.ChunkPlan.build(10, 3)
        assert bkt.assign_query_to_chunks(2, 9, plan) == [(0, 2, 4), (1, 4, 7), (2, 7, 9)]
        assert bkt.assign_query_to_chunks(6, 8, plan) == [(1, 6, 7), (2, 7, 8)]

    @given(st.data())
    def test_clips_partition_the_range(self, data):
        n = data.draw(st.integers(1, 500))
        num = data.draw(st.integers(1, n))
        lo = data.draw(st.integers(0, n - 1))
        hi = data.draw(st.integers(lo + 1, n))
        triples = bkt.assign_query_to_chunks(lo, hi, bkt.ChunkPlan.build(n, num))
        cursor = lo
        for _, clo, chi in triples:
            assert clo == cursor and clo < chi
            cursor = chi
        assert cursor == hi

    def test_plan_chunks_capacity(self):
        with pytest.raises(ValueError, match="use at least"):
            bkt.plan_chunks(1000, 2, 500, 20)
        assert bkt.plan_chunks(1000, 50, 500, 20).num_chunks == 50


def test_chunk_queries():
    assert bkt.chunk_queries(10, 4) == [(0, 4), (4, 7), (7, 10)]
    assert bkt.chunk_queries(0, 4) == []
    with pytest.raises(ValueError):
        bkt.chunk_queries(5, 0)


def test_packed_key_order_and_batch():
    d = np.float32([[2.0, 1.0, 1.0, 0.0]])
    i = np.uint64([[0, 9, 3, 5]])
    keys = np.sort(bkt.pack_keys(d, i), axis=1)
    _, idx = bkt.unpack_keys(keys)
    assert idx.tolist() == [[5, 3, 9, 0]]
    assert bkt.pack_keys(np.float32([[1e30]]), np.uint64([[bkt.INDEX_SENTINEL - 1]]))[0, 0] < bkt.EMPTY_KEY
    nb = bkt.NeighborBatch(2, 3)
    assert np.isinf(nb.kth_sq_dists()).all()
    assert (nb.indices == bkt.INDEX_SENTINEL).all()


def test_sizing_helpers():
    assert bkt.auto_height(65536) == 9 and bkt.auto_height(2) == 1 and bkt.auto_height(1 << 20) == 9
    assert bkt.query_block_bytes(10, 3, 2) == 10 * (12 + 16 + 32)
    qb = bkt.query_block_bytes(1000, 8, 10)
    num = bkt.auto_num_chunks(60_000, 8, qb, 1 << 20)
    assert 2 * bkt.chunk_required(-(-60_000 // num), 8) + qb <= 1 << 20
    assert num == 1 or 2 * bkt.chunk_required(-(-60_000 // (num - 1)), 8) + qb > 1 << 20


def test_result_digest_matches_golden(knn_golden):
    for c in knn_golden[:5]:
        nb = bkt.NeighborBatch.from_keys(c["keys"], c["counts"])
        assert bkt.result_digest(nb) == c["digest"]


def test_gen_mixture_matches_golden_queries():
    g = np.load(GOLDEN / "c2_sample.npz")
    q = bkt.gen_mixture(12_000_000, 10, seed=1)[0].data[2_000_000:2_000_256]
    assert np.array_equal(q, g["queries"])
