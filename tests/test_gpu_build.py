"""Device-side tree build (bkt_build_tree_device) against the reference's
golden builds and the host build: identical split values, leaf bounds and
leaf point sets (the order inside a leaf is not part of the contract,
reference buffer_tree.py:149-197 / kdtree.py:55-70)."""
import numpy as np
import pytest

import paper_1512_02831_b200 as bkt
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def leaf_sets(tree):
    st = np.asarray(tree.leaves.leaf_starts)
    oi = np.asarray(tree.leaves.original_index)
    return [np.sort(oi[st[i]:st[i + 1]]) for i in range(len(st) - 1)]


def assert_same_build(a, b):
    assert np.array_equal(a.top.split_values, b.top.split_values)
    assert np.array_equal(a.leaves.leaf_starts, b.leaves.leaf_starts)
    for x, y in zip(leaf_sets(a), leaf_sets(b)):
        assert np.array_equal(x, y)


def test_gpu_build_matches_reference_golden():
    g = np.load(GOLDEN / "build_kat.npz")
    for name in g["names"]:
        name = str(name)
        tree = bkt.build_buffer_tree(g[name + "/refs"], int(g[name + "/h"]), device=0)
        members = np.concatenate(leaf_sets(tree))
        assert np.array_equal(tree.top.split_values, g[name + "/split_values"]), name
        assert np.array_equal(tree.leaves.leaf_starts, g[name + "/leaf_starts"]), name
        assert np.array_equal(members, g[name + "/members"]), name


def test_eight_point_line():
    tree = bkt.build_buffer_tree(np.float32([[7], [3], [5], [1], [8], [2], [6], [4]]), 2, device=0)
    assert tree.top.split_values.tolist() == [5.0, 3.0, 7.0]
    assert tree.leaves.leaf_starts.tolist() == [0, 2, 4, 6, 8]


@pytest.mark.parametrize("n,d,h", [(1000, 3, 5), (65537, 10, 8), (250_001, 7, 11), (4096, 1, 12)])
def test_gpu_build_equals_host(n, d, h):
    rng = np.random.default_rng(n + d + h)
    refs = rng.random((n, d), dtype=np.float32)
    host = bkt.build_buffer_tree(refs, h)
    dev = bkt.build_buffer_tree(refs, h, device=0)
    assert_same_build(host, dev)
    # the gathered leaf-sorted points are the rows of original_index
    assert np.array_equal(np.asarray(dev.leaves.points), refs[np.asarray(dev.leaves.original_index)])
    bkt.validate_structure(dev, refs)


def test_gpu_build_ties_signed_zero_and_negatives():
    rng = np.random.default_rng(5)
    refs = rng.integers(-3, 4, size=(20_000, 4)).astype(np.float32)  # heavy ties
    refs[::7, 0] = -0.0
    refs[1::7, 0] = 0.0
    for h in (3, 9):
        assert_same_build(bkt.build_buffer_tree(refs, h), bkt.build_buffer_tree(refs, h, device=0))


def test_gpu_build_search_is_exact():
    rng = np.random.default_rng(9)
    refs = rng.random((30_000, 10), dtype=np.float32)
    q = rng.random((3_000, 10), dtype=np.float32)
    a = bkt.lazy_search(bkt.build_buffer_tree(refs, 7), q, bkt.SearchParams(k=10))
    b = bkt.lazy_search(bkt.build_buffer_tree(refs, 7, device=0), q, bkt.SearchParams(k=10))
    assert np.array_equal(a.keys, b.keys)


def test_gpu_build_validation():
    with pytest.raises(ValueError):
        bkt.build_buffer_tree(np.zeros((3, 2), np.float32), 2, device=0)
