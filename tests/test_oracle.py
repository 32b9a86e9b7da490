"""Pin the CPU oracle against the reference's own outputs (tests/golden/).

The golden fixtures were produced by tests/golden/make_golden.py, which runs
the reference package (bufferknn) in the build container.  These tests run
on CPU anywhere.
"""
import hashlib
import json

import numpy as np
import pytest

from oracle import oracle as O
from conftest import GOLDEN


def _seqs_flat(seq, visited):
    return np.concatenate([seq[i, : visited[i]] for i in range(len(visited))]).astype(np.int64)


def test_oracle_knn_matches_reference_golden(knn_golden):
    for c in knn_golden:
        s = c["spec"]
        tree = O.build_tree(c["refs"], s["h"])
        r = O.knn_tree(tree, c["queries"], s["k"], threads=4, max_seq=1 << s["h"])
        assert np.array_equal(r["keys"], c["keys"]), s
        assert np.array_equal(r["visited"], c["visited"]), s
        assert np.array_equal(_seqs_flat(r["seq"], r["visited"]), c["seq"]), s


def test_oracle_brute_matches_reference_golden(knn_golden):
    for c in knn_golden[:12]:
        s = c["spec"]
        assert np.array_equal(O.brute_keys(c["refs"], c["queries"], s["k"], threads=4), c["keys"]), s


def test_numpy_restatement_agrees_with_c_oracle(knn_golden):
    for c in knn_golden[:6]:
        s = c["spec"]
        assert np.array_equal(O.np_brute_keys(c["refs"], c["queries"], s["k"]), c["keys"]), s


def test_scalar_distance_kats():
    # reference tests/test_core.py:33-41
    assert O.np_sq_dist(np.float32([0, 0]), np.float32([3, 4])) == np.float32(25.0)
    a = np.float32([1.5, -2.25, 7.0])
    assert O.np_sq_dist(a, a) == np.float32(0.0)
    assert O.np_sq_dist(np.float32([2.0]), np.float32([-1.0])) == np.float32(9.0)


def test_oracle_build_matches_reference_golden():
    b = np.load(GOLDEN / "build_kat.npz")
    for name in b["names"]:
        name = str(name)
        h = int(b[name + "/h"])
        tree = O.build_tree(b[name + "/refs"], h)
        st = tree.leaf_starts
        members = np.concatenate([np.sort(tree.original_index[st[i]:st[i + 1]]) for i in range(len(st) - 1)])
        assert np.array_equal(tree.split_values, b[name + "/split_values"]), name
        assert np.array_equal(st, b[name + "/leaf_starts"]), name
        assert np.array_equal(members, b[name + "/members"]), name
        sv, starts, sets = O.py_build(b[name + "/refs"], h)
        assert np.array_equal(sv, b[name + "/split_values"]), name
        assert np.array_equal(starts, b[name + "/leaf_starts"]), name


def test_eight_point_line_kat():
    # reference tests/test_buffer_tree.py:52-61
    tree = O.build_tree(np.float32([[7], [3], [5], [1], [8], [2], [6], [4]]), 2)
    assert tree.split_values.tolist() == [5.0, 3.0, 7.0]
    assert tree.leaf_starts.tolist() == [0, 2, 4, 6, 8]


def test_oracle_config1_digest():
    """BASELINE configs[0] in full: the reference digest 4a6f28e1...."""
    gold = json.load(open(GOLDEN / "c1_digest.json"))
    rng = np.random.default_rng(0)
    refs = rng.random((65536, 10), dtype=np.float32)
    queries = rng.random((65536, 10), dtype=np.float32)
    tree = O.build_tree(refs, 8)
    r = O.knn_tree(tree, queries, 10, threads=O.default_threads())
    idx = (r["keys"] & np.uint64(0xFFFFFFFF)).astype("<i8")
    assert hashlib.sha256(idx.tobytes()).hexdigest() == gold["digest_indices_sha256"]
    assert hashlib.sha256(r["keys"].astype("<u8").tobytes()).hexdigest() == gold["keys_sha256"]
    assert int(r["visited"].sum()) == gold["leaf_scan_events"]


def test_oracle_config2_sample():
    """Config-2 shape sample (mixture n=2M, h=9): first 256 queries."""
    from paper_1512_02831_b200.datasets import gen_mixture
    g = np.load(GOLDEN / "c2_sample.npz")
    # labels are drawn for all n + m rows before the normals, so the joint
    # 12M draw is regenerated exactly as the fixture did
    pts, _ = gen_mixture(12_000_000, 10, components=8, spread=0.05, seed=1)
    refs = pts.data[:2_000_000]
    assert hashlib.sha256(refs.tobytes()).hexdigest() == str(g["refs_sha256"])
    q = pts.data[2_000_000:2_000_256]
    assert np.array_equal(q, g["queries"])
    tree = O.build_tree(refs, 9)
    assert np.array_equal(tree.split_values, g["split_values"])
    r = O.knn_tree(tree, q, 10, threads=O.default_threads())
    assert np.array_equal(r["keys"], g["keys"])
    assert np.array_equal(r["visited"], g["visited"])
