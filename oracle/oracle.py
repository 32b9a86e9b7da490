"""CPU oracle for the buffer k-d tree k-NN path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this module; it is the checker, never the
product.  It restates the reference package's (bufferknn, /root/reference/pkg)
arithmetic and traversal:

* ``bkt_oracle.c`` (compiled by ``oracle/Makefile`` into
  ``oracle/_build/libbkt_oracle.so``): tree build (median splits), classic
  per-query traversal with the reference pruning rule, brute force; float32
  with two roundings per dimension (-ffp-contract=off).
* pure numpy / Python restatements below for small cases, independent of the
  C code: ``np_sq_dist`` (core.py:108-122), ``np_brute_keys`` (brute.py:41-80
  via core.py:138-178), ``py_build`` (buffer_tree.py:149-197).

Pinned against the reference's own outputs: tests/golden/*.npz were produced
by tests/golden/make_golden.py importing /root/reference/pkg/src/bufferknn;
tests/test_oracle.py checks this module against them.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libbkt_oracle.so"
EMPTY_KEY = np.uint64((0x7F800000 << 32) | 0xFFFFFFFF)

_lib = None


def build() -> Path:
    """Compile the C oracle (gcc, seconds)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        P = ctypes.c_void_p
        L.or_build_tree.argtypes = [P, ctypes.c_int64, ctypes.c_int, ctypes.c_int, P, P, P]
        L.or_build_tree.restype = ctypes.c_int
        L.or_knn_tree.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, P, P, P, P, P, ctypes.c_int64,
                                  ctypes.c_int, P, P, P, ctypes.c_int, ctypes.c_int]
        L.or_knn_tree.restype = ctypes.c_int64
        L.or_brute.argtypes = [P, ctypes.c_int64, ctypes.c_int, P, ctypes.c_int64, ctypes.c_int, P, ctypes.c_int]
        L.or_brute.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleTree:
    """Output of the oracle build: the reference BufferKdTree's arrays."""

    def __init__(self, h, d, split_values, points, original_index, leaf_starts):
        self.h, self.d = h, d
        self.split_values = split_values
        self.points = points
        self.original_index = original_index
        self.leaf_starts = leaf_starts

    @property
    def n(self) -> int:
        return self.points.shape[0]


def build_tree(refs: np.ndarray, h: int) -> OracleTree:
    """buffer_tree.py:149-197 restated in C (or_build_tree)."""
    refs = np.ascontiguousarray(refs, dtype=np.float32)
    n, d = refs.shape
    split = np.empty((1 << h) - 1, np.float32)
    order = np.empty(n, np.int64)
    starts = np.empty((1 << h) + 1, np.int64)
    rc = lib().or_build_tree(_p(refs), n, d, h, _p(split), _p(order), _p(starts))
    if rc != 0:
        raise ValueError(f"oracle build failed ({rc})")
    return OracleTree(h, d, split, np.ascontiguousarray(refs[order]), order, starts)


def knn_tree(tree: OracleTree, queries: np.ndarray, k: int, threads: int = 1,
             max_seq: int = 0) -> dict:
    """Classic traversal k-NN (kdtree.py:157-204 order == lazy_search order).

    Returns keys (m, k) uint64 ascending, visited (m,) int32, pairs, and
    (if max_seq) seq (m, max_seq) int32 padded with -1."""
    q = np.ascontiguousarray(queries, dtype=np.float32)
    m = q.shape[0]
    keys = np.empty((m, k), np.uint64)
    visited = np.empty(m, np.int32)
    seq = np.empty((m, max_seq), np.int32) if max_seq else None
    pairs = lib().or_knn_tree(tree.h, tree.d, tree.n, _p(tree.split_values), _p(tree.points),
                              _p(tree.original_index), _p(tree.leaf_starts), _p(q), m, k,
                              _p(keys), _p(visited), _p(seq) if seq is not None else None,
                              max_seq, threads)
    if pairs < 0:
        raise ValueError("oracle search failed")
    return {"keys": keys, "visited": visited, "pairs": int(pairs), "seq": seq}


def brute_keys(refs: np.ndarray, queries: np.ndarray, k: int, threads: int = 1) -> np.ndarray:
    """brute.py:41-80 restated in C."""
    r = np.ascontiguousarray(refs, dtype=np.float32)
    q = np.ascontiguousarray(queries, dtype=np.float32)
    keys = np.empty((q.shape[0], k), np.uint64)
    lib().or_brute(_p(r), r.shape[0], r.shape[1], _p(q), q.shape[0], k, _p(keys), threads)
    return keys


# ---------------------------------------------------------------- numpy / Python


def np_sq_dist(a, b) -> np.float32:
    """core.py:108-122: left-to-right float32, two roundings per dimension."""
    acc = np.float32(0.0)
    for j in range(len(a)):
        diff = np.float32(a[j]) - np.float32(b[j])
        acc = np.float32(acc + np.float32(diff * diff))
    return acc


def np_pack(dists: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """core.py:152-160."""
    bits = np.ascontiguousarray(dists, dtype=np.float32).view(np.uint32)
    return (bits.astype(np.uint64) << np.uint64(32)) | np.asarray(idx).astype(np.uint64)


def np_unpack(keys: np.ndarray):
    """core.py:163-167."""
    dists = (keys >> np.uint64(32)).astype(np.uint32).view(np.float32)
    idx = (keys & np.uint64(0xFFFFFFFF)).astype(np.int64)
    return dists, idx


def np_sq_dist_block(queries: np.ndarray, points: np.ndarray) -> np.ndarray:
    """core.py:138-146 (elementwise numpy float32, no FMA)."""
    acc = np.zeros((queries.shape[0], points.shape[0]), np.float32)
    for j in range(queries.shape[1]):
        diff = queries[:, j][:, None] - points[:, j][None, :]
        acc += diff * diff
    return acc


def np_brute_keys(refs: np.ndarray, queries: np.ndarray, k: int) -> np.ndarray:
    """brute.py:41-80 / core.py:170-178 restated in numpy (small cases)."""
    refs = np.asarray(refs, np.float32)
    queries = np.asarray(queries, np.float32)
    out = np.empty((queries.shape[0], k), np.uint64)
    ids = np.arange(refs.shape[0], dtype=np.uint64)
    for lo in range(0, queries.shape[0], 256):
        dm = np_sq_dist_block(queries[lo:lo + 256], refs)
        keys = np_pack(dm, ids[None, :])
        keys.sort(axis=1)
        if keys.shape[1] >= k:
            out[lo:lo + 256] = keys[:, :k]
        else:
            out[lo:lo + 256] = EMPTY_KEY
            out[lo:lo + 256, :keys.shape[1]] = keys
    return out


def _order_bits(v: np.ndarray) -> np.ndarray:
    """kdtree.py:46-52."""
    bits = np.ascontiguousarray(v, dtype=np.float32).view(np.uint32)
    neg = (bits & np.uint32(0x80000000)) != 0
    out = bits ^ np.uint32(0x80000000)
    out[neg] = ~bits[neg]
    return out


def py_build(refs: np.ndarray, h: int):
    """buffer_tree.py:149-197 + kdtree.py:55-70 restated in numpy.

    Returns (split_values, leaf_starts, leaf member sets as sorted arrays)."""
    refs = np.asarray(refs, np.float32)
    n, d = refs.shape
    subsets = [np.arange(n, dtype=np.int64)]
    split = []
    for depth in range(h):
        dim = depth % d
        nxt = []
        for sub in subsets:
            s = sub.shape[0]
            keys = (_order_bits(refs[sub, dim]).astype(np.uint64) << np.uint64(32)) | sub.astype(np.uint64)
            order = np.argsort(keys)
            mid = s // 2
            split.append(refs[sub[order[mid]], dim])
            nxt.append(sub[order[:mid]])
            nxt.append(sub[order[mid:]])
        subsets = nxt
    sizes = np.array([s.shape[0] for s in subsets], np.int64)
    starts = np.zeros(len(subsets) + 1, np.int64)
    np.cumsum(sizes, out=starts[1:])
    return np.asarray(split, np.float32), starts, [np.sort(s) for s in subsets]


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)
