"""Exact brute-force k-NN on the B200 (the paper's brute baseline and the
tree engine's cross-check), API of the reference's brute.py:41-113.

``brute_knn`` runs the engine's own leaf scans (the tensor-core filter with
exact re-evaluation, or the CUDA-core scan) over every (query, reference)
pair: the reference set becomes an *exhaustive* two-leaf structure whose
root split value is NaN.  Every query then descends to one leaf (``q < NaN``
is false: right) and visits the other as well (the slab test
``(q - NaN)^2 > kth`` is false, so nothing is pruned) -- a full scan, with
the best k of the union, i.e. brute force, bit-identical to the reference's
numpy scan (same float32 distance order, same (distance, index) key order).
``brute_knn_chunked`` (and ``brute_knn(num_chunks > 1)``) streams the
reference set chunk by chunk through the device seam (``ChunkPipeline`` ->
``GpuDevice.enqueue_brute_kernel`` -> ``bkt_scan_groups``), as the
reference's chunked brute force does.  There is no CPU path.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .buffer_tree import BufferKdTree, LeafStructure, TopTree, lazy_search
from .core import NeighborBatch, SearchParams, as_point_matrix

__all__ = ["EvalCounter", "brute_knn", "brute_knn_chunked", "exhaustive_tree"]


@dataclass
class EvalCounter:
    """Evaluated (query, reference) pairs (brute.py:30-34)."""

    pairs: int = 0


def _queries(refs, queries) -> np.ndarray:
    q = np.ascontiguousarray(queries.data if hasattr(queries, "data") else queries, dtype=np.float32)
    if q.ndim != 2 or q.shape[1] != refs.d:
        raise ValueError(f"queries must be (m, {refs.d}), got {q.shape}")
    return q


def brute_knn_chunked(refs, queries, params: SearchParams, device, plan) -> NeighborBatch:
    """brute.py:86-113: every chunk of `plan` against every query."""
    from .device import ChunkPipeline

    pm = as_point_matrix(refs)
    q = _queries(pm, queries)
    params.validate(pm.n)
    if plan.n != pm.n:
        raise ValueError(f"plan covers {plan.n} points but refs has {pm.n}")
    m = q.shape[0]
    if m == 0:
        return NeighborBatch(0, params.k)
    out = NeighborBatch(m, params.k)
    rows = np.arange(m, dtype=np.int64)
    ids = np.arange(pm.n, dtype=np.int64)
    pipe = ChunkPipeline(device, pm.data, ids, plan)
    try:
        pipe.run_round([[(rows, lo, hi)] for lo, hi in plan.ranges()], q, out)
    finally:
        pipe.close()
    return out


def brute_knn(refs, queries, params: SearchParams, workers: int = 1, counter: EvalCounter | None = None,
              device=None, num_chunks: int = 1) -> NeighborBatch:
    """brute.py:41-83 on the GPU.  `workers` is accepted for API parity (the
    reference's thread count never changes a result); `device` defaults to
    CUDA device 0; `num_chunks` > 1 streams the reference set."""
    from .device import default_device
    from .scheduler import ChunkPlan

    if workers < 1:
        raise ValueError("workers must be >= 1")
    pm = as_point_matrix(refs)
    q = _queries(pm, queries)
    params.validate(pm.n)
    m = q.shape[0]
    if m == 0:
        return NeighborBatch(0, params.k)
    dev = device if device is not None else default_device(0)
    if num_chunks == 1 and pm.n >= 2:
        out = lazy_search(exhaustive_tree(pm), q, params, device=dev)
    else:
        out = brute_knn_chunked(pm, q, params, dev, ChunkPlan.build(pm.n, num_chunks))
    if counter is not None:
        counter.pairs += m * pm.n
    return out


def exhaustive_tree(refs) -> BufferKdTree:
    """The reference set as a two-leaf structure (points in their original
    order, split at n // 2) whose root split value is NaN: a search over it
    visits both leaves for every query, so the engine's leaf scans compute
    brute force."""
    pm = as_point_matrix(refs)
    if pm.n < 2:
        raise ValueError("an exhaustive structure needs at least 2 points")
    top = TopTree(1, pm.d, np.array([np.nan], np.float32), np.zeros(1, np.int32))
    leaves = LeafStructure(np.ascontiguousarray(pm.data, dtype=np.float32), np.arange(pm.n, dtype=np.int64),
                           np.array([0, pm.n // 2, pm.n], np.int64))
    return BufferKdTree(top, leaves)
