"""Exact brute-force k-NN on the B200 (the paper's brute baseline and the
tree engine's cross-check), API of the reference's brute.py:41-113.

Both entry points run the leaf-scan kernel of libbkt.so over every
(query, reference) pair through the device seam (``ChunkPipeline`` ->
``GpuDevice.enqueue_brute_kernel`` -> ``bkt_scan_groups``): one chunk when the
reference set fits the device, else the reference set streams through the
two chunk buffers.  Results are bit-identical to the reference's numpy scan
(same float32 distance order, same (distance, index) key order).  There is no
CPU path.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import NeighborBatch, SearchParams, as_point_matrix

__all__ = ["EvalCounter", "brute_knn", "brute_knn_chunked"]


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
    out = brute_knn_chunked(pm, q, params, dev, ChunkPlan.build(pm.n, num_chunks))
    if counter is not None:
        counter.pairs += m * pm.n
    return out
