"""Distance-based outlier scoring (the paper's sec. 4.3 all-NN use case) on
the B200 engine: a self-query k+1 nearest neighbours per point, the point
itself dropped, the mean neighbour distance as the score.

Mirrors the reference's outliers.py (exclude_self_matches 22-38,
outlier_scores 41-43, rank_outliers 46-51, self_excluded_knn 54-65); the
k-NN itself runs through ``lazy_search`` (or any engine with the reference's
``engine(refs, queries, params) -> NeighborBatch`` signature).
"""
from __future__ import annotations

import numpy as np

from .core import PointMatrix, SearchParams, as_point_matrix

__all__ = ["exclude_self_matches", "outlier_scores", "rank_outliers", "self_excluded_knn", "gpu_engine"]


def exclude_self_matches(indices: np.ndarray, sq_dists: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Drop one column per row of an (n, k+1) self-query (outliers.py:22-38):
    the column holding the row's own index, or the last column when the
    point was pushed out by equal-distance neighbours."""
    rows, width = indices.shape
    if width < 2:
        raise ValueError("need at least 2 columns to drop the self match")
    hit = indices == np.arange(rows, dtype=indices.dtype).reshape(rows, 1)
    col = np.where(hit.any(axis=1), np.argmax(hit, axis=1), width - 1)
    # gather the surviving columns: positions 0..width-2 shifted past the dropped one
    pos = np.arange(width - 1).reshape(1, width - 1)
    pos = pos + (pos >= col.reshape(rows, 1))
    return np.take_along_axis(indices, pos, axis=1), np.take_along_axis(sq_dists, pos, axis=1)


def outlier_scores(sq_dists: np.ndarray) -> np.ndarray:
    """Mean Euclidean neighbour distance, float64 (outliers.py:41-43)."""
    return np.mean(np.sqrt(np.asarray(sq_dists, dtype=np.float64)), axis=1)


def rank_outliers(scores: np.ndarray) -> np.ndarray:
    """Most to least outlying (outliers.py:46-51): descending (score, index)."""
    n = int(scores.shape[0])
    ascending = np.lexsort((np.arange(n), scores))
    return ascending[::-1]


def gpu_engine(height: int | None = None, device=None, exact: bool = True):
    """An ``engine(refs, queries, params)`` callable running the B200 buffer
    k-d tree (build + lazy_search)."""
    from .buffer_tree import build_buffer_tree, lazy_search
    from .engine import auto_height

    def run(refs, queries, params: SearchParams):
        pm = as_point_matrix(refs)
        tree = build_buffer_tree(pm, height if height is not None else auto_height(pm.n))
        return lazy_search(tree, queries, params, device=device, exact=exact)

    return run


def self_excluded_knn(points: PointMatrix, k: int, engine=None) -> tuple[np.ndarray, np.ndarray]:
    """outliers.py:54-65: the k nearest other points of every point (a k+1
    self-query with the self match removed).  engine None runs the B200 engine."""
    pm = as_point_matrix(points)
    if k < 1:
        raise ValueError("k must be >= 1")
    if k + 1 > pm.n:
        raise ValueError(f"k={k} needs at least {k + 1} points, have {pm.n}")
    run = engine if engine is not None else gpu_engine()
    res = run(pm, pm.data, SearchParams(k=k + 1))
    return exclude_self_matches(res.indices, res.sq_dists)
