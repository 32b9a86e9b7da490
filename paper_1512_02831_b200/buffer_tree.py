"""Buffer k-d tree: build and LazySearch on the B200.

Reference: ``buffer_tree.py`` (arXiv 1512.02831 Alg. 1).
Same public names, arguments, result type and exceptions as the reference;
the work happens in libbkt.so:

* ``build_buffer_tree`` -- native host build (``bkt_build_tree``): level-order
  top tree of 2^h - 1 split values and the leaf-sorted point copy
  (buffer_tree.py:149-197, kdtree.py:55-70).
* ``lazy_search`` -- the device-resident round loop (``bkt_search``): every
  round scans each active query against its current leaf on the GPU
  (ProcessAllBuffers), fuses FindLeafBatch into the scan epilogue, and
  re-buckets the survivors by leaf with warp-aggregated atomics and prefix
  sums (the reference's buffers / reinsert queue).  Results are the
  reference's bit for bit (``exact=True``, the default) because each query
  visits its leaves in the same order with the same float32 arithmetic; the
  buffering knobs of ``BufferConfig`` only schedule work in the reference and
  are accepted and validated here.
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _native
from .core import NeighborBatch, SearchParams, as_point_matrix

__all__ = [
    "DONE",
    "BufferConfig",
    "TopTree",
    "LeafStructure",
    "BufferKdTree",
    "BufferOverflowError",
    "SearchStats",
    "build_buffer_tree",
    "validate_structure",
    "lazy_search",
]

DONE = -1  # buffer_tree.py:50


class BufferOverflowError(RuntimeError):
    """buffer_tree.py:53-58 (kept for API compatibility: the device buffers are
    sized per round by a prefix sum and cannot overflow)."""


@dataclass(frozen=True)
class BufferConfig:
    """buffer_tree.py:61-92."""

    buffer_capacity: int
    fetch_count: int
    half_full_threshold: int

    def __post_init__(self) -> None:
        if self.buffer_capacity < 1:
            raise ValueError("buffer_capacity must be >= 1")
        if self.fetch_count < 1:
            raise ValueError("fetch_count must be >= 1")
        if not 1 <= self.half_full_threshold <= self.buffer_capacity:
            raise ValueError("half_full_threshold must be in [1, buffer_capacity]")

    @classmethod
    def for_height(cls, height: int, buffer_capacity: int | None = None, fetch_multiple: int = 10,
                   half_full_threshold: int | None = None) -> "BufferConfig":
        cap = buffer_capacity if buffer_capacity is not None else 2 ** max(0, 24 - height)
        thr = half_full_threshold if half_full_threshold is not None else max(1, cap // 2)
        return cls(buffer_capacity=cap, fetch_count=fetch_multiple * cap, half_full_threshold=thr)


@dataclass(frozen=True)
class TopTree:
    """buffer_tree.py:95-110."""

    height: int
    d: int
    split_values: np.ndarray  # (2**height - 1,) float32, level order
    levels: np.ndarray        # (2**height - 1,) int32

    @property
    def n_internal(self) -> int:
        return self.split_values.shape[0]

    @property
    def n_leaves(self) -> int:
        return self.n_internal + 1


@dataclass(frozen=True)
class LeafStructure:
    """buffer_tree.py:113-128."""

    points: np.ndarray
    original_index: np.ndarray
    leaf_starts: np.ndarray

    def bounds(self, leaf: int) -> tuple[int, int]:
        return int(self.leaf_starts[leaf]), int(self.leaf_starts[leaf + 1])


@dataclass(frozen=True)
class BufferKdTree:
    """buffer_tree.py:131-146."""

    top: TopTree
    leaves: LeafStructure

    @property
    def n(self) -> int:
        return self.leaves.points.shape[0]

    @property
    def d(self) -> int:
        return self.leaves.points.shape[1]

    @property
    def n_leaves(self) -> int:
        return self.top.n_leaves


def build_buffer_tree(refs, height: int, store_path: str | None = None, *,
                      device: int | None = None) -> BufferKdTree:
    """buffer_tree.py:149-197 via the native build.

    device None: multithreaded host build (bkt_build_tree).  device = a CUDA
    device ordinal: the same splits computed on that GPU (bkt_build_tree_device:
    per level, radix selection of every subset's positional median and a
    scan-based partition; the leaf-sorted points are gathered on the device).
    Both give the reference's split values and leaf sets exactly; the order of
    points inside a leaf is not part of the contract."""
    refs = as_point_matrix(refs)
    if height < 1:
        raise ValueError(f"height must be >= 1, got {height}")
    if 2 ** height > refs.n:
        raise ValueError(f"height {height} needs at least {2 ** height} points, have {refs.n}")
    if height > 30:
        raise ValueError(f"height {height} exceeds the supported maximum (30)")
    data = refs.data
    nl = 1 << height
    split = np.empty(nl - 1, np.float32)
    order = np.empty(refs.n, np.int64)
    starts = np.empty(nl + 1, np.int64)
    if device is None:
        _native.check(_native.lib().bkt_build_tree(_native.ptr(data), refs.n, refs.d, height, _native.ptr(split),
                                                   _native.ptr(order), _native.ptr(starts), 0))
        points = np.ascontiguousarray(data[order])
    else:
        points = np.empty_like(data)
        rc = _native.lib().bkt_build_tree_device(int(device), _native.ptr(data), refs.n, refs.d, height,
                                                 _native.ptr(split), _native.ptr(order), _native.ptr(starts),
                                                 _native.ptr(points))
        if rc != 0:
            msg = _native.lib().bkt_build_tree_device_error().decode()
            raise (ValueError if rc == _native.BKT_EINVAL else RuntimeError)(msg)
    levels = np.empty(nl - 1, dtype=np.int32)
    for lvl in range(height):
        levels[2 ** lvl - 1: 2 ** (lvl + 1) - 1] = lvl
    if store_path is not None:
        np.save(store_path, points)
        path = store_path if store_path.endswith(".npy") else store_path + ".npy"
        points = np.load(path, mmap_mode="r")
    top = TopTree(height=height, d=refs.d, split_values=split, levels=levels)
    return BufferKdTree(top=top, leaves=LeafStructure(points=points, original_index=order, leaf_starts=starts))


def validate_structure(tree: BufferKdTree, refs=None) -> None:
    """Structural audit (buffer_tree.py:200-241); raises ValueError."""
    top, leaves = tree.top, tree.leaves
    starts = leaves.leaf_starts
    n = tree.n
    if starts[0] != 0 or starts[-1] != n or np.any(np.diff(starts) < 1):
        raise ValueError("leaf ranges do not partition the point set")
    sizes = np.diff(starts)
    if sizes.max() - sizes.min() > 1:
        raise ValueError(f"leaf sizes differ by more than one: {sizes.min()}..{sizes.max()}")
    if not np.array_equal(np.sort(leaves.original_index), np.arange(n)):
        raise ValueError("original_index is not a permutation")
    if refs is not None:
        refs = as_point_matrix(refs)
        if not np.array_equal(np.asarray(leaves.points), refs.data[leaves.original_index]):
            raise ValueError("rearranged points do not match the input rows")
    pts = np.asarray(leaves.points)
    stack = [(0, 0, tree.n_leaves)]
    while stack:
        node, leaf_lo, leaf_hi = stack.pop()
        if node >= top.n_internal:
            continue
        mid = (leaf_lo + leaf_hi) // 2
        dim = int(top.levels[node]) % tree.d
        sv = top.split_values[node]
        left = pts[starts[leaf_lo]: starts[mid], dim]
        right = pts[starts[mid]: starts[leaf_hi], dim]
        if left.size and left.max() > sv:
            raise ValueError(f"node {node}: left subtree exceeds split value")
        if right.size == 0 or right.min() != sv:
            raise ValueError(f"node {node}: right subtree does not start at the split value")
        stack.append((2 * node + 1, leaf_lo, mid))
        stack.append((2 * node + 2, mid, leaf_hi))


@dataclass
class SearchStats:
    """buffer_tree.py:436-448, filled from the device counters.

    iterations / process_rounds = device rounds; leaf_scan_events = (query,
    leaf) scans; find_leaf_seconds is fused into the scan and reported as 0;
    buffer_seconds = host wall time outside the device search.  Extra
    B200 fields: pairs (algorithmic distance pairs), leafscan_ms, search_ms,
    kernel_launches, stream_bytes."""

    record_sequences: bool = False
    iterations: int = 0
    process_rounds: int = 0
    leaf_scan_events: int = 0
    spilled: int = 0
    find_leaf_seconds: float = 0.0
    buffer_seconds: float = 0.0
    visited_per_query: np.ndarray | None = None
    leaf_sequences: list[list[int]] | None = None
    pairs: int = 0
    leafscan_ms: float = 0.0
    search_ms: float = 0.0
    kernel_launches: int = 0
    leafscan_launches: int = 0
    stream_bytes: int = 0  # host-resident structure: bytes streamed into the device chunk slots


def _sequences(seq: np.ndarray, m: int) -> list[list[int]]:
    """(query, visit#, leaf) triples -> per-query leaf lists in visit order."""
    out: list[list[int]] = [[] for _ in range(m)]
    if seq.size:
        order = np.lexsort((seq[:, 1], seq[:, 0]))
        s = seq[order]
        qs, first = np.unique(s[:, 0], return_index=True)
        cuts = np.append(first, s.shape[0])
        for i, qq in enumerate(qs.tolist()):
            out[qq] = s[cuts[i]:cuts[i + 1], 2].astype(int).tolist()
    return out


def lazy_search(tree: BufferKdTree, queries, params: SearchParams, config: BufferConfig | None = None,
                device=None, plan=None, *, stats: SearchStats | None = None, debug_audit: bool = False,
                exact: bool = True, kernel: str = "auto") -> NeighborBatch:
    """Batched exact k-NN over the buffered tree on a B200 (buffer_tree.py:523-646).

    device: a ``GpuDevice`` (``device_init``); None uses CUDA device 0.
    plan: a ``ChunkPlan``; more than one chunk keeps the leaf structure in
    pinned host memory and streams it through two device chunk buffers per
    round (the paper's out-of-core workflow).  exact=False uses FMA distance
    accumulation (faster; distances within 1e-6 relative, indices equal
    except near-ties).  kernel: "auto" (tensor-core filter + exact
    re-evaluation when the tree is resident and d <= 31, else the CUDA-core
    scan), "direct" (CUDA-core scan) or "tc"; all give identical results.
    """
    from .device import DeviceConfigError, chunk_required, default_device
    from .scheduler import ChunkPlan

    t0 = time.perf_counter()
    qarr = np.ascontiguousarray(queries.data if hasattr(queries, "data") else queries, dtype=np.float32)
    if qarr.ndim != 2 or qarr.shape[1] != tree.d:
        raise ValueError(f"queries must be (m, {tree.d}), got {qarr.shape}")
    params.validate(tree.n)
    m = qarr.shape[0]
    if m == 0:
        return NeighborBatch(0, params.k)
    if config is None:
        config = BufferConfig.for_height(tree.top.height)
    if plan is not None and plan.n != tree.n:
        raise ValueError(f"plan covers {plan.n} points, structure has {tree.n}")
    dev = device if device is not None else default_device(0)
    # chunk capacity (device.py:384-392): with no plan the reference builds a
    # one-chunk plan, so the whole structure must fit one chunk buffer
    eff_plan = plan if plan is not None else ChunkPlan.build(tree.n, 1)
    if dev.chunk_bytes is not None:
        need = chunk_required(eff_plan.max_len, tree.d)
        if need > dev.chunk_bytes:
            per_point = 4 * tree.d + 8
            fit = max(1, (dev.chunk_bytes - 7) // per_point)
            suggest = -(-eff_plan.n // fit)
            raise DeviceConfigError(
                f"largest chunk ({eff_plan.max_len} points) needs {need} bytes but chunk "
                f"buffers hold {dev.chunk_bytes}; use at least {suggest} chunks")
    record = stats is not None and stats.record_sequences
    visited = np.empty(m, np.int32) if (stats is not None or debug_audit) else None
    with dev.lock:
        dev.ensure_tree(tree, plan if (plan is not None and plan.num_chunks > 1) else None)
        t1 = time.perf_counter()
        # the visit log holds one (query, visit, leaf) triple per visit that
        # happens: start from 64 per query and, if the device counted more
        # (it reports the total even when the log is full), repeat the
        # deterministic search with the exact size
        seq_cap = min(m * tree.n_leaves, 64 * m) if record else 0
        keys, st, seq = dev.search(qarr, params.k, exact=exact, visited=visited, seq_cap=seq_cap,
                                   timing=stats is not None, kernel=kernel, allow_seq_overflow=record)
        if record and st.get("seq_needed", 0) > seq_cap:
            keys, st, seq = dev.search(qarr, params.k, exact=exact, visited=visited,
                                       seq_cap=int(st["seq_needed"]), timing=True, kernel=kernel)
    t2 = time.perf_counter()
    result = NeighborBatch.from_keys(keys, params.k)  # every row is full: counts built on first access

    if debug_audit:
        # query conservation (buffer_tree.py:632-637): every query finished
        # with k real neighbours after visiting at least its home leaf
        if int(visited.min()) < 1 or int(visited.sum()) != st["leaf_visits"]:
            raise AssertionError("query conservation violated: visit counters disagree")
        if np.any((keys & np.uint64(0xFFFFFFFF)) == np.uint64(0xFFFFFFFF)):
            raise AssertionError("query conservation violated: unfinished top-k list")

    if stats is not None:
        stats.iterations += int(st["rounds"])
        stats.process_rounds += int(st["rounds"])
        stats.leaf_scan_events += int(st["leaf_visits"])
        stats.buffer_seconds += (t1 - t0) + max(0.0, (t2 - t1) - st["search_ms"] / 1e3)
        stats.visited_per_query = visited.astype(np.int64)
        stats.pairs += int(st["pairs"])
        stats.leafscan_ms += float(st["leafscan_ms"])
        stats.search_ms += float(st["search_ms"])
        stats.kernel_launches += int(st["kernel_launches"])
        stats.leafscan_launches += int(st["leafscan_launches"])
        stats.stream_bytes += int(st.get("stream_bytes", 0))
        if record:
            stats.leaf_sequences = _sequences(seq, m)
    return result
