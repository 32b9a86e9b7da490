"""Engine runner and sizing helpers (reference bench.py:41-204 subset).

``run_engine("bufferkdtree", ...)`` is the reference's end-to-end caller of
the hot path (bench.py:138-204): pick the height, build, size the chunk plan,
search on one GPU or a fleet, report.  Only the buffer k-d tree engine is in
scope; ``brute``/``kdtree`` are CPU baselines of the
reference and are not rebuilt.
"""
from __future__ import annotations

import hashlib
import math
import time

import numpy as np

from .buffer_tree import BufferConfig, SearchStats, build_buffer_tree, lazy_search
from .core import NeighborBatch, SearchParams, as_point_matrix
from .device import DeviceSpec, chunk_required, device_init, trace_phase_totals
from .scheduler import ChunkPlan, DeviceFleet, run_multi_device

__all__ = [
    "ENGINES",
    "DEFAULT_DEVICE_MEMORY",
    "result_digest",
    "query_block_bytes",
    "auto_height",
    "auto_num_chunks",
    "run_engine",
]

ENGINES = ("brute", "bufferkdtree")
DEFAULT_DEVICE_MEMORY = 512 * 2 ** 20  # bench.py:42 (the simulator's budget)
_PER_QUERY_OVERHEAD = 32


def result_digest(neighbors) -> str:
    """bench.py:53-57: sha256 of the (m, k) int64 index matrix."""
    idx = neighbors.indices if isinstance(neighbors, NeighborBatch) else neighbors
    arr = np.ascontiguousarray(idx, dtype="<i8")
    return hashlib.sha256(arr.tobytes()).hexdigest()


def query_block_bytes(m: int, d: int, k: int) -> int:
    """bench.py:60-62."""
    return m * (4 * d + 8 * k + _PER_QUERY_OVERHEAD)


def auto_height(n: int) -> int:
    """bench.py:65-67."""
    return max(1, min(9, int(math.log2(max(2, n // 32)))))


def auto_num_chunks(n: int, d: int, qblock: int, memory_capacity: int) -> int:
    """bench.py:70-89."""
    avail = memory_capacity - qblock
    per_point = 4 * d + 8
    if avail <= 0 or 2 * chunk_required(1, d) + qblock > memory_capacity:
        raise ValueError(f"device memory {memory_capacity} cannot hold the {qblock}-byte "
                         f"query block plus two one-point chunks")
    fit = max(1, (avail // 2 - 7) // per_point)
    num = min(n, max(1, -(-n // fit)))
    while 2 * chunk_required(-(-n // num), d) + qblock > memory_capacity:
        num += 1
        if num > n:
            raise ValueError(f"device memory {memory_capacity} too small even with one point per chunk")
    while num > 1 and 2 * chunk_required(-(-n // (num - 1)), d) + qblock <= memory_capacity:
        num -= 1
    return num


def run_engine(engine: str, refs, queries, params: SearchParams, *, height: int | None = None,
               num_chunks: int | None = None, devices: int = 1, device_memory: int | None = None,
               copy_rate: float | None = None, buffer_capacity: int | None = None, fetch_multiple: int = 10,
               half_full_threshold: int | None = None, query_chunk_size: int | None = None, workers: int = 1,
               trace_out: str | None = None, collect_stats: bool = False, exact: bool = True,
               ) -> tuple[NeighborBatch, dict]:
    """bench.py:99-204 for engines "bufferkdtree" and "brute" on B200s.

    device_memory None (default) sizes for the real GPU: one chunk, leaf
    structure resident in HBM.  An explicit budget reproduces the
    reference's chunk sizing (auto_num_chunks) and streams the leaf
    structure from pinned host memory."""
    if engine not in ENGINES:
        raise ValueError(f"unknown engine {engine!r}, expected one of {ENGINES}")
    refs = as_point_matrix(refs)
    qarr = np.ascontiguousarray(queries.data if hasattr(queries, "data") else queries, dtype=np.float32)
    m = qarr.shape[0]
    info: dict = {"engine": engine, "n": refs.n, "m": m, "d": refs.d, "k": params.k}
    if engine == "brute":
        # bench.py:119-125: the full pairwise scan, here on the GPU leaf-scan kernel
        from .brute import EvalCounter, brute_knn
        counter = EvalCounter()
        dev = device_init(DeviceSpec(cuda_device=0))
        try:
            t0 = time.perf_counter()
            res = brute_knn(refs, qarr, params, workers=workers, counter=counter, device=dev,
                            num_chunks=num_chunks or 1)
            info["query_seconds"] = time.perf_counter() - t0
        finally:
            dev.close()
        info["pairs"] = counter.pairs
        info["build_seconds"] = 0.0
        return res, info
    h = height if height is not None else auto_height(refs.n)
    t0 = time.perf_counter()
    tree = build_buffer_tree(refs, h)
    info["build_seconds"] = time.perf_counter() - t0
    config = BufferConfig.for_height(h, buffer_capacity, fetch_multiple, half_full_threshold)
    if num_chunks is None:
        if device_memory is None:
            num = 1
        else:
            resident = m if devices == 1 else max(1, min(-(-m // devices), query_chunk_size or m))
            num = auto_num_chunks(refs.n, refs.d, query_block_bytes(max(1, resident), refs.d, params.k),
                                  device_memory)
    else:
        num = num_chunks
    plan = ChunkPlan.build(refs.n, num)
    info.update(height=h, num_chunks=num, devices=devices, buffer_capacity=config.buffer_capacity,
                fetch_count=config.fetch_count, half_full_threshold=config.half_full_threshold)
    stats_list: list[SearchStats] = []
    t0 = time.perf_counter()
    if devices == 1:
        dev = device_init(DeviceSpec(cuda_device=0))
        try:
            st = SearchStats() if collect_stats else None
            res = lazy_search(tree, qarr, params, config, dev, plan, stats=st, exact=exact)
            if st is not None:
                stats_list.append(st)
            info["query_seconds"] = time.perf_counter() - t0
            phases = trace_phase_totals(dev.trace)
            info["hazard_violations"] = 0
        finally:
            dev.close()
    else:
        fleet = DeviceFleet.all_gpus(devices)
        try:
            res = run_multi_device(fleet, tree, qarr, params, config, plan, query_chunk_size,
                                   stats_out=stats_list if collect_stats else None, exact=exact)
            info["query_seconds"] = time.perf_counter() - t0
            phases = {}
            info["hazard_violations"] = 0
        finally:
            fleet.close()
    info["phase_seconds"] = phases
    if stats_list:
        info["phase_seconds"]["compute"] = sum(s.leafscan_ms for s in stats_list) / 1e3
        info["phase_seconds"]["find_leaf"] = 0.0
        info["phase_seconds"]["buffer"] = sum(s.buffer_seconds for s in stats_list)
        info["process_rounds"] = sum(s.process_rounds for s in stats_list)
        info["leaf_scan_events"] = sum(s.leaf_scan_events for s in stats_list)
        info["spilled"] = 0
        info["pairs"] = sum(s.pairs for s in stats_list)
        visited = np.concatenate([s.visited_per_query for s in stats_list if s.visited_per_query is not None])
        info["mean_leaves_visited"] = float(visited.mean()) if visited.size else 0.0
    return res, info
