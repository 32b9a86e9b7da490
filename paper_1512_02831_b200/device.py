"""The B200 device handle: budget checks, tree residency, and the reference's
device plugin seam.

Reference counterpart: ``device.py`` (SimulatedDevice, DeviceSpec,
device_init, ChunkPipeline, chunk_required).  The reference simulates a
constrained-memory accelerator with two Python-thread command queues; here a
``GpuDevice`` owns one CUDA context of libbkt (``bkt_open``), two CUDA streams
and real device buffers:

* the coarse seam (what ``lazy_search``/``run_multi_device`` use): the tree is
  uploaded once per device (``bkt_load_tree``) and each search runs the whole
  device-resident round loop (``bkt_search``);
* the fine seam the reference's ``ChunkPipeline`` drives
  (``enqueue_stage``/``enqueue_copy``/``enqueue_brute_kernel``/``wait``,
  device.py:228-349): staging is host-side, the brute kernel runs on the GPU
  (``bkt_scan_groups``).  Commands complete before ``enqueue_*`` returns, so
  the returned events are already done and CUDA stream order makes the
  reference's reader/writer hazard checker unnecessary
  (``hazard_violations`` stays empty).
"""
from __future__ import annotations

import ctypes
import os
import threading
import time
from dataclasses import dataclass

import numpy as np

from . import _native
from .core import NeighborBatch

__all__ = [
    "DeviceSpec",
    "DeviceConfigError",
    "PipelineHazardError",
    "Event",
    "GpuDevice",
    "ChunkPipeline",
    "device_init",
    "run_chunk_pipeline",
    "chunk_required",
    "trace_phase_totals",
    "default_device",
]


# leaf-scan kernel selection (bkt_search_opts.kernel): "auto" uses the
# tensor-core filter whenever the tree is resident and d <= 31
_KERNELS = {"auto": 0, "direct": 1, "tc": 2}


class DeviceConfigError(ValueError):
    """A requested configuration does not fit the device (device.py:49-50)."""


class PipelineHazardError(RuntimeError):
    """Kept for API compatibility (device.py:53-54); CUDA stream ordering
    rules out the simulator's buffer hazards, so it is never raised."""


def chunk_required(n_points: int, d: int) -> int:
    """device.py:57-61: bytes of one chunk buffer (f32 coords + i64 ids)."""
    pts = n_points * d * 4
    return (pts + 7) // 8 * 8 + n_points * 8


class Event:
    """Completion handle (device.py:64-88).  A chunk copy's event waits for
    the CUDA event its slot recorded on the copy stream (bkt_seam_sync);
    other commands complete before they return.  A failed command re-raises
    on wait."""

    __slots__ = ("_exc", "_sync", "_done")

    def __init__(self, exc: BaseException | None = None, sync=None) -> None:
        self._exc = exc
        self._sync = sync
        self._done = sync is None

    @property
    def done(self) -> bool:
        return self._done

    def wait(self, timeout: float | None = None) -> None:
        if self._exc is not None:
            raise self._exc
        if not self._done:
            self._sync()
            self._done = True


@dataclass(frozen=True)
class DeviceSpec:
    """device.py:165-178 plus the CUDA ordinal.

    memory_capacity None means "the GPU's free memory".  worker_lanes and
    simulated_copy_rate are simulator knobs; they are accepted and ignored
    (the GPU's own parallelism and PCIe rate apply)."""

    memory_capacity: int | None = None
    worker_lanes: int = 1
    simulated_copy_rate: float | None = None
    cuda_device: int = 0
    # host-resident (chunked) structures in file-backed pages under this
    # directory instead of page-locked RAM (bkt_set_spill_dir): disk -> host
    # -> device streaming for structures larger than host memory
    spill_dir: str | None = None


class GpuDevice:
    """One B200 (device.py:181-358 SimulatedDevice counterpart)."""

    def __init__(self, spec: DeviceSpec, chunk_bytes: int | None = None,
                 query_block_bytes: int = 0) -> None:
        if chunk_bytes is not None and (chunk_bytes < 1 or query_block_bytes < 0):
            raise DeviceConfigError("chunk_bytes must be >= 1 and query block >= 0")
        if spec.worker_lanes < 1:
            raise DeviceConfigError("worker_lanes must be >= 1")
        if chunk_bytes is not None and spec.memory_capacity is not None:
            required = 2 * chunk_bytes + query_block_bytes
            if required > spec.memory_capacity:
                raise DeviceConfigError(
                    f"device memory exceeded: need {required} bytes "
                    f"(2 x {chunk_bytes} chunk buffers + {query_block_bytes} query block), "
                    f"capacity is {spec.memory_capacity}")
        self.spec = spec
        self.chunk_bytes = chunk_bytes
        self.query_block_bytes = query_block_bytes
        self.hazard_violations: list[str] = []
        self.trace: list[tuple[str, str, int, int, int]] = []
        # staged chunks live in page-locked buffers (so the slot copy is an
        # asynchronous DMA); the device slots hold (L, d, chunk id) of their chunk
        self._staging: list[tuple[np.ndarray, np.ndarray] | None] = [None, None]
        self._resident: list[tuple[int, int, int] | None] = [None, None]
        self._staged_len = [0, 0]
        self._tree_key = None
        self._tree_ref = None
        self._closed = False
        # One bkt context serves one call at a time (include/bkt.h): calls
        # from several host threads on this device serialise here.
        self.lock = threading.RLock()
        h = ctypes.c_void_p()
        _native.check(_native.lib().bkt_open(int(spec.cuda_device), ctypes.byref(h)))
        self._ctx = h
        if spec.spill_dir:
            _native.check(_native.lib().bkt_set_spill_dir(h, os.fsencode(spec.spill_dir)), h)

    # ------------------------------------------------------------------ info
    @property
    def ctx(self):
        if self._closed:
            raise RuntimeError("device is closed")
        return self._ctx

    def info(self) -> dict:
        sm = ctypes.c_int32()
        clk = ctypes.c_int32()
        fr = ctypes.c_int64()
        to = ctypes.c_int64()
        L = _native.lib()
        _native.check(L.bkt_device_info(self.ctx, ctypes.byref(sm), ctypes.byref(clk), ctypes.byref(fr),
                                        ctypes.byref(to)), self.ctx)
        return {"sm_count": sm.value, "sm_clock_khz": clk.value, "free_bytes": fr.value,
                "total_bytes": to.value, "cuda_device": self.spec.cuda_device}

    def fp32_peak_tflops(self) -> float:
        v = ctypes.c_double()
        _native.check(_native.lib().bkt_fp32_peak(self.ctx, ctypes.byref(v)), self.ctx)
        return v.value

    def _record(self, kind: str, queue_id: str, chunk_id: int, t0: int, t1: int) -> None:
        self.trace.append((kind, queue_id, chunk_id, t0, t1))

    def write_trace(self, path: str) -> None:
        """device.py:219-224 CSV format."""
        with open(path, "w", encoding="utf-8") as fh:
            for kind, qid, cid, t0, t1 in self.trace:
                fh.write(f"{kind},{qid},{cid},{t0},{t1}\n")

    # ------------------------------------------------------- coarse seam
    def ensure_tree(self, tree, plan=None) -> None:
        """Upload `tree` (once) with the residency the plan asks for.

        plan None or one chunk: leaf structure resident in HBM.  More chunks:
        host-resident pinned copy streamed through two device chunk buffers
        each round (sec. 3.2)."""
        num = 1 if plan is None else plan.num_chunks
        bounds = None if plan is None else np.ascontiguousarray(plan.bounds, dtype=np.int64)
        key = (id(tree), num, None if bounds is None else bounds.tobytes())
        with self.lock:
            if self._tree_key == key and self._tree_ref is tree:
                return
            self._load_tree(tree, num, bounds, key)

    def _load_tree(self, tree, num, bounds, key) -> None:
        top, leaves = tree.top, tree.leaves
        pts = np.ascontiguousarray(np.asarray(leaves.points), dtype=np.float32)
        orig = np.ascontiguousarray(leaves.original_index, dtype=np.int64)
        starts = np.ascontiguousarray(leaves.leaf_starts, dtype=np.int64)
        split = np.ascontiguousarray(top.split_values, dtype=np.float32)
        residency = 0 if num == 1 else 1
        _native.check(_native.lib().bkt_load_tree(
            self.ctx, int(top.height), int(tree.d), int(tree.n), _native.ptr(split), _native.ptr(pts),
            _native.ptr(orig), _native.ptr(starts), residency, int(num), _native.ptr(bounds)), self.ctx)
        self._tree_key = key
        self._tree_ref = tree

    def search(self, queries: np.ndarray, k: int, *, exact: bool = True, visited: np.ndarray | None = None,
               seq_cap: int = 0, timing: bool = False, batch_queries: int = 0,
               out_keys: np.ndarray | None = None, kernel: str = "auto",
               allow_seq_overflow: bool = False) -> tuple[np.ndarray, dict, np.ndarray | None]:
        """bkt_search on host arrays; returns (keys, stats, seq triples).
        stats["seq_needed"] is the number of visits the device counted; with
        allow_seq_overflow a log smaller than that is returned truncated
        (the caller repeats the search with the exact size)."""
        q = np.ascontiguousarray(queries, dtype=np.float32)
        m = q.shape[0]
        keys = out_keys if out_keys is not None else _native.host_empty((m, k), np.uint64)
        opts = _native.SearchOpts()
        opts.exact = 1 if exact else 0
        opts.record_timing = 1 if timing else 0
        opts.batch_queries = int(batch_queries)
        opts.kernel = _KERNELS[kernel]
        if visited is not None:
            opts.visited_out = visited.ctypes.data
        seq = None
        seq_count = ctypes.c_int64(0)
        if seq_cap:
            seq = np.empty((seq_cap, 3), dtype=np.int32)
            opts.seq_log = seq.ctypes.data
            opts.seq_cap = int(seq_cap)
            opts.seq_count_out = ctypes.addressof(seq_count)
        st = _native.Stats()
        with self.lock:
            _native.check(_native.lib().bkt_search(self.ctx, _native.ptr(q), m, int(k), ctypes.byref(opts),
                                                   _native.ptr(keys), ctypes.byref(st)), self.ctx)
        out = st.as_dict()
        if seq is not None:
            out["seq_needed"] = int(seq_count.value)
            if seq_count.value > seq_cap and not allow_seq_overflow:
                raise RuntimeError("leaf sequence log overflowed")
            seq = seq[: min(seq_count.value, seq_cap)]
        return keys, out, seq

    def search_device(self, q_dev_ptr: int, m: int, k: int, keys_dev_ptr: int, *, exact: bool = True,
                      timing: bool = False, kernel: str = "auto") -> dict:
        """bkt_search with inputs and outputs already in this GPU's memory
        (raw device pointers, e.g. from torch tensors)."""
        opts = _native.SearchOpts()
        opts.exact = 1 if exact else 0
        opts.queries_on_device = 1
        opts.keys_on_device = 1
        opts.record_timing = 1 if timing else 0
        opts.kernel = _KERNELS[kernel]
        st = _native.Stats()
        with self.lock:
            _native.check(_native.lib().bkt_search(self.ctx, ctypes.c_void_p(q_dev_ptr), int(m), int(k),
                                                   ctypes.byref(opts), ctypes.c_void_p(keys_dev_ptr),
                                                   ctypes.byref(st)), self.ctx)
        return st.as_dict()

    # --------------------------------------------------------- fine seam
    def enqueue_stage(self, queue_id: str, slot: int, points_src: np.ndarray, ids_src: np.ndarray,
                      chunk_id: int, deps: tuple = ()) -> Event:
        """device.py:228-254: host slice -> staging[slot]."""
        L, d = points_src.shape
        need = chunk_required(L, d)
        if self.chunk_bytes is not None and need > self.chunk_bytes:
            raise DeviceConfigError(
                f"chunk of {L} points x {d} dims needs {need} bytes, "
                f"chunk buffers hold {self.chunk_bytes}")
        for dep in deps:
            dep.wait()
        t0 = time.monotonic_ns()
        # the slot's previous copy must have left its staging buffer
        _native.check(_native.lib().bkt_seam_sync(self.ctx, int(slot)), self.ctx)
        cur = self._staging[slot]
        if cur is None or cur[0].shape[0] < L or cur[0].shape[1] != d:
            pts = _native.pinned_empty((max(L, 1), d), np.float32)
            ids = np.empty(max(L, 1), np.int64)
            cur = (pts, ids)
        cur[0][:L] = points_src
        cur[1][:L] = ids_src
        self._staging[slot] = cur
        self._staged_len[slot] = L
        self._record("stage", queue_id, chunk_id, t0, time.monotonic_ns())
        return Event()

    def enqueue_copy(self, queue_id: str, slot: int, nbytes: int, chunk_id: int, deps: tuple = ()) -> Event:
        """device.py:256-281: staging[slot] -> device chunk buffer `slot`."""
        if self.chunk_bytes is not None and nbytes > self.chunk_bytes:
            raise DeviceConfigError(f"copy of {nbytes} bytes exceeds chunk buffer")
        for dep in deps:
            dep.wait()
        t0 = time.monotonic_ns()
        pts, ids = self._staging[slot]
        L = self._staged_len[slot]
        _native.check(_native.lib().bkt_seam_copy(self.ctx, int(slot), _native.ptr(pts), _native.ptr(ids), L,
                                                  int(pts.shape[1])), self.ctx)
        self._resident[slot] = (L, int(pts.shape[1]), chunk_id)
        self._record("copy", queue_id, chunk_id, t0, time.monotonic_ns())
        ctx = self.ctx
        return Event(sync=lambda: _native.check(_native.lib().bkt_seam_sync(ctx, int(slot)), ctx))

    def enqueue_brute_kernel(self, queue_id: str, slot: int, chunk_lo: int, chunk_hi: int, d: int,
                             groups: list, queries: np.ndarray, neighbors: NeighborBatch, chunk_id: int,
                             deps: tuple = ()) -> Event:
        """device.py:283-337: scan the resident chunk for each (rows, lo, hi)
        group on the GPU and merge into `neighbors` (core.py:251-262)."""
        for rows, lo, hi in groups:
            if not (chunk_lo <= lo < hi <= chunk_hi):
                raise ValueError(f"group range [{lo}, {hi}) outside chunk [{chunk_lo}, {chunk_hi})")
            if rows.shape[0] == 0:
                raise ValueError("empty query group")
        for dep in deps:
            dep.wait()
        t0 = time.monotonic_ns()
        res = self._resident[slot]
        if res is None or res[0] != chunk_hi - chunk_lo:
            raise ValueError("resident chunk does not match [chunk_lo, chunk_hi)")
        if groups:
            rows_all = np.concatenate([np.asarray(r, np.int64) for r, _, _ in groups])
            ptr = np.zeros(len(groups) + 1, np.int64)
            np.cumsum([len(r) for r, _, _ in groups], out=ptr[1:])
            glo = np.array([lo - chunk_lo for _, lo, _ in groups], np.int64)
            ghi = np.array([hi - chunk_lo for _, _, hi in groups], np.int64)
            q = np.ascontiguousarray(queries, np.float32)
            keys = neighbors.keys
            if not keys.flags.c_contiguous:
                raise ValueError("neighbors.keys must be C-contiguous")
            # the scan waits for the slot's copy on the device (stream order), not on the host
            _native.check(_native.lib().bkt_seam_scan(
                self.ctx, int(slot), _native.ptr(q), q.shape[0], int(neighbors.k), _native.ptr(keys), len(groups),
                _native.ptr(ptr), _native.ptr(rows_all), _native.ptr(glo), _native.ptr(ghi), 1), self.ctx)
            for rows, lo, hi in groups:
                neighbors.counts[rows] = np.minimum(neighbors.counts[rows] + (hi - lo), neighbors.k)
        self._record("compute", queue_id, chunk_id, t0, time.monotonic_ns())
        return Event()

    def wait(self, target) -> None:
        """device.py:339-349."""
        if isinstance(target, Event):
            target.wait()
            return
        now = time.monotonic_ns()
        self._record("marker", target, -1, now, now)

    def close(self) -> None:
        if self._closed:
            return
        self._closed = True
        _native.lib().bkt_close(self._ctx)
        self._tree_ref = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass


def device_init(spec: DeviceSpec, chunk_bytes: int | None = None, query_block_bytes: int = 0) -> GpuDevice:
    """device.py:361-364."""
    return GpuDevice(spec, chunk_bytes, query_block_bytes)


_DEFAULT: dict[int, GpuDevice] = {}
_DEFAULT_LOCK = threading.Lock()


def default_device(cuda_device: int = 0) -> GpuDevice:
    """Process-wide device used when lazy_search gets device=None (its
    ``lock`` serialises concurrent callers; the reference instead builds a
    private simulated device per call, buffer_tree.py:553-561)."""
    with _DEFAULT_LOCK:
        dev = _DEFAULT.get(cuda_device)
        if dev is None or dev._closed:
            dev = GpuDevice(DeviceSpec(cuda_device=cuda_device))
            _DEFAULT[cuda_device] = dev
        return dev


class ChunkPipeline:
    """Streams (points, ids) chunks through a device's two chunk buffers
    (device.py:367-457) over the fine seam: per chunk j the brute kernel runs
    on the resident chunk, then the next chunk is staged and copied into the
    other slot."""

    def __init__(self, device: GpuDevice, points: np.ndarray, ids: np.ndarray, plan) -> None:
        if points.shape[0] != plan.n:
            raise ValueError(f"plan covers {plan.n} points, structure has {points.shape[0]}")
        need = chunk_required(plan.max_len, points.shape[1])
        if device.chunk_bytes is not None and need > device.chunk_bytes:
            d = points.shape[1]
            per_point = 4 * d + 8
            fit = max(1, (device.chunk_bytes - 7) // per_point)
            suggest = -(-plan.n // fit)
            raise DeviceConfigError(
                f"largest chunk ({plan.max_len} points) needs {need} bytes but chunk "
                f"buffers hold {device.chunk_bytes}; use at least {suggest} chunks")
        self.device = device
        self.points = points
        self.ids = ids
        self.plan = plan
        self._next_slot = 0
        self._slot_chunk: list[int | None] = [None, None]

    def _load(self, chunk_id: int, queue_id: str) -> None:
        slot = self._next_slot
        self._next_slot ^= 1
        lo, hi = self.plan.range(chunk_id)
        self.device.enqueue_stage(queue_id, slot, self.points[lo:hi], self.ids[lo:hi], chunk_id)
        self.device.enqueue_copy(queue_id, slot, chunk_required(hi - lo, self.points.shape[1]), chunk_id)
        if self._slot_chunk[1 - slot] == chunk_id:
            self._slot_chunk[1 - slot] = None
        self._slot_chunk[slot] = chunk_id

    def run_round(self, groups_per_chunk: list, queries: np.ndarray, neighbors: NeighborBatch) -> None:
        plan = self.plan
        N = plan.num_chunks
        if len(groups_per_chunk) != N:
            raise ValueError(f"expected {N} group lists, got {len(groups_per_chunk)}")
        d = self.points.shape[1]
        if self._slot_chunk[0] is None and self._slot_chunk[1] is None:
            self._load(0, "A")
        for j in range(N):
            kq = "A" if j % 2 == 0 else "B"
            slot = self._slot_chunk.index(j)
            lo, hi = plan.range(j)
            # the next chunk is staged and its copy issued into the other slot
            # first, so the DMA (queue B) runs while this chunk's kernel (queue
            # A) scans (device.py:432-446)
            if N > 1:
                nxt = j + 1 if j + 1 < N else 0
                self._load(nxt, "B" if kq == "A" else "A")
            if groups_per_chunk[j]:
                ev = self.device.enqueue_brute_kernel(kq, slot, lo, hi, d, groups_per_chunk[j], queries,
                                                      neighbors, chunk_id=j)
                self.device.wait(ev)

    def close(self) -> None:
        pass


def run_chunk_pipeline(device: GpuDevice, points: np.ndarray, ids: np.ndarray, plan, groups_per_chunk,
                       queries: np.ndarray, neighbors: NeighborBatch) -> None:
    """device.py:460-468."""
    pipeline = ChunkPipeline(device, points, ids, plan)
    try:
        pipeline.run_round(groups_per_chunk, queries, neighbors)
    finally:
        pipeline.close()


def trace_phase_totals(trace) -> dict[str, float]:
    """device.py:474-479."""
    out: dict[str, float] = {}
    for kind, _qid, _cid, t0, t1 in trace:
        out[kind] = out.get(kind, 0.0) + (t1 - t0) / 1e9
    return out
