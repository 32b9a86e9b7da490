"""ctypes binding of libbkt.so (include/bkt.h).

The library is built in-tree by ``python -m paper_1512_02831_b200.build`` (or
``__graft_entry__.build()``).  There is no fallback: if the library is
missing, every engine call raises ``NativeLibraryMissing``.
"""
from __future__ import annotations

import ctypes
import mmap
import os
import threading
import weakref
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "_lib" / os.environ.get("BKT_LIB_NAME", "libbkt.so")

BKT_OK = 0
BKT_EINVAL = -1
BKT_ECONFIG = -2
BKT_ECUDA = -3
BKT_ENOMEM = -4
BKT_ESTATE = -5

# every symbol include/bkt.h declares
EXPORTS = ("bkt_open", "bkt_close", "bkt_last_error", "bkt_device_info", "bkt_build_tree",
           "bkt_build_tree_device", "bkt_build_tree_device_error", "bkt_load_tree", "bkt_search",
           "bkt_scan_groups", "bkt_seam_copy", "bkt_seam_sync", "bkt_seam_scan", "bkt_fp32_peak",
           "bkt_host_alloc", "bkt_host_free", "bkt_set_spill_dir")


class NativeLibraryMissing(RuntimeError):
    """libbkt.so is not built; the engine has no CPU fallback."""


class SearchOpts(ctypes.Structure):
    _fields_ = [
        ("exact", ctypes.c_int32),
        ("queries_on_device", ctypes.c_int32),
        ("keys_on_device", ctypes.c_int32),
        ("record_timing", ctypes.c_int32),
        ("batch_queries", ctypes.c_int64),
        ("visited_out", ctypes.c_void_p),
        ("seq_log", ctypes.c_void_p),
        ("seq_cap", ctypes.c_int64),
        ("seq_count_out", ctypes.c_void_p),
        ("kernel", ctypes.c_int32),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("rounds", ctypes.c_int64),
        ("leaf_visits", ctypes.c_int64),
        ("pairs", ctypes.c_int64),
        ("kernel_launches", ctypes.c_int64),
        ("leafscan_launches", ctypes.c_int64),
        ("leafscan_ms", ctypes.c_double),
        ("search_ms", ctypes.c_double),
        ("h2d_ms", ctypes.c_double),
        ("d2h_ms", ctypes.c_double),
        ("h2d_bytes", ctypes.c_int64),
        ("d2h_bytes", ctypes.c_int64),
        ("stream_bytes", ctypes.c_int64),
        ("stream_copies", ctypes.c_int64),
    ]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None
_lock = threading.Lock()


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise NativeLibraryMissing(
                f"{LIB_PATH} is not built; run `python -m paper_1512_02831_b200.build` "
                "(this engine has no CPU fallback)")
        L = ctypes.CDLL(str(LIB_PATH))
        P = ctypes.c_void_p
        i32, i64 = ctypes.c_int32, ctypes.c_int64
        L.bkt_open.argtypes = [ctypes.c_int, ctypes.POINTER(P)]
        L.bkt_close.argtypes = [P]
        L.bkt_close.restype = None
        L.bkt_last_error.argtypes = [P]
        L.bkt_last_error.restype = ctypes.c_char_p
        L.bkt_device_info.argtypes = [P, P, P, P, P]
        L.bkt_build_tree.argtypes = [P, i64, i32, i32, P, P, P, i32]
        L.bkt_build_tree_device.argtypes = [ctypes.c_int, P, i64, i32, i32, P, P, P, P]
        L.bkt_build_tree_device_error.argtypes = []
        L.bkt_build_tree_device_error.restype = ctypes.c_char_p
        L.bkt_load_tree.argtypes = [P, i32, i32, i64, P, P, P, P, i32, i32, P]
        L.bkt_set_spill_dir.argtypes = [P, ctypes.c_char_p]
        L.bkt_search.argtypes = [P, P, i64, i32, ctypes.POINTER(SearchOpts), P, ctypes.POINTER(Stats)]
        L.bkt_scan_groups.argtypes = [P, P, P, i64, i32, P, i64, i32, P, i32, P, P, P, P, i32]
        L.bkt_seam_copy.argtypes = [P, i32, P, P, i64, i32]
        L.bkt_seam_sync.argtypes = [P, i32]
        L.bkt_seam_scan.argtypes = [P, i32, P, i64, i32, P, i32, P, P, P, P, i32]
        L.bkt_fp32_peak.argtypes = [P, ctypes.POINTER(ctypes.c_double)]
        L.bkt_host_alloc.argtypes = [i64]
        L.bkt_host_alloc.restype = P
        L.bkt_host_free.argtypes = [P]
        L.bkt_host_free.restype = None
        for name in EXPORTS:
            fn = getattr(L, name)
            if fn.restype is ctypes.c_int:  # default
                fn.restype = ctypes.c_int
        _lib = L
        return _lib


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.c_void_p)


def check(rc: int, ctx=None) -> None:
    """Map a libbkt return code to the reference's exception types."""
    if rc == BKT_OK:
        return
    msg = lib().bkt_last_error(ctx).decode(errors="replace") if lib() else ""
    if rc == BKT_EINVAL:
        raise ValueError(msg)
    if rc == BKT_ECONFIG:
        from .device import DeviceConfigError
        raise DeviceConfigError(msg)
    raise RuntimeError(msg or f"libbkt error {rc}")


class _PinnedPool:
    """Recycles page-locked host buffers for result arrays.  cudaHostAlloc of
    hundreds of MB costs more than the search, so a buffer goes back to the
    pool (keyed by size) when the last array viewing it is collected, and the
    next result of that size reuses it.  Results then leave the GPU at full
    PCIe speed straight into the array the caller keeps."""

    def __init__(self, max_bytes: int = 4 << 30, per_size: int = 2) -> None:
        self._free: dict[int, list[int]] = {}
        self._count: dict[int, int] = {}
        self._lock = threading.Lock()
        self._held = 0
        self._max = max_bytes
        self._per_size = per_size
        self._filling: set[int] = set()

    def _fill(self, nbytes: int) -> None:
        # page-lock buffers of this size one after another up to `per_size`
        # (a caller that keeps its previous result alive needs two; a third
        # covers one more live reference, e.g. a checker's copy)
        while True:
            with self._lock:
                if self._held + nbytes > self._max or self._count.get(nbytes, 0) >= self._per_size:
                    self._filling.discard(nbytes)
                    return
            try:
                addr = lib().bkt_host_alloc(nbytes)
            except Exception:  # pragma: no cover - no driver
                addr = None
            with self._lock:
                if not addr:
                    self._filling.discard(nbytes)
                    return
                self._held += nbytes
                self._count[nbytes] = self._count.get(nbytes, 0) + 1
                self._free.setdefault(nbytes, []).append(addr)

    def take(self, nbytes: int):
        # A free buffer of this size is handed out at once.  Otherwise the
        # caller gets ordinary memory now and a buffer is page-locked in the
        # background (cudaHostAlloc costs ~0.4 s per 800 MB), up to
        # `per_size` per size in one go: a caller that keeps many results
        # alive (a stream) never waits for the allocation.
        with self._lock:
            lst = self._free.get(nbytes)
            if lst:
                return lst.pop()
            if (self._held + nbytes > self._max or self._count.get(nbytes, 0) >= self._per_size
                    or nbytes in self._filling):
                return None
            self._filling.add(nbytes)
        threading.Thread(target=self._fill, args=(nbytes,), daemon=True).start()
        return None

    def give(self, nbytes: int, addr: int) -> None:
        with self._lock:
            self._free.setdefault(nbytes, []).append(addr)


_PINNED = _PinnedPool(max_bytes=0 if os.environ.get("BKT_NO_PINNED_POOL") else 6 << 30, per_size=3)


def pinned_empty(shape, dtype) -> np.ndarray:
    """A page-locked host array (bkt_host_alloc), freed when the array is
    collected.  Query arrays in page-locked memory reach the device in one
    direct DMA (bkt_search skips its staging copy)."""
    dt = np.dtype(dtype)
    nbytes = max(1, int(np.prod(shape)) * dt.itemsize)
    addr = lib().bkt_host_alloc(nbytes)
    if not addr:
        raise MemoryError(f"bkt_host_alloc({nbytes}) failed")
    buf = (ctypes.c_char * nbytes).from_address(addr)
    weakref.finalize(buf, lib().bkt_host_free, addr)
    return np.frombuffer(buf, dtype=dt, count=int(np.prod(shape))).reshape(shape)


def host_empty(shape, dtype) -> np.ndarray:
    """np.empty for large host result arrays.

    Large arrays come from the page-locked pool (see _PinnedPool); if that is
    unavailable (no GPU driver, pool exhausted) they fall back to 2 MB
    transparent huge pages when the kernel allows it (madvise mode): writing a
    fresh 800 MB result through 4 KB pages costs ~140 ms of page faults, more
    than its DMA."""
    dt = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dt.itemsize
    if nbytes < (64 << 20):
        return np.empty(shape, dt)
    try:
        addr = _PINNED.take(nbytes)
    except NativeLibraryMissing:
        addr = None
    if addr:
        buf = (ctypes.c_char * nbytes).from_address(addr)
        weakref.finalize(buf, _PINNED.give, nbytes, addr)
        return np.frombuffer(buf, dtype=dt).reshape(shape)
    if not hasattr(mmap, "MADV_HUGEPAGE"):
        return np.empty(shape, dt)
    mm = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    try:
        mm.madvise(mmap.MADV_HUGEPAGE)
    except OSError:
        pass
    return np.frombuffer(mm, dtype=dt).reshape(shape)
