"""Break down the end-to-end lazy_search time on host arrays (GPU box)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1512_02831_b200 as bkt  # noqa: E402
from paper_1512_02831_b200.datasets import gen_mixture  # noqa: E402

print("THP:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
n, m = 2_000_000, 10_000_000
pts, _ = gen_mixture(n + m, 10, components=8, spread=0.05, seed=1)
refs, queries = np.ascontiguousarray(pts.data[:n]), np.ascontiguousarray(pts.data[n:])
tree = bkt.build_buffer_tree(refs, 9)
dev = bkt.device_init(bkt.DeviceSpec(cuda_device=0))
dev.ensure_tree(tree)
for i in range(3):
    t0 = time.perf_counter()
    a = np.empty((m, 10), np.uint64)
    a.fill(0)
    t1 = time.perf_counter()
    print("fresh 800 MB fill %.1f ms" % (1e3 * (t1 - t0)))
for i in range(3):
    t0 = time.perf_counter()
    keys, st, _ = dev.search(queries, 10, timing=True)
    t1 = time.perf_counter()
    print("dev.search %.1f ms: search_ms %.1f h2d_ms %.1f d2h_ms %.1f" % (1e3 * (t1 - t0), st["search_ms"], st["h2d_ms"], st["d2h_ms"]))
out = np.empty((m, 10), np.uint64)
for i in range(2):
    t0 = time.perf_counter()
    keys, st, _ = dev.search(queries, 10, timing=True, out_keys=out)
    t1 = time.perf_counter()
    print("dev.search (reused out) %.1f ms: search_ms %.1f h2d_ms %.1f d2h_ms %.1f" % (1e3 * (t1 - t0), st["search_ms"], st["h2d_ms"], st["d2h_ms"]))
for i in range(2):
    t0 = time.perf_counter()
    res = bkt.lazy_search(tree, queries, bkt.SearchParams(k=10), device=dev)
    t1 = time.perf_counter()
    print("lazy_search %.1f ms" % (1e3 * (t1 - t0)))
