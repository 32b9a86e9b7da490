"""Break down lazy_search on host arrays (GPU box): pageable vs page-locked
queries, wall time vs the engine's own timers."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1512_02831_b200 as bkt  # noqa: E402
from paper_1512_02831_b200 import _native  # noqa: E402
from paper_1512_02831_b200.datasets import gen_mixture  # noqa: E402

n, m = 2_000_000, 10_000_000
pts, _ = gen_mixture(n + m, 10, components=8, spread=0.05, seed=1)
refs, queries = np.ascontiguousarray(pts.data[:n]), np.ascontiguousarray(pts.data[n:])
qp = _native.pinned_empty(queries.shape, np.float32)
qp[...] = queries
tree = bkt.build_buffer_tree(refs, 9)
dev = bkt.device_init(bkt.DeviceSpec(cuda_device=0))
dev.ensure_tree(tree)
for name, q in (("pageable", queries), ("pinned", qp)):
    res = None
    for i in range(5):
        t0 = time.perf_counter()
        keys, st, _ = dev.search(q, 10, timing=True)
        t1 = time.perf_counter()
        print(f"{name} dev.search wall {1e3 * (t1 - t0):.1f} ms: search_ms {st['search_ms']:.1f} "
              f"h2d_ms {st['h2d_ms']:.1f} d2h_ms {st['d2h_ms']:.1f} leafscan_ms {st['leafscan_ms']:.1f}", flush=True)
        res = keys
    for i in range(4):
        t0 = time.perf_counter()
        r = bkt.lazy_search(tree, q, bkt.SearchParams(k=10), device=dev)
        t1 = time.perf_counter()
        print(f"{name} lazy_search wall {1e3 * (t1 - t0):.1f} ms", flush=True)
dev.close()
