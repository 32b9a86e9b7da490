import sys, time, gc
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1512_02831_b200 as bkt
from paper_1512_02831_b200 import _native
from paper_1512_02831_b200.datasets import gen_mixture
n, m = 2_000_000, 10_000_000
pts, _ = gen_mixture(n + m, 10, components=8, spread=0.05, seed=1)
refs, queries = np.ascontiguousarray(pts.data[:n]), np.ascontiguousarray(pts.data[n:])
tree = bkt.build_buffer_tree(refs, 9)
dev = bkt.device_init(bkt.DeviceSpec(cuda_device=0))
dev.ensure_tree(tree)
res = None
for i in range(6):
    t0 = time.perf_counter()
    res = bkt.lazy_search(tree, queries, bkt.SearchParams(k=10), device=dev)
    t1 = time.perf_counter()
    print("call", i, "%.1f ms" % (1e3 * (t1 - t0)), "pool held %.0f MB" % (_native._PINNED._held / 1e6),
          {k: len(v) for k, v in _native._PINNED._free.items()}, flush=True)
