import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1512_02831_b200 as bkt
from paper_1512_02831_b200.datasets import gen_mixture
n, m = 2_000_000, 10_000_000
pts, _ = gen_mixture(n + m, 10, components=8, spread=0.05, seed=1)
refs, queries = np.ascontiguousarray(pts.data[:n]), np.ascontiguousarray(pts.data[n:])
tree = bkt.build_buffer_tree(refs, 9)
dev = bkt.device_init(bkt.DeviceSpec(cuda_device=0))
flush = torch.empty(64 << 20, dtype=torch.float32, device='cuda')
res = None
for mode in ("plain", "flush", "flush+hold", "plain+hold"):
    ts = []
    for i in range(5):
        if "flush" in mode:
            flush.fill_(1.0); torch.cuda.synchronize()
        if "hold" not in mode:
            res = None
        t0 = time.perf_counter()
        r = bkt.lazy_search(tree, queries, bkt.SearchParams(k=10), device=dev)
        ts.append(time.perf_counter() - t0)
        res = r
        del r
    print(mode, ["%.1f" % (1e3 * t) for t in ts], flush=True)
