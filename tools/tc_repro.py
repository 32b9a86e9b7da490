"""Parity probe for small-leaf tensor-core cases (fuzz seed 11 case 68 shape):
n ~ 4K points, d = 16 (KT = 32), h = 9 (8-point leaves), k = 10, m = 1771."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02831_b200 as bkt
from oracle import oracle as O

dev = bkt.device_init(bkt.DeviceSpec(cuda_device=0))
for fam in ("normal", "uniform"):
    for (n, d, h, k, m) in [(4147, 16, 9, 10, 1771), (4147, 16, 7, 10, 1771), (4147, 10, 9, 10, 1771),
                            (4147, 16, 9, 5, 1771), (20000, 16, 9, 10, 1771), (4147, 20, 9, 10, 1771),
                            (4147, 16, 9, 10, 200)]:
        rng = np.random.default_rng(5)
        x = rng.normal(0, 3, (n + m, d)) if fam == "normal" else rng.random((n + m, d))
        x = x.astype(np.float32)
        refs, q = x[:n], x[n:]
        tree = bkt.build_buffer_tree(refs, h)
        want = O.knn_tree(O.build_tree(refs, h), q, k, threads=8)
        out = {"fam": fam, "n": n, "d": d, "h": h, "k": k, "m": m}
        for kern in ("tc", "direct"):
            res = bkt.lazy_search(tree, q, bkt.SearchParams(k=k), device=dev, kernel=kern)
            out[kern] = int((res.keys != want["keys"]).any(axis=1).sum())
        print(json.dumps(out), flush=True)
dev.close()
