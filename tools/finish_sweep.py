"""Tail-finisher threshold sweep (BKT_FINISH_AT) on small-leaf trees: config-5
refs (n = 8M mixture), m queries, HBM-resident, h in {11, 14}, k = 10.

    python tools/finish_sweep.py [--m 1e6]
"""
import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1512_02831_b200 as bkt  # noqa: E402
from paper_1512_02831_b200.datasets import gen_mixture  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=float, default=1e6)
ap.add_argument("--at", default="-1,7104,30000")
a = ap.parse_args()
n, m = 8_000_000, int(a.m)
pts, _ = gen_mixture(n + m, 10, seed=1)
refs, queries = pts.data[:n], pts.data[n:]
for h in (11, 14):
    tree = bkt.build_buffer_tree(refs, h)
    dev = bkt.device_init(bkt.DeviceSpec(cuda_device=0))
    dev.ensure_tree(tree)
    ref = None
    for fa in a.at.split(","):
        if fa == "default":
            os.environ.pop("BKT_FINISH_AT", None)
            dev.search(queries, 10)
            keys, st, _ = dev.search(queries, 10, timing=True)
            print(json.dumps({"h": h, "finish_at": "default", "qps_device": m / (st["search_ms"] / 1e3),
                              "rounds": st["rounds"], "keys_equal_first": ref is None or bool(np.array_equal(keys, ref))}), flush=True)
            continue
        os.environ["BKT_FINISH_AT"] = fa
        dev.search(queries, 10)
        keys, st, _ = dev.search(queries, 10, timing=True)
        same = True if ref is None else bool(np.array_equal(keys, ref))
        ref = keys if ref is None else ref
        print(json.dumps({"h": h, "finish_at": int(fa), "qps_device": m / (st["search_ms"] / 1e3),
                          "rounds": st["rounds"], "search_ms": st["search_ms"], "keys_equal_first": same}), flush=True)
    dev.close()
