"""Height x mode sweep of the config-2 workload on one GPU (device-resident).

    python tools/sweep.py [--m 10000000] [--heights 9 10 11 12] [--modes fma exact]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1512_02831_b200 as bkt  # noqa: E402
from paper_1512_02831_b200.datasets import gen_mixture  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2_000_000)
    ap.add_argument("--m", type=int, default=10_000_000)
    ap.add_argument("--d", type=int, default=10)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--heights", type=int, nargs="+", default=[9, 10, 11, 12])
    ap.add_argument("--modes", nargs="+", default=["fma", "exact"])
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--kernels", nargs="+", default=["direct", "tc"])
    a = ap.parse_args()
    import torch
    t0 = time.time()
    pts, _ = gen_mixture(a.n + a.m, a.d, seed=1)
    refs, queries = pts.data[: a.n], pts.data[a.n:]
    print(f"data {time.time() - t0:.1f}s", flush=True)
    dev = bkt.device_init(bkt.DeviceSpec(cuda_device=0))
    peak = dev.fp32_peak_tflops()
    q = torch.from_numpy(np.ascontiguousarray(queries)).cuda()
    keys = torch.empty((a.m, a.k), dtype=torch.int64, device="cuda")
    for h in a.heights:
        tree = bkt.build_buffer_tree(refs, h)
        dev.ensure_tree(tree)
        for mode, kern in [(mo, ke) for ke in a.kernels for mo in a.modes]:
            best = None
            for r in range(a.reps + 1):
                st = dev.search_device(q.data_ptr(), a.m, a.k, keys.data_ptr(), exact=(mode == "exact"), timing=True, kernel=kern)
                if (r > 0 or a.reps == 0) and (best is None or st["search_ms"] < best["search_ms"]):
                    best = st
            st = best
            qps = a.m / (st["search_ms"] / 1e3)
            tf = 3 * a.d * st["pairs"] / (st["leafscan_ms"] / 1e3) / 1e12
            print(json.dumps({"h": h, "mode": mode, "kernel": kern, "qps": round(qps), "search_ms": round(st["search_ms"], 1),
                              "leafscan_ms": round(st["leafscan_ms"], 1), "rounds": st["rounds"],
                              "pairs_per_q": round(st["pairs"] / a.m), "leafscan_tflops": round(tf, 2),
                              "frac_peak": round(tf / peak, 3), "peak": round(peak, 1),
                              "launches": st["kernel_launches"]}), flush=True)
    dev.close()


if __name__ == "__main__":
    main()
