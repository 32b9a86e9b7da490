"""Randomised exactness sweep of the B200 engine against the CPU oracle.

Covers the round engine (split rounds for leaves of >= 2 windows, leaf-level
rounds, home-order renumbering for m >= 65,536) and the general-domain path
(k > 64, d > 32, h > 16).

    python tools/fuzz_parity.py [--cases 200] [--seed 1] [--seconds 600]

Each case draws n, m, d, k, h, a data family (uniform, Gaussian mixture with
tiny or wide spreads, large offsets, per-dimension scales spanning 1e-3..1e3,
integer grids with heavy ties, duplicated points, negative coordinates) and a
kernel (auto / tc / direct, exact mode), runs lazy_search on cuda:0 and
requires bit-identical keys and visited counts.  One JSON line per failure,
a summary line at the end.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1512_02831_b200 as bkt  # noqa: E402
from oracle import oracle as O  # noqa: E402


def draw(rng, n, d):
    fam = rng.choice(["uniform", "mixture_tight", "mixture_wide", "offset", "scales", "grid", "dups", "negative"])
    if fam == "uniform":
        x = rng.random((n, d))
    elif fam == "mixture_tight":
        c = rng.random((4, d))
        x = c[rng.integers(0, 4, n)] + rng.normal(0, 1e-3, (n, d))
    elif fam == "mixture_wide":
        c = rng.random((16, d)) * 10
        x = c[rng.integers(0, 16, n)] + rng.normal(0, 0.5, (n, d))
    elif fam == "offset":
        x = 1e4 + rng.random((n, d))
    elif fam == "scales":
        x = rng.random((n, d)) * (10.0 ** rng.uniform(-3, 3, d))
    elif fam == "grid":
        x = rng.integers(0, 4, (n, d)).astype(np.float64)
    elif fam == "dups":
        base = rng.random((max(1, n // 8), d))
        x = base[rng.integers(0, base.shape[0], n)]
    else:
        x = rng.normal(0, 3, (n, d))
    return fam, x.astype(np.float32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=200)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--seconds", type=float, default=600)
    ap.add_argument("--only", type=int, default=-1, help="replay the generator and run only this case")
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    dev = bkt.device_init(bkt.DeviceSpec(cuda_device=0))
    t0 = time.time()
    done = fails = 0
    for case in range(a.cases):
        if time.time() - t0 > a.seconds:
            break
        d = int(rng.choice([1, 2, 3, 5, 8, 9, 10, 11, 12, 13, 15, 16, 20, 27, 31, 33, 40]))
        n = int(rng.integers(300, 60_000)) if rng.random() < 0.8 else int(rng.integers(60_000, 400_000))
        h = int(rng.integers(1, max(2, min(12, int(np.log2(n)) - 2))))
        if rng.random() < 0.05 and n >= (1 << 18):
            h = int(rng.integers(17, int(np.log2(n))))  # general-domain path: h > 16
        k = int(min(n, rng.choice([1, 2, 5, 10, 16, 33, 50, 64, 65, 100, 200])))
        m = int(rng.integers(1, 6000)) if rng.random() < 0.85 else int(rng.integers(65_536, 150_000))
        fam, pts = draw(rng, n + m, d)
        refs, q = pts[:n], pts[n:]
        if rng.random() < 0.2:  # some queries exactly on reference points
            take = rng.integers(0, n, size=m // 3)
            q[: take.size] = refs[take]
        kernel = str(rng.choice(["auto", "tc", "direct"])) if d <= 31 and k <= 64 and h <= 16 else "auto"
        dev_build = rng.random() < 0.5
        # host-resident structure streamed in chunks (the out-of-core drain)
        chunks = int(rng.integers(2, 10)) if rng.random() < 0.3 else 1
        if a.only >= 0 and case != a.only:
            continue
        print(json.dumps({"running": case, "fam": fam, "n": n, "m": m, "d": d, "k": k, "h": h, "kernel": kernel,
                          "chunks": chunks}),
              file=sys.stderr, flush=True)
        tree = bkt.build_buffer_tree(refs, h, device=0 if dev_build else None)
        st = bkt.SearchStats()
        plan = bkt.ChunkPlan.build(n, chunks) if chunks > 1 else None
        res = bkt.lazy_search(tree, q, bkt.SearchParams(k=k), device=dev, plan=plan, stats=st, kernel=kernel)
        want = O.knn_tree(O.build_tree(refs, h), q, k, threads=8)
        ok = bool(np.array_equal(res.keys, want["keys"])) and bool(
            np.array_equal(st.visited_per_query, want["visited"].astype(np.int64)))
        done += 1
        if not ok:
            fails += 1
            bad = int((res.keys != want["keys"]).any(axis=1).sum())
            if a.only >= 0:
                rows = np.nonzero((res.keys != want["keys"]).any(axis=1))[0]
                for r in rows[:5]:
                    print("row", int(r), "got", bkt.unpack_keys(res.keys[r:r + 1]), "want",
                          bkt.unpack_keys(want["keys"][r:r + 1]), "visited", int(st.visited_per_query[r]),
                          int(want["visited"][r]), file=sys.stderr)
            print(json.dumps({"case": case, "fam": fam, "n": n, "m": m, "d": d, "k": k, "h": h, "kernel": kernel,
                              "chunks": chunks, "rows_differing": bad}), flush=True)
    print(json.dumps({"cases": done, "failures": fails, "seconds": round(time.time() - t0, 1)}), flush=True)
    dev.close()


if __name__ == "__main__":
    main()
