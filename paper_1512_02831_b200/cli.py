"""Command-line front end on the B200 engine (reference cli.py:105-177).

    python -m paper_1512_02831_b200.cli build    --refs R [--height H] [--out tree.npz]
    python -m paper_1512_02831_b200.cli query    --refs R --queries Q --k 10 [--engine bufferkdtree|brute]
    python -m paper_1512_02831_b200.cli outliers --data D --k 10 [--top 10] [--out ranking.csv]

R / Q / D are BKNN binary or CSV point sets (datasets.py, reference
datasets.py:30-111).  The engine flags and outputs mirror the reference's
subcommands: `query` prints the result digest (bench.py:53-57) and saves
indices / squared distances; `outliers` ranks points by their k-th
neighbour distance over the self-excluded all-NN search.  The reference's
`bench` subcommand drives its engine zoo and simulated devices; here
`bench.py` at the repository root measures the B200 engine.
"""
from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

from .buffer_tree import build_buffer_tree, validate_structure
from .core import SearchParams
from .datasets import load_dataset
from .engine import ENGINES, auto_height, result_digest, run_engine
from .outliers import gpu_engine, outlier_scores, rank_outliers, self_excluded_knn


def _write_report(path, info: dict) -> None:
    if path is not None:
        with open(path, "w") as f:
            json.dump(info, f, indent=1, default=float)


def _add_engine_flags(p: argparse.ArgumentParser) -> None:
    p.add_argument("--k", type=int, default=10, help="neighbours per query")
    p.add_argument("--engine", choices=ENGINES, default="bufferkdtree")
    p.add_argument("--height", type=int, default=None, help="tree height (default: auto_height(n))")
    p.add_argument("--num-chunks", type=int, default=None,
                   help="> 1: leaf structure host-resident, streamed in this many chunks")
    p.add_argument("--devices", type=int, default=1, help="GPUs the queries are sharded over")
    p.add_argument("--fma", action="store_true", help="FMA distance accumulation (default: exact)")
    p.add_argument("--report-out", default=None, help="metrics JSON path")


def _engine_kwargs(args) -> dict:
    return {"height": args.height, "num_chunks": args.num_chunks, "devices": args.devices, "exact": not args.fma}


def _cmd_build(args) -> int:
    refs = load_dataset(args.refs)
    h = args.height if args.height is not None else auto_height(refs.n)
    t0 = time.perf_counter()
    tree = build_buffer_tree(refs, h, device=0 if args.on_gpu else None)
    secs = time.perf_counter() - t0
    validate_structure(tree)
    print(f"built height-{h} tree over {tree.n} x {tree.d} points: "
          f"{tree.n_leaves} leaves, {secs:.3f}s, structure audit passed")
    if args.out is not None:
        np.savez(args.out, points=np.asarray(tree.leaves.points), original_index=tree.leaves.original_index,
                 leaf_starts=tree.leaves.leaf_starts, split_values=tree.top.split_values,
                 levels=tree.top.levels, height=np.int64(h))
        print(f"saved tree arrays to {args.out}")
    _write_report(args.report_out, {"n": tree.n, "d": tree.d, "height": h, "n_leaves": tree.n_leaves,
                                    "build_seconds": secs})
    return 0


def _cmd_query(args) -> int:
    refs = load_dataset(args.refs)
    queries = load_dataset(args.queries)
    res, info = run_engine(args.engine, refs, queries.data, SearchParams(k=args.k), collect_stats=True,
                           **_engine_kwargs(args))
    info["digest"] = result_digest(res)
    if args.out is not None:
        np.savez(args.out, indices=res.indices, sq_dists=res.sq_dists)
        print(f"saved neighbours to {args.out}")
    print(f"{args.engine}: {queries.n} queries x k={args.k} in {info['query_seconds']:.3f}s, "
          f"digest {info['digest'][:16]}")
    _write_report(args.report_out, info)
    return 0


def _cmd_outliers(args) -> int:
    pts = load_dataset(args.data)
    t0 = time.perf_counter()
    _, sq = self_excluded_knn(pts, args.k, gpu_engine(height=args.height, exact=not args.fma))
    scores = outlier_scores(sq)
    order = rank_outliers(scores)
    secs = time.perf_counter() - t0
    top = order[:args.top]
    print(f"scored {pts.n} points on the B200 engine (k={args.k}) in {secs:.3f}s")
    print("rank\tindex\tscore")
    for r, i in enumerate(top, start=1):
        print(f"{r}\t{i}\t{scores[i]:.6f}")
    if args.out is not None:
        with open(args.out, "w") as f:
            f.write("rank,index,score\n")
            for r, i in enumerate(order, start=1):
                f.write(f"{r},{i},{scores[i]:.9g}\n")
        print(f"saved full ranking to {args.out}")
    _write_report(args.report_out, {"n": pts.n, "k": args.k, "seconds": secs,
                                    "top": [[int(i), float(scores[i])] for i in top]})
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_1512_02831_b200.cli", description=__doc__.split("\n\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("build", help="build a tree and audit it")
    b.add_argument("--refs", required=True)
    b.add_argument("--height", type=int, default=None)
    b.add_argument("--on-gpu", action="store_true", help="median splits on the GPU (bkt_build_tree_device)")
    b.add_argument("--out", default=None, help="npz of the tree arrays")
    b.add_argument("--report-out", default=None)
    b.set_defaults(fn=_cmd_build)
    q = sub.add_parser("query", help="k-NN of a query set")
    q.add_argument("--refs", required=True)
    q.add_argument("--queries", required=True)
    q.add_argument("--out", default=None, help="npz of indices and squared distances")
    _add_engine_flags(q)
    q.set_defaults(fn=_cmd_query)
    o = sub.add_parser("outliers", help="rank points by their k-th neighbour distance")
    o.add_argument("--data", required=True)
    o.add_argument("--k", type=int, default=10)
    o.add_argument("--height", type=int, default=None)
    o.add_argument("--top", type=int, default=10)
    o.add_argument("--fma", action="store_true")
    o.add_argument("--out", default=None, help="CSV of the full ranking")
    o.add_argument("--report-out", default=None)
    o.set_defaults(fn=_cmd_outliers)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    return args.fn(args)


if __name__ == "__main__":
    sys.exit(main())
