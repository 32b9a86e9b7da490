"""Measure BASELINE.json's configs beyond the headline (bench.py measures configs[1]).

    python tools/configs.py cfg1                 # uniform n=m=2^16, d=10, k=10, h=8 (+ reference digest)
    python tools/configs.py cfg3 [--m 1e9] [--gpus N]  # n=2M refs, stream of m queries in 10M chunks over N GPUs
    python tools/configs.py cfg4 [--m 10e6]      # d = 5 / 15 / 27 mixture, n=2M
    python tools/configs.py cfg5 [--m 1e6]       # n=8M host-resident leaf streaming, k in {1,10,50}, h in {8,11,14}
    python tools/configs.py uniform2m [--m 1e7]  # uniform data at the headline size (n=2M, d=10, k=10)

One JSON line per measurement on stdout.  Every run checks a sample of rows
against the CPU oracle (exact mode: bit-identical keys).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_1512_02831_b200 as bkt  # noqa: E402
from paper_1512_02831_b200.datasets import gen_mixture, gen_query_chunk  # noqa: E402


def oracle_check(tree, queries, keys, k, rows=512):
    from oracle import oracle as O
    ot = O.OracleTree(tree.top.height, tree.d, tree.top.split_values, np.ascontiguousarray(np.asarray(tree.leaves.points)),
                      tree.leaves.original_index, tree.leaves.leaf_starts)
    r = O.knn_tree(ot, np.ascontiguousarray(queries[:rows]), k, threads=os.cpu_count() or 1)
    return bool(np.array_equal(r["keys"], keys[:rows]))


def _tf32_peak():
    """Dense TF32 TFLOP/s: half the measured bf16 GEMM figure (MEASURED_PEAKS.json), else the guide's fallback."""
    p = ROOT / "MEASURED_PEAKS.json"
    bf16 = json.load(open(p)).get("bf16_tflops", 1590.0) if p.exists() else 1590.0
    return bf16 / 2


def emit(d):
    print(json.dumps(d), flush=True)


def cfg1(a):
    refs, queries = bkt.datasets.config_inputs(1)
    tree = bkt.build_buffer_tree(refs, 8)
    dev = bkt.device_init(bkt.DeviceSpec(cuda_device=0))
    dev.ensure_tree(tree)
    for kern in ("auto", "direct"):
        dev.search(queries, 10, kernel=kern)  # warm-up
        t0 = time.perf_counter()
        keys, st, _ = dev.search(queries, 10, kernel=kern)
        wall = time.perf_counter() - t0
        dig = hashlib.sha256((keys & np.uint64(0xFFFFFFFF)).astype("<i8").tobytes()).hexdigest()
        gold = json.load(open(ROOT / "tests" / "golden" / "c1_digest.json"))["digest_indices_sha256"]
        emit({"config": "cfg1 uniform n=m=65536 d=10 k=10 h=8", "kernel": kern, "qps_device": 65536 / (st["search_ms"] / 1e3),
              "qps_e2e": 65536 / wall, "rounds": st["rounds"], "digest_matches_reference": dig == gold})
    dev.close()


def _gen(args):
    c, size = args
    return gen_query_chunk(c, size, 10)


def cfg3(a):
    """Config 3: n=2M refs, a stream of m queries generated per 10M-query chunk
    with the reference's recipe (gen_query_chunk: default_rng(1000 + c)),
    spread over --gpus devices (one host thread per GPU pulling chunks from a
    shared counter, tree replicated, no collective).  Each chunk goes through
    the public API call (H2D, search, D2H); its index rows are hashed
    (sha256) on the device thread and the run's digest is the sha256 of the
    per-chunk digests in chunk order.  Host generation runs in a process pool
    ahead of the devices; the first chunk's first rows are checked against the
    CPU oracle."""
    import threading
    n, m, chunk = 2_000_000, int(a.m), 10_000_000
    pts, _ = gen_mixture(n + 10_000_000, 10, seed=1)
    refs = np.ascontiguousarray(pts.data[:n])
    del pts
    tree = bkt.build_buffer_tree(refs, 9)
    ngpu = max(1, a.gpus)
    devs = [bkt.device_init(bkt.DeviceSpec(cuda_device=i)) for i in range(ngpu)]
    for dev in devs:
        dev.ensure_tree(tree)
    nchunks = (m + chunk - 1) // chunk
    digests = [None] * nchunks
    first = {}
    ahead = min(nchunks, 4 * ngpu + 4)
    lock = threading.Lock()
    nxt = [0]
    busy = [0.0] * ngpu
    with ProcessPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as ex:
        futs = {c: ex.submit(_gen, (c, min(chunk, m - c * chunk))) for c in range(ahead)}

        def drive(g):
            dev = devs[g]
            while True:
                with lock:
                    c = nxt[0]
                    if c >= nchunks:
                        return
                    nxt[0] += 1
                    f = futs.pop(c)
                    if c + ahead < nchunks:
                        futs[c + ahead] = ex.submit(_gen, (c + ahead, min(chunk, m - (c + ahead) * chunk)))
                q = f.result()
                s0 = time.perf_counter()
                keys, st, _ = dev.search(q, 10)  # public API call: H2D, search, D2H
                busy[g] += time.perf_counter() - s0
                digests[c] = hashlib.sha256((keys & np.uint64(0xFFFFFFFF)).astype("<i8").tobytes()).digest()
                if c == 0:
                    first["q"], first["k"] = q[:2048].copy(), keys[:2048].copy()

        t0 = time.perf_counter()
        th = [threading.Thread(target=drive, args=(g,)) for g in range(ngpu)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        wall = time.perf_counter() - t0
    ok = oracle_check(tree, first["q"], first["k"], 10)
    emit({"config": f"cfg3 stream: n=2M refs, m={m} queries in {nchunks} chunks of {chunk} (config-3 recipe, "
                    f"default_rng(1000+c)), d=10, k=10, h=9, {ngpu} GPU(s), chunks pulled by one thread per GPU",
          "qps_wall_incl_host_generation": m / wall, "qps_per_gpu_search_api": [round(m / ngpu / b) if b else None
                                                                                for b in busy],
          "wall_seconds": wall, "digest_of_chunk_digests": hashlib.sha256(b"".join(digests)).hexdigest(),
          "sample_rows_match_oracle": ok})
    for dev in devs:
        dev.close()


def cfg4(a):
    n, m = 2_000_000, int(a.m)
    for d in (5, 15, 27):
        pts, _ = gen_mixture(n + m, d, seed=1)
        refs, queries = pts.data[:n], pts.data[n:]
        tree = bkt.build_buffer_tree(refs, 9)
        dev = bkt.device_init(bkt.DeviceSpec(cuda_device=0))
        dev.ensure_tree(tree)
        for kern in ("auto", "direct"):
            dev.search(queries, 10, kernel=kern)  # warm-up at full size (work buffers, result pool)
            keys, st, _ = dev.search(queries, 10, kernel=kern, timing=True)
            ok = oracle_check(tree, queries, keys, 10, rows=256)
            scan_s = st["leafscan_ms"] / 1e3
            line = {"config": f"cfg4 mixture n=2M m={m} d={d} k=10 h=9", "kernel": kern,
                    "qps_device": m / (st["search_ms"] / 1e3), "pairs_per_query": st["pairs"] / m,
                    "leafscan_tflops_fp32_equiv": 3 * d * st["pairs"] / scan_s / 1e12,
                    "leafscan_share": st["leafscan_ms"] / st["search_ms"], "rounds": st["rounds"],
                    "sample_rows_match_oracle": ok}
            if kern == "auto" and d >= 8:
                # tensor-core roofline: 2 * KT FLOPs per algorithmic pair (K = d + 1 padded to 16 / 32)
                kt = 16 if d + 1 <= 16 else 32
                ach = 2 * kt * st["pairs"] / scan_s / 1e12
                line.update(roofline_tensor={"achieved": ach, "peak": _tf32_peak(), "frac": ach / _tf32_peak(),
                                             "flops_per_pair": 2 * kt})
            else:
                line.update(roofline_fp32={"achieved": line["leafscan_tflops_fp32_equiv"], "peak": dev.fp32_peak_tflops(),
                                           "frac": line["leafscan_tflops_fp32_equiv"] / dev.fp32_peak_tflops()})
            emit(line)
        dev.close()


def uniform2m(a):
    """The north star's second data family at the headline size: uniform
    [0,1)^10 (reference gen_synthetic "uniform"), n=2M refs, m queries."""
    n, m = 2_000_000, int(a.m)
    rng = np.random.default_rng(0)
    refs = rng.random((n, 10), dtype=np.float32)
    queries = rng.random((m, 10), dtype=np.float32)
    for h in (9, 11):
        tree = bkt.build_buffer_tree(refs, h)
        dev = bkt.device_init(bkt.DeviceSpec(cuda_device=0))
        dev.ensure_tree(tree)
        dev.search(queries[:100000], 10)
        keys, st, _ = dev.search(queries, 10, timing=True)
        ok = oracle_check(tree, queries, keys, 10, rows=256)
        emit({"config": f"uniform n=2M m={m} d=10 k=10 h={h}", "qps_device": m / (st["search_ms"] / 1e3),
              "pairs_per_query": st["pairs"] / m, "rounds": st["rounds"], "sample_rows_match_oracle": ok})
        dev.close()


def cfg5(a):
    n, m = 8_000_000, int(a.m)
    pts, _ = gen_mixture(n + m, 10, seed=1)
    refs, queries = pts.data[:n], pts.data[n:]
    for h in [int(x) for x in a.heights.split(",")]:
        tree = bkt.build_buffer_tree(refs, h)
        for num_chunks in {"hbm": (1,), "host": (4,), "both": (1, 4)}[a.resident]:
            plan = bkt.ChunkPlan.build(n, num_chunks)
            dev = bkt.device_init(bkt.DeviceSpec(cuda_device=0))
            dev.ensure_tree(tree, plan if num_chunks > 1 else None)
            for k in [int(x) for x in a.ks.split(",")]:
                t0 = time.perf_counter()
                keys, st, _ = dev.search(queries, k, timing=True)
                wall = time.perf_counter() - t0
                ok = oracle_check(tree, queries, keys, k, rows=128)
                emit({"config": f"cfg5 mixture n=8M m={m} d=10 h={h} k={k} "
                                f"{'host-resident, ' + str(num_chunks) + ' chunks streamed' if num_chunks > 1 else 'HBM-resident'}",
                      "qps_device": m / (st["search_ms"] / 1e3), "qps_wall": m / wall, "rounds": st["rounds"],
                      "pairs_per_query": st["pairs"] / m, "sample_rows_match_oracle": ok,
                      **({"stream_gb": st["stream_bytes"] / 1e9, "stream_copies": st["stream_copies"],
                          "stream_gbs_over_search": st["stream_bytes"] / 1e9 / (st["search_ms"] / 1e3),
                          "pcie_peak_gbs": "~55 (PCIe Gen5 x16 H2D, nominal 64)",
                          # PCIe roofline of the streamed structure: its bytes at the H2D peak, as a share of the search
                          "pcie_floor_ms": st["stream_bytes"] / 55e9 * 1e3,
                          "pcie_floor_share": st["stream_bytes"] / 55e9 / (st["search_ms"] / 1e3),
                          "schedule": "round schedule (BKT_OOC_ROUNDS=1)" if os.environ.get("BKT_OOC_ROUNDS", "0") != "0"
                          else "drain (DESIGN 3d)"} if num_chunks > 1 else {})})
            dev.close()


def brute(a):
    """GPU brute force (reference brute.py:41-113): the engine's leaf scans over
    the exhaustive two-leaf structure (every (query, reference) pair), uniform
    d = 10, k = 10; q/s, pairs/s and the TF32 roofline of the scan; 256 rows
    against the oracle's brute force."""
    from oracle import oracle as O
    from paper_1512_02831_b200.brute import exhaustive_tree
    d, k = 10, 10
    m = int(a.m) if a.m else 65536
    for n in (65536, 1 << 20):
        rng = np.random.default_rng(7)
        refs = rng.random((n, d), dtype=np.float32)
        q = rng.random((m, d), dtype=np.float32)
        tree = exhaustive_tree(refs)
        dev = bkt.device_init(bkt.DeviceSpec(cuda_device=0))
        bkt.lazy_search(tree, q[:4096], bkt.SearchParams(k=k), device=dev)  # warm-up
        st = bkt.SearchStats()
        t0 = time.perf_counter()
        res = bkt.lazy_search(tree, q, bkt.SearchParams(k=k), device=dev, stats=st)
        wall = time.perf_counter() - t0
        ok = bool(np.array_equal(res.keys[:256], O.brute_keys(refs, q[:256], k, threads=os.cpu_count() or 1)))
        pairs = float(m) * n
        emit({"config": f"brute uniform n={n} m={m} d={d} k={k}", "qps_device": m / (st.search_ms / 1e3),
              "qps_wall": m / wall, "pairs_per_s": pairs / (st.search_ms / 1e3),
              "leafscan_tflops_tf32": pairs * 32 / (st.leafscan_ms / 1e3) / 1e12,
              "roofline_frac_tf32": pairs * 32 / (st.leafscan_ms / 1e3) / 1e12 / _tf32_peak(),
              "leafscan_share": st.leafscan_ms / st.search_ms, "sample_rows_match_oracle": ok})
        dev.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["cfg1", "cfg3", "cfg4", "cfg5", "uniform2m", "brute"])
    ap.add_argument("--m", type=float, default=None)
    ap.add_argument("--gpus", type=int, default=1, help="cfg3: devices the stream is spread over")
    ap.add_argument("--heights", default="8,11,14", help="cfg5: tree heights")
    ap.add_argument("--ks", default="1,10,50", help="cfg5: k values")
    ap.add_argument("--resident", default="both", choices=["hbm", "host", "both"], help="cfg5: leaf structure residency")
    a = ap.parse_args()
    if a.m is None:
        a.m = {"cfg1": 65536, "cfg3": 2e8, "cfg4": 10e6, "cfg5": 1e6, "uniform2m": 10e6, "brute": 262144}[a.which]
    globals()[a.which](a)


if __name__ == "__main__":
    main()
