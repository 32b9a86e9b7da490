"""Benchmark: k-NN queries/sec (k=10, d=10, n=2M) on 1..8 B200 + % of FP32 roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--mode fma|exact] [--height H]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N
    python bench.py --impl reference ...     # the reference CPU path (oracle port) on host cores

Workload (BASELINE.json configs[1], "astronomy-like synthetic n=2M refs, m=10M
queries, d=10, k=10, single B200 in-memory"): gen_mixture(n+m, 10, seed=1)
drawn jointly, refs = first 2M rows, queries = the other 10M.  With N GPUs
(one process per GPU, torchrun) the tree is replicated and queries shard with
no data-path collective:
  --scaling weak (default): every rank searches its own 10M queries; rank 0
      the config-2 queries, rank r>0 config 3's per-chunk recipe with chunk r;
  --scaling strong: the config-2 10M queries split with shard_range.
The tree is built once before timing.  One step = one search over the rank's
queries.  Every rank checks --check-rows of its rows against the CPU oracle.

value: queries/sec of the whole job, inputs resident in HBM, device time of
the search (CUDA events on the engine's stream), max over ranks.
e2e:   the same through the public API (lazy_search on host numpy arrays):
H2D of the queries and D2H of the (m, k) keys inside the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_REFS = 2_000_000
M_QUERIES = 10_000_000
DIM = 10
K = 10
METRIC = "kNN queries/sec (k=10,d=10,n=2M) at 1/2/4/8 B200; % FP32/HBM roofline"
UNIT = "queries/s"


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--mode", default="exact", choices=["fma", "exact"],
                    help="exact: bit-identical to the reference (default); fma: fused multiply-add distances")
    ap.add_argument("--kernel", default="auto", choices=["auto", "direct", "tc"],
                    help="leaf scan: tensor-core filter (auto/tc) or CUDA-core direct scan")
    ap.add_argument("--height", type=int, default=9, help="tree height (results do not depend on it)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every rank searches its own m queries; strong: m queries sharded over the ranks")
    ap.add_argument("--m", type=int, default=M_QUERIES)
    ap.add_argument("--n", type=int, default=N_REFS)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0, help="queries in the CPU baseline sample (0 = auto)")
    ap.add_argument("--check-rows", type=int, default=1000,
                    help="rows of every rank's result checked against the CPU oracle (0 = off)")
    return ap.parse_args(argv)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def shard_range(m: int, rank: int, world: int) -> tuple[int, int]:
    """Even split, remainder to the front ranks (reference scheduler.py:172-183).
    Same rule as paper_1512_02831_b200.dist.shard_range; restated here so the
    reference arm never imports the product package."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("rank must be in [0, world)")
    base, rem = divmod(m, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def mixture_rows(n: int, m: int, lo: int, hi: int, d: int = DIM, seed: int = 1):
    """refs = rows [0, n) and queries = rows [n+lo, n+hi) of the reference's
    gen_mixture(n+m, d, components=8, spread=0.05, seed) (datasets.py:127-136),
    drawn jointly as the reference does but only up to row n+hi: the normal
    stream is consumed in order, so rows drawn in pieces equal the joint draw."""
    rng = np.random.default_rng(seed)
    centers = rng.random((8, d))
    labels = rng.integers(0, 8, size=n + m)
    refs = (centers[labels[:n]] + rng.normal(0.0, 0.05, size=(n, d))).astype(np.float32)
    skip = lo
    while skip > 0:  # rows before the shard: drawn and dropped, 1M at a time
        t = min(skip, 1 << 20)
        rng.normal(0.0, 0.05, size=(t, d))
        skip -= t
    q = (centers[labels[n + lo:n + hi]] + rng.normal(0.0, 0.05, size=(hi - lo, d))).astype(np.float32)
    return np.ascontiguousarray(refs), np.ascontiguousarray(q)


def query_chunk(chunk: int, size: int, d: int = DIM, seed: int = 1) -> np.ndarray:
    """Config 3's per-chunk query recipe: the config-2 mixture
    centres with default_rng(1000 + chunk)."""
    centers = np.random.default_rng(seed).random((8, d))
    r = np.random.default_rng(1000 + chunk)
    return (centers[r.integers(0, 8, size=size)] + r.normal(0.0, 0.05, (size, d))).astype(np.float32)


def rank_work(scaling: str, rank: int, world: int, n: int, m: int) -> dict:
    """Which queries a rank searches.  weak: rank 0 the config-2 queries, rank
    r > 0 config 3's query chunk r (m each); strong: rows shard_range(m) of
    the config-2 queries."""
    if scaling == "strong":
        lo, hi = shard_range(m, rank, world)
        return {"kind": "cfg2", "lo": lo, "hi": hi, "total": m}
    if rank == 0:
        return {"kind": "cfg2", "lo": 0, "hi": m, "total": m * world}
    return {"kind": "chunk", "chunk": rank, "size": m, "total": m * world}


def workload(w: dict, n: int, m: int):
    if w["kind"] == "cfg2":
        return mixture_rows(n, m, w["lo"], w["hi"])
    refs, _ = mixture_rows(n, m, 0, 0)
    return refs, np.ascontiguousarray(query_chunk(w["chunk"], w["size"]))


def job_value(total_queries: int, steps: int, rank_seconds: list[float]) -> float:
    """Whole-job throughput: every query all ranks searched / the slowest rank's time."""
    return steps * total_queries / max(rank_seconds)


def reduce_ranks(dev_ms: float, e2e_s: float | None, parity_ok: bool | None, device=None) -> dict:
    """The only cross-rank traffic of a bench run: the slowest rank's device
    and end-to-end times (max over ranks) and the AND of the per-rank parity
    checks.  Every rank calls it in the same order (collectives)."""
    from paper_1512_02831_b200.dist import max_over_ranks
    out = {"dev_ms_max": max_over_ranks(dev_ms, device=device)}
    if e2e_s is not None:
        out["e2e_s_max"] = max_over_ranks(e2e_s, device=device)
    if parity_ok is not None:
        out["parity_all"] = -max_over_ranks(-float(parity_ok), device=device) >= 1.0
    return out


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows: list[list[str]] = []
        self._proc = None

    def start(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except FileNotFoundError:
            self._proc = None

    def _read(self):
        for line in self._proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self) -> dict:
        if self._proc is not None:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except Exception:
                self._proc.kill()
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) < 8:
                continue
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        loaded = [s for s in sm if s > 300] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons), "samples": len(self.rows)}


def oracle_tree_of(tree):
    """The CPU oracle's view of a built tree (checker input; no product code runs)."""
    from oracle import oracle as O
    return O.OracleTree(tree.top.height, tree.d, tree.top.split_values,
                        np.ascontiguousarray(np.asarray(tree.leaves.points)), tree.leaves.original_index,
                        tree.leaves.leaf_starts)


def cpu_baseline(otree, queries, sample: int, threads: int, label: str) -> dict:
    """The reference CPU path restated in C (oracle/, kind "port"): classic
    per-query traversal with the reference pruning rule == lazy_search's
    per-query leaf order, float32 two roundings per dimension."""
    from oracle import oracle as O
    q = np.ascontiguousarray(queries[:sample])
    t0 = time.perf_counter()
    r = O.knn_tree(otree, q, K, threads=threads)
    secs = time.perf_counter() - t0
    return {"value": sample / secs, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{sample} {label} (h={otree.h}), C restatement of the reference traversal, "
                      f"{threads} threads, {secs:.1f}s",
            "keys": r["keys"], "seconds": secs}


def check_rows(otree, queries, got_keys, rows: int, threads: int, exact: bool) -> bool:
    """Parity of a sample of one rank's result rows against the CPU oracle:
    exact mode bit-identical keys; fma mode distances within 1e-5 relative."""
    from oracle import oracle as O
    rows = min(rows, queries.shape[0])
    if rows <= 0:
        return True
    want = O.knn_tree(otree, np.ascontiguousarray(queries[:rows]), K, threads=threads)["keys"]
    got = np.asarray(got_keys[:rows]).view(np.uint64)
    if exact:
        return bool(np.array_equal(got, want))
    gd = (got >> np.uint64(32)).astype(np.uint32).view(np.float32).astype(np.float64)
    wd = (want >> np.uint64(32)).astype(np.uint32).view(np.float32).astype(np.float64)
    return bool(np.all(np.abs(gd - wd) <= 1e-5 * np.maximum(wd, 1e-30)))


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference_arm(a) -> None:
    """The reference's CPU path on the box's host cores: the oracle's C
    restatement of the reference build (buffer_tree.py:149-197) and traversal
    (kdtree.py:157-204 == lazy_search's per-query order), all host threads.
    Nothing from paper_1512_02831_b200 is imported or loaded here.  Each step
    times a bounded sample of the config-2 queries (the whole 10M would take
    ~10 min per step), so the line's workload is a sample of the B200 arm's."""
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    O.build()
    threads = os.cpu_count() or 1
    h = a.height
    sample = a.cpu_sample or max(2000, 1500 * threads)
    nsteps = a.warmup + a.steps
    rows = min(a.m, sample * nsteps)
    refs, queries = mixture_rows(a.n, a.m, 0, rows)
    t0 = time.perf_counter()
    otree = O.build_tree(refs, h)
    build_s = time.perf_counter() - t0
    vals = []
    for step in range(nsteps):
        lo = (step * sample) % max(1, rows - sample + 1)
        r = cpu_baseline(otree, queries[lo:], sample, threads, "config-2 queries per step")
        if step >= a.warmup:
            vals.append(r["value"])
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * sample / v, "higher_is_better": True,
            "scaling": a.scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"cfg2 mixture n={a.n} refs, d={DIM}, k={K}, h={h}; bounded sample of "
                                   f"{sample} queries per step (same_config: a sample of the B200 arm's "
                                   f"{a.m} queries, by design: the full set takes minutes per step on the CPU)",
                       "model": "bufferkdtree-cpu-port", "build_seconds": build_s},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{sample} queries/step of the config-2 queries, C port of the reference "
                                       f"build and traversal (oracle/bkt_oracle.c), {threads} threads ({cpu_model()})"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main() -> None:
    a = parse()
    if a.impl == "reference":
        run_reference_arm(a)
        return
    world, rank, local = dist_env()
    import torch
    import torch.distributed as dist
    # one process per GPU; on a box with fewer GPUs than ranks (smoke-testing the
    # multi-rank flow) ranks share devices round-robin
    ngpu = max(1, torch.cuda.device_count())
    local = local % ngpu
    torch.cuda.set_device(local)
    shared = world > ngpu  # NCCL refuses two ranks on one GPU: use gloo for the control collectives
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev_t = torch.device("cuda", local)
    red_t = torch.device("cpu") if shared else dev_t

    import paper_1512_02831_b200 as bkt
    w = rank_work(a.scaling, rank, world, a.n, a.m)
    refs, queries = workload(w, a.n, a.m)
    m = queries.shape[0]
    h = a.height
    t0 = time.perf_counter()
    tree = bkt.build_buffer_tree(refs, h)
    build_s = time.perf_counter() - t0
    gpu = bkt.device_init(bkt.DeviceSpec(cuda_device=local))
    t0 = time.perf_counter()
    gpu.ensure_tree(tree)
    load_s = time.perf_counter() - t0
    exact = a.mode == "exact"
    peak_measured = gpu.fp32_peak_tflops()
    info = gpu.info()

    q_dev = torch.from_numpy(queries).to(dev_t)
    # e2e inputs live in page-locked host memory (the contract's "pinned host
    # memory"): filled once here, outside every timed region
    from paper_1512_02831_b200 import _native
    queries_h = _native.pinned_empty(queries.shape, np.float32)
    queries_h[...] = queries
    keys_dev = torch.empty((max(m, 1), K), dtype=torch.int64, device=dev_t)
    flush = torch.empty(256 * 2 ** 20 // 4, dtype=torch.float32, device=dev_t)

    def barrier():
        if world > 1:
            dist.barrier()

    def step_device():
        flush.fill_(1.0)  # L2 flush (256 MiB > 126 MB L2)
        torch.cuda.synchronize()
        barrier()
        w0 = time.perf_counter()
        st = gpu.search_device(q_dev.data_ptr(), m, K, keys_dev.data_ptr(), exact=exact, timing=True,
                               kernel=a.kernel)
        torch.cuda.synchronize()
        w1 = time.perf_counter()
        barrier()
        return st, w1 - w0

    for _ in range(a.warmup):
        step_device()
    clocks = ClockSampler(local)
    clocks.start()
    sts, walls = [], []
    for _ in range(a.steps):
        st, wt = step_device()
        sts.append(st)
        walls.append(wt)
    clk = clocks.stop()

    dev_ms = sum(s["search_ms"] for s in sts)
    scan_ms = sum(s["leafscan_ms"] for s in sts)
    pairs = sum(s["pairs"] for s in sts)
    scan_launches = sum(s["leafscan_launches"] for s in sts)
    launches = sum(s["kernel_launches"] for s in sts)
    rounds = sts[-1]["rounds"]
    wall_ms = 1e3 * sum(walls)

    # e2e through the public API with host buffers
    e2e = None
    if not a.no_e2e:
        e2e_steps = max(1, min(a.steps, 3))
        # warm-up calls: the same W as the device loop (at least 2, so that the
        # page-locked result pool holds the buffers a result and its successor need)
        e2e_warm = max(2, a.warmup)
        tot = 0.0
        for i in range(e2e_warm + e2e_steps):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            barrier()
            w0 = time.perf_counter()
            res = bkt.lazy_search(tree, queries_h, bkt.SearchParams(k=K), device=gpu, exact=exact, kernel=a.kernel)
            w1 = time.perf_counter()
            barrier()
            if i >= e2e_warm:
                tot += w1 - w0
            if os.environ.get("BKT_BENCH_DEBUG"):
                print(f"e2e call {i}: {1e3 * (w1 - w0):.1f} ms", file=sys.stderr, flush=True)
        # device and host paths must agree
        if not np.array_equal(res.keys, keys_dev[:m].cpu().numpy().view(np.uint64)):
            raise RuntimeError("device-resident and host API results differ")
        e2e = {"steps": e2e_steps, "seconds": tot}

    # every rank checks a sample of its own rows against the CPU oracle
    threads = os.cpu_count() or 1
    otree = None
    ok = None
    if a.check_rows > 0:
        otree = oracle_tree_of(tree)
        ok = check_rows(otree, queries, keys_dev[:m].cpu().numpy(), a.check_rows,
                        max(1, threads // max(1, world)), exact)

    # reductions across ranks: the slowest rank's device / e2e time, parity AND
    red = reduce_ranks(dev_ms, e2e["seconds"] if e2e else None, ok, device=red_t)
    dev_ms_max = red["dev_ms_max"]
    value = job_value(w["total"], a.steps, [dev_ms_max / 1e3])
    if e2e is not None:
        e2e = {"value": job_value(w["total"], e2e["steps"], [red["e2e_s_max"]]), "unit": UNIT,
               "inputs": "queries in page-locked host memory (bkt_host_alloc), keys returned into host arrays",
               "h2d_bytes_per_step": int(m * DIM * 4), "d2h_bytes_per_step": int(m * K * 8)}
    parity = None
    if ok is not None:
        parity = {"rows_per_rank": min(a.check_rows, m), "ranks": world, "all_match": bool(red["parity_all"]),
                  "rule": "exact: bit-identical keys" if exact else "fma: distances within 1e-5 relative"}

    # Roofline of the dominant kernel (the leaf scan).  It runs on the tensor
    # cores: per (query, reference point) pair the TF32 MMA does 2*KT = 32 FLOPs
    # (K = 16 = d + 1 padded), so `roofline` is TF32 FLOP/s over the TF32 dense
    # peak (half the bf16 GEMM figure of MEASURED_PEAKS.json, else of the
    # profiling guide's fallback).  `roofline_fp32_equiv` restates the same time
    # in the reference's CUDA-core arithmetic (3d FLOPs per pair) against the
    # measured FFMA peak: above 1 because the work is not on the FP32 pipe.
    peaks = json.load(open(ROOT / "MEASURED_PEAKS.json")) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    bf16 = peaks.get("bf16_tflops", 1590.0)
    tf32_peak = bf16 / 2
    peak_src = "of measured (MEASURED_PEAKS.json bf16 / 2)" if peaks else "of fallback (1.59 PF bf16 / 2, B200_PROFILING.md)"
    tc_used = a.kernel in ("auto", "tc") and DIM <= 31
    # the leaf scans of a step: the home visit (leafscan_tc_kernel, one launch)
    # and the later visits as (leaf, window) items (splitscan_tc_kernel, one
    # launch per round); `achieved` counts the algorithmic pairs of both
    kernel_name = ("splitscan_tc_kernel + leafscan_tc_kernel (home round)" if tc_used else "leafscan_kernel")
    traffic = None
    tfs = sorted(ROOT.glob("profiles/r*/ncu_traffic.json"))  # the latest round's capture
    tf = tfs[-1] if tfs else None
    if tf is not None and tc_used and scan_launches:
        t = json.load(open(tf))
        # dram bytes of the captured launch per pair, times this run's mean pairs per launch
        traffic = t["dram_bytes_per_pair"] * pairs / scan_launches
    if tc_used:
        ach = 2.0 * 16 * pairs / (scan_ms / 1e3) / 1e12 if scan_ms > 0 else None
        roofline = {"bound": "tensor", "achieved": ach, "peak": tf32_peak, "unit": "TFLOP/s",
                    "frac": (ach / tf32_peak) if ach else None, "traffic": traffic,
                    "traffic_unit": f"bytes per launch (ncu dram read+write, {tf.relative_to(ROOT) if tf else None})",
                    "kernel": kernel_name, "peak_source": peak_src, "flops_per_pair": 32,
                    "leafscan_ms_per_step": scan_ms / a.steps,
                    "leafscan_share": scan_ms / dev_ms if dev_ms else None, "leafscan_launches": scan_launches}
    else:
        ach = 3.0 * DIM * pairs / (scan_ms / 1e3) / 1e12 if scan_ms > 0 else None
        roofline = {"bound": "fp32", "achieved": ach, "peak": peak_measured, "unit": "TFLOP/s",
                    "frac": (ach / peak_measured) if ach else None, "traffic": None, "kernel": kernel_name,
                    "peak_source": "measured FFMA probe (bkt_fp32_peak)", "flops_per_pair": 3 * DIM,
                    "leafscan_ms_per_step": scan_ms / a.steps,
                    "leafscan_share": scan_ms / dev_ms if dev_ms else None, "leafscan_launches": scan_launches}
    fp32_ach = 3.0 * DIM * pairs / (scan_ms / 1e3) / 1e12 if scan_ms > 0 else None
    nominal = info["sm_count"] * 128 * 2 * 1965e6 / 1e12
    roofline_fp32 = {"bound": "fp32", "achieved": fp32_ach, "peak": peak_measured, "unit": "TFLOP/s",
                     "frac": (fp32_ach / peak_measured) if fp32_ach else None, "flops_per_pair": 3 * DIM,
                     "peak_source": f"measured FFMA probe (bkt_fp32_peak); nominal {nominal:.1f} at 1965 MHz"}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        sample = a.cpu_sample or max(2000, 1500 * threads)
        if otree is None:
            otree = oracle_tree_of(tree)
        cb = cpu_baseline(otree, queries, sample, threads, "first rank-0 config-2 queries")
        got = keys_dev[:sample].cpu().numpy().view(np.uint64)
        if exact:
            match = bool(np.array_equal(got, cb["keys"]))
        else:
            gd, gi = bkt.unpack_keys(got)
            wd, wi = bkt.unpack_keys(cb["keys"])
            match = bool(np.all(np.abs(gd.astype(np.float64) - wd) <= 1e-5 * np.maximum(wd, 1e-30)))
        cpu = {k_: v_ for k_, v_ in cb.items() if k_ not in ("keys", "seconds")}
        cpu["sample"] += f" ({cpu_model()}); GPU rows match: {match}"

    if rank == 0:
        per_gpu = f"{m} queries per GPU" if a.scaling == "weak" else f"{a.m} queries sharded over {world} GPU(s)"
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": dev_ms_max / a.steps, "higher_is_better": True,
            "scaling": a.scaling, "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference gen_mixture recipe, seed 1; 8 gaussians, spread 0.05)",
            "config": {"workload": f"cfg2: mixture n={a.n} refs, {per_gpu}, d={DIM}, k={K}, "
                                   + ("ranks sharing GPUs (smoke test), " if shared else "")
                                   + "in-memory", "height": h, "mode": a.mode, "kernel": a.kernel,
                       "parallelism": f"query-sharded x{world} (tree replicated, no collective)",
                       "l2": "256 MiB write between steps; per-step inputs (1.2 GB) > L2",
                       "rounds": rounds, "pairs_per_query": pairs / (a.steps * max(m, 1)),
                       "build_seconds": build_s, "load_tree_seconds": load_s,
                       "wall_ms_per_step": wall_ms / a.steps},
            "e2e": e2e,
            "gpu_launches": launches,
            "roofline": roofline,
            "roofline_fp32_equiv": roofline_fp32,
            "cpu_baseline": cpu,
            "parity": parity,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    gpu.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
