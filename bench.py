"""Benchmark: k-NN queries/sec (k=10, d=10, n=2M) on 1..8 B200 + % of FP32 roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--mode fma|exact] [--height H]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N
    python bench.py --impl reference ...     # the reference CPU path (oracle port) on host cores

Workload (BASELINE.json configs[1], "astronomy-like synthetic n=2M refs, m=10M
queries, d=10, k=10, single B200 in-memory"): gen_mixture(n+m, 10, seed=1)
drawn jointly, refs = first 2M rows, queries = the other 10M (rank 0).  With
N GPUs each rank searches its own 10M queries (weak scaling): rank r>0 uses
config 3's per-chunk query recipe with chunk r.  The tree (replicated per
GPU) is built once before timing.  One step = one lazy_search over the
rank's 10M queries.

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


def parse():
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
    ap.add_argument("--m", type=int, default=M_QUERIES)
    ap.add_argument("--n", type=int, default=N_REFS)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=0, help="queries in the CPU baseline sample (0 = auto)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload(rank: int, n: int, m: int):
    from paper_1512_02831_b200.datasets import gen_mixture, gen_query_chunk
    pts, _ = gen_mixture(n + m, DIM, components=8, spread=0.05, seed=1)
    refs = pts.data[:n]
    if rank == 0:
        queries = pts.data[n:]
    else:
        queries = gen_query_chunk(rank, m, DIM)
    return np.ascontiguousarray(refs), np.ascontiguousarray(queries)


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


def cpu_baseline(tree, queries, sample: int, threads: int) -> dict:
    """The reference CPU path restated in C (oracle/, kind "port"): classic
    per-query traversal with the reference pruning rule == lazy_search's
    per-query leaf order, float32 two roundings per dimension."""
    from oracle import oracle as O
    ot = O.OracleTree(tree.top.height, tree.d, tree.top.split_values,
                      np.ascontiguousarray(np.asarray(tree.leaves.points)), tree.leaves.original_index,
                      tree.leaves.leaf_starts)
    q = np.ascontiguousarray(queries[:sample])
    t0 = time.perf_counter()
    r = O.knn_tree(ot, q, K, threads=threads)
    secs = time.perf_counter() - t0
    return {"value": sample / secs, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"first {sample} of the rank-0 config-2 queries (h={tree.top.height}), "
                      f"C restatement of the reference traversal, {threads} threads, {secs:.1f}s",
            "keys": r["keys"], "seconds": secs}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference_arm(a) -> None:
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import paper_1512_02831_b200 as bkt
    from oracle import oracle as O
    O.build()
    threads = os.cpu_count() or 1
    refs, queries = workload(0, a.n, a.m)
    h = a.height
    tree = bkt.build_buffer_tree(refs, h)
    sample = a.cpu_sample or max(2000, 1500 * threads)
    vals = []
    for step in range(a.warmup + a.steps):
        lo = (step * sample) % max(1, queries.shape[0] - sample)
        r = cpu_baseline(tree, queries[lo:], sample, threads)
        if step >= a.warmup:
            vals.append(r["value"])
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": 1e3 * sample / v, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"cfg2 mixture n={a.n} refs, d={DIM}, k={K}, h={h}; bounded sample of "
                                   f"{sample} queries per step", "model": "bufferkdtree-cpu-port"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{sample} queries/step of the config-2 queries, C port of the reference "
                                       f"traversal, {threads} threads ({cpu_model()})"},
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
    refs, queries = workload(rank, a.n, a.m)
    m = queries.shape[0]
    h = a.height
    t0 = time.perf_counter()
    tree = bkt.build_buffer_tree(refs, h)
    build_s = time.perf_counter() - t0
    gpu = bkt.device_init(bkt.DeviceSpec(cuda_device=local))
    gpu.ensure_tree(tree)
    exact = a.mode == "exact"
    peak_measured = gpu.fp32_peak_tflops()
    info = gpu.info()

    q_dev = torch.from_numpy(queries).to(dev_t)
    keys_dev = torch.empty((m, K), dtype=torch.int64, device=dev_t)
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
        st, w = step_device()
        sts.append(st)
        walls.append(w)
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
            res = bkt.lazy_search(tree, queries, bkt.SearchParams(k=K), device=gpu, exact=exact, kernel=a.kernel)
            w1 = time.perf_counter()
            barrier()
            if i >= e2e_warm:
                tot += w1 - w0
            if os.environ.get("BKT_BENCH_DEBUG"):
                print(f"e2e call {i}: {1e3 * (w1 - w0):.1f} ms", file=sys.stderr, flush=True)
        e2e_local = e2e_steps * m / tot
        e2e = {"value": e2e_local, "unit": UNIT, "h2d_bytes_per_step": int(m * DIM * 4),
               "d2h_bytes_per_step": int(m * K * 8)}
        # device and host paths must agree
        if not np.array_equal(res.keys, keys_dev.cpu().numpy().view(np.uint64)):
            raise RuntimeError("device-resident and host API results differ")

    # reductions across ranks: max time, sum of queries
    def allmax(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_t)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    dev_ms_max = allmax(dev_ms)
    if e2e is not None:
        e2e_time_max = allmax(e2e_steps * m / e2e["value"])
        e2e["value"] = world * e2e_steps * m / e2e_time_max
    value = world * a.steps * m / (dev_ms_max / 1e3)

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
    kernel_name = "leafscan_tc_kernel" if tc_used else "leafscan_kernel"
    traffic = None
    tf = ROOT / "profiles" / "r1f" / "ncu_traffic.json"
    if tf.exists() and tc_used and scan_launches:
        t = json.load(open(tf))
        # dram bytes of the captured launch per pair, times this run's mean pairs per launch
        traffic = t["dram_bytes_per_pair"] * pairs / scan_launches
    if tc_used:
        ach = 2.0 * 16 * pairs / (scan_ms / 1e3) / 1e12 if scan_ms > 0 else None
        roofline = {"bound": "tensor", "achieved": ach, "peak": tf32_peak, "unit": "TFLOP/s",
                    "frac": (ach / tf32_peak) if ach else None, "traffic": traffic,
                    "traffic_unit": "bytes per launch (ncu dram read+write, profiles/r1f/ncu_traffic.json)",
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
        threads = os.cpu_count() or 1
        sample = a.cpu_sample or max(2000, 1500 * threads)
        cb = cpu_baseline(tree, queries, sample, threads)
        got = keys_dev[:sample].cpu().numpy().view(np.uint64)
        if exact:
            parity = bool(np.array_equal(got, cb["keys"]))
        else:
            gd, gi = bkt.unpack_keys(got)
            wd, wi = bkt.unpack_keys(cb["keys"])
            parity = bool(np.all(np.abs(gd.astype(np.float64) - wd) <= 1e-5 * np.maximum(wd, 1e-30)))
        cpu = {k_: v_ for k_, v_ in cb.items() if k_ not in ("keys", "seconds")}
        cpu["sample"] += f" ({cpu_model()}); GPU rows match: {parity}"

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": dev_ms_max / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference gen_mixture recipe, seed 1; 8 gaussians, spread 0.05)",
            "config": {"workload": f"cfg2: mixture n={a.n} refs, m={m} queries per GPU, d={DIM}, k={K}, "
                                   + ("ranks sharing GPUs (smoke test), " if shared else "")
                                   + 
                                   f"in-memory", "height": h, "mode": a.mode, "kernel": a.kernel,
                       "parallelism": f"query-sharded x{world} (tree replicated, no collective)",
                       "l2": "256 MiB write between steps; per-step inputs (1.2 GB) > L2",
                       "rounds": rounds, "pairs_per_query": pairs / (a.steps * m),
                       "build_seconds": build_s, "wall_ms_per_step": wall_ms / a.steps},
            "e2e": e2e,
            "gpu_launches": launches,
            "roofline": roofline,
            "roofline_fp32_equiv": roofline_fp32,
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    gpu.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
