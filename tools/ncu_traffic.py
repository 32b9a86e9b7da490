"""DRAM bytes per algorithmic pair of one captured split-scan launch
(bench.py `roofline.traffic` reads the latest profiles/r*/ncu_traffic.json).

    python tools/ncu_traffic.py CAPTURE.ncu-rep TRACE.err ROUND N NL > ncu_traffic.json

CAPTURE: `ncu --set full -k regex:splitscan -s S -c 1` of one bench step (the
split launch of round ROUND = S + 1: round 0 is the home round);
TRACE: stderr of a `BKT_TRACE_ROUNDS=1` run of the same step (per-round
active queries); N / NL: points and leaves (leaves hold N / NL points
within one, so the round's pairs are its active queries x N / NL).
"""
import csv
import io
import json
import subprocess
import sys


def main(rep, trace, rnd, n, nl):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    d = dict(zip(hdr, rows[2]))
    u = dict(zip(hdr, units))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = float(d["dram__bytes_read.sum"]) * scale[u["dram__bytes_read.sum"]]
    wr = float(d["dram__bytes_write.sum"]) * scale[u["dram__bytes_write.sum"]]
    tscale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
    ms = float(d["gpu__time_duration.sum"]) * tscale[u["gpu__time_duration.sum"]]
    active = None
    for line in open(trace):
        f = line.split()
        if len(f) >= 4 and f[0] == "round" and int(f[1]) == rnd:
            active = int(f[3])
    pairs = active * n / nl
    print(json.dumps({
        "kernel": d.get("Kernel Name", "?"),
        "capture": f"ncu --set full, split-scan launch of round {rnd} of config 2 ({rep})",
        "dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr, "duration_ms": ms,
        "active_queries": active, "mean_leaf_points": n / nl, "pairs": pairs,
        "dram_bytes_per_pair": (rd + wr) / pairs,
        "algorithmic_bytes_per_pair": 200.0 / (n / nl),
        "note": "algorithmic bytes = 200 B per (query, leaf visit): query 4d + top-k 2*8k (SURVEY.md sec. 8(d)), "
                "per pair = 200 / mean leaf points"}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), float(sys.argv[4]), float(sys.argv[5]))
