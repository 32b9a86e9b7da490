#!/bin/bash
# run the bench under several env settings (diag build) and summarise
for v in "$@"; do
  env $v BKT_TC_COUNTERS=1 python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/var.log 2> gpurun_out/var.err
  python - "$v" <<'PY'
import json, sys
l = [x for x in open("gpurun_out/var.log") if x.startswith("{")]
c = [x for x in open("gpurun_out/var.err") if x.startswith("tc counters")]
if not l:
    print(sys.argv[1], "FAILED", open("gpurun_out/var.err").read()[-1500:]); sys.exit()
j = json.loads(l[-1])
f = c[-1].split()
d = {f[i]: int(f[i + 1]) for i in range(2, len(f) - 1, 2)}
print("%-40s value %.2fM leafscan %.0f ms scanned %.3f warp_mine %.3f surv/q %.0f trips %d" % (
    sys.argv[1], j["value"] / 1e6, j["roofline"]["leafscan_ms_per_step"], j["config"]["scanned_fraction"],
    d["warp_chunks_mine"] / max(1, d["warp_chunks"]), d["survivors"] / 1e7, d["loop_trips"]))
PY
done
