#!/bin/bash
# quick GPU iteration: parity tests, a short bench, a TC timeline
# usage: tools/gpu_quick.sh TAG [extra bench args]
tag=$1; shift
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
BKT_TC_COUNTERS=1 python bench.py --steps 3 --warmup 2 --no-cpu "$@" > gpurun_out/bench_$tag.log 2> gpurun_out/bench_$tag.err
python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
l = [x for x in open(f"gpurun_out/bench_{tag}.log") if x.startswith("{")]
if l:
    j = json.loads(l[-1])
    print("value %.3fM e2e %.3fM leafscan_ms %.1f share %.3f frac %.3f" % (j["value"]/1e6, (j["e2e"] or {}).get("value", 0)/1e6,
          j["roofline"]["leafscan_ms_per_step"], j["roofline"]["leafscan_share"], j["roofline"]["frac"]))
else:
    print(open(f"gpurun_out/bench_{tag}.err").read()[-2000:])
PY
grep "tc counters" gpurun_out/bench_$tag.err | tail -1
BKT_TC_DEBUG=1 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu "$@" > /dev/null 2> gpurun_out/timeline_$tag.log
python tools/timeline.py gpurun_out/timeline_$tag.log
