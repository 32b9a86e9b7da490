#!/bin/bash
# quickbench.sh TAG [env...]: one short bench line summary
tag=$1; shift
env "$@" python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/qb_$tag.log 2>&1
python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
l = [x for x in open(f"gpurun_out/qb_{tag}.log") if x.startswith("{")]
if not l:
    print(tag, "FAILED"); print(open(f"gpurun_out/qb_{tag}.log").read()[-1500:]); sys.exit()
j = json.loads(l[-1])
print(tag, "value %.3fM leafscan %.1f ms step %.1f ms" % (j["value"] / 1e6, j["roofline"]["leafscan_ms_per_step"], j["ms_per_step"]))
PY
