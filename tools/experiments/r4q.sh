#!/bin/bash
# programmatic dependent launch in the fused leaf-level rounds: GPU suite + config 1 A/B + config 4
out=gpurun_out/${1:-r4q}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q -x > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
for r in 1 2 3; do
  python tools/configs.py cfg1 > $out/cfg1_pdl_$r.jsonl 2>&1
  BKT_PDL=0 python tools/configs.py cfg1 > $out/cfg1_nopdl_$r.jsonl 2>&1
done
for f in $out/cfg1_*.jsonl; do echo "$f $(grep -o '"kernel": "auto", "qps_device": [0-9.]*' $f) $(grep -o '"kernel": "direct", "qps_device": [0-9.]*' $f) $(grep -o 'digest_matches_reference": [a-z]*' $f | head -1)"; done > $out/summary.txt
timeout 600 python tools/configs.py cfg4 > $out/cfg4.jsonl 2> $out/cfg4.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1
bash tools/quickbench.sh base > $out/qb.txt 2>&1
echo done
