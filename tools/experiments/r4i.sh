#!/bin/bash
# spilled structure test + full suite; config 1 with three TC CTAs per SM (one accumulator each)
out=gpurun_out/${1:-r4i}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
python tools/configs.py cfg1 > $out/cfg1_base.jsonl 2>&1
BKT_TC_CPS=3 BKT_TC_N=128 python tools/configs.py cfg1 > $out/cfg1_cps3_n128.jsonl 2>&1
BKT_TC_CPS=3 python tools/configs.py cfg1 > $out/cfg1_cps3_n64.jsonl 2>&1
BKT_TC_N=64 python tools/configs.py cfg1 > $out/cfg1_n64.jsonl 2>&1
for f in $out/cfg1_*.jsonl; do echo "$f $(grep -o '"kernel": "auto", "qps_device": [0-9.]*' $f) $(grep -o 'digest_matches_reference": [a-z]*' $f | head -1)"; done > $out/summary.txt
echo done
