#!/bin/bash
# config 1: tail-finisher thresholds (warp and CTA finishers) against the plain round loop
out=gpurun_out/${1:-r4c}; mkdir -p $out
python tools/configs.py cfg1 > $out/cfg1_base.jsonl 2>&1
for f in 512 2048 4096 8192 16384; do
  BKT_FINISH_AT=$f BKT_FINISH_CTA=0 python tools/configs.py cfg1 > $out/cfg1_warp_$f.jsonl 2>&1
  BKT_FINISH_AT=$f BKT_FINISH_CTA=1 python tools/configs.py cfg1 > $out/cfg1_cta_$f.jsonl 2>&1
done
for f in $out/cfg1_*.jsonl; do echo "$f $(grep -o '"kernel": "auto", "qps_device": [0-9.]*' $f) $(grep -o 'digest_matches_reference": [a-z]*' $f | head -1)"; done > $out/summary.txt
echo done
