#!/bin/bash
# config 1: warp tail finisher at high thresholds (a third to all of the batch)
out=gpurun_out/${1:-r4n}; mkdir -p $out
python tools/configs.py cfg1 > $out/cfg1_base.jsonl 2>&1
for f in 24000 32000 40000 50000 65536; do
  BKT_FINISH_AT=$f BKT_FINISH_CTA=0 python tools/configs.py cfg1 > $out/cfg1_warp_$f.jsonl 2>&1
done
for f in $out/cfg1_*.jsonl; do echo "$f $(grep -o '"kernel": "auto", "qps_device": [0-9.]*' $f) $(grep -o 'digest_matches_reference": [a-z]*' $f | head -1)"; done > $out/summary.txt
echo done
