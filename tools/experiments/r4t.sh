#!/bin/bash
# batched warp merge A/B with repeated searches (second search of each k counts)
out=gpurun_out/${1:-r4t}; mkdir -p $out
timeout 900 python tools/configs.py cfg5 --m 2e6 --heights 11,14 --ks 16,16,50,50 --resident hbm > $out/k_batch.jsonl 2>&1
BKT_MERGE_BATCH=0 timeout 900 python tools/configs.py cfg5 --m 2e6 --heights 11,14 --ks 16,16,50,50 --resident hbm > $out/k_serial.jsonl 2>&1
echo done
