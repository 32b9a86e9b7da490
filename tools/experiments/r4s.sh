#!/bin/bash
# batched warp merge (k > 10 split rounds): GPU suite, k = 16/50 A/B, fuzz
out=gpurun_out/${1:-r4s}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q -x > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
timeout 900 python tools/configs.py cfg5 --m 2e6 --heights 8,11 --ks 16,50 --resident hbm > $out/k_batch.jsonl 2>&1
BKT_MERGE_BATCH=0 timeout 900 python tools/configs.py cfg5 --m 2e6 --heights 8,11 --ks 16,50 --resident hbm > $out/k_serial.jsonl 2>&1
timeout 600 python tools/fuzz_parity.py --cases 3000 --seed 31 --seconds 420 > $out/fuzz_parity_seed31.jsonl 2> $out/fuzz.err
echo done
