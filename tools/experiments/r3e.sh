#!/bin/bash
# split-scan float2 query loads, k-aware candidate slices: parity, bench, cfg5 k sweep
out=gpurun_out/${1:-r3e}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q -x > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
bash tools/quickbench.sh e_1 >> $out/ab.txt
bash tools/quickbench.sh e_2 >> $out/ab.txt
timeout 900 python tools/configs.py cfg5 --m 1e7 --resident hbm --ks 10,50 > $out/cfg5_hbm.jsonl 2> $out/cfg5_hbm.err
echo done
