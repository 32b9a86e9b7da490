#!/bin/bash
# split scan 3 (default now) vs 4 CTAs/SM; parity of the default
out=gpurun_out/${1:-r3p}; mkdir -p $out
for r in 1 2; do
  bash tools/quickbench.sh c3_$r >> $out/ab.txt
  bash tools/quickbench.sh c4_$r BKT_LIB_NAME=libbkt_c4.so >> $out/ab.txt
done
timeout 1200 python -m pytest tests -m gpu -q -x > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
timeout 900 python tools/configs.py cfg5 --m 1e7 --resident hbm --ks 10,50 > $out/cfg5_hbm.jsonl 2> $out/cfg5_hbm.err
echo done
