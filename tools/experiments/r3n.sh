#!/bin/bash
# home-round scan: last two groups processed from registers (A/B)
out=gpurun_out/${1:-r3n}; mkdir -p $out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -m gpu -q -x > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
for r in 1 2; do
  bash tools/quickbench.sh hr1_$r BKT_LIB_NAME=libbkt_hr1.so >> $out/ab.txt
  bash tools/quickbench.sh hr0_$r BKT_LIB_NAME=libbkt_hr0.so >> $out/ab.txt
done
echo done
