#!/bin/bash
# split scan: 3 CTAs/SM with one accumulator each vs 2 CTAs with two (A/B); parity on the 3-CTA build
out=gpurun_out/${1:-r3o}; mkdir -p $out
for r in 1 2; do
  bash tools/quickbench.sh c2_$r >> $out/ab.txt
  bash tools/quickbench.sh c3_$r BKT_LIB_NAME=libbkt_c3.so >> $out/ab.txt
done
BKT_LIB_NAME=libbkt_c3.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -m gpu -q -x > $out/pytest_c3.txt 2>&1; echo "rc=$?" >> $out/pytest_c3.txt
echo done
