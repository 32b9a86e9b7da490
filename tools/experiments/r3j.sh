#!/bin/bash
# split scan: one-pass masks, release before writes (A/B), parity, timeline
out=gpurun_out/${1:-r3j}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q -x > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
for r in 1 2; do
  bash tools/quickbench.sh op1_$r >> $out/ab.txt
  bash tools/quickbench.sh op0_$r BKT_LIB_NAME=libbkt_op0.so >> $out/ab.txt
done
BKT_SPLIT_DEBUG=20 timeout 300 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2> $out/tl_20.err
python tools/split_timeline.py $out/tl_20.err > $out/tl_20.txt 2>&1
echo done
