#!/bin/bash
# per-lane merge with batched candidate loads (launch bounds 3 vs 2 CTAs/SM), route f32x2 box tests
out=gpurun_out/${1:-r2t}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
for r in 1 2; do
  bash tools/quickbench.sh a3_$r BKT_LIB_NAME=libbkt_a3.so >> $out/ab.txt
  bash tools/quickbench.sh a2_$r BKT_LIB_NAME=libbkt_a2.so >> $out/ab.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2>&1
python tools/launch_summary.py $out/launches.csv > $out/launches_summary.txt
echo done
