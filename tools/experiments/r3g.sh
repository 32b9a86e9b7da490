#!/bin/bash
# deferred survivor evaluation (split scan writes survivor rows; advance evaluates): parity, A/B, cfg5
out=gpurun_out/${1:-r3g}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q -x > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
for r in 1 2; do
  bash tools/quickbench.sh new_$r >> $out/ab.txt
  bash tools/quickbench.sh old_$r BKT_LIB_NAME=libbkt_old.so >> $out/ab.txt
done
BKT_VERBOSE=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --check-rows 0 > /dev/null 2> $out/verbose.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2>&1
python tools/launch_summary.py $out/launches.csv > $out/launches_summary.txt
timeout 900 python tools/configs.py cfg5 --m 1e7 --resident hbm --ks 10,50 > $out/cfg5_hbm.jsonl 2> $out/cfg5_hbm.err
echo done
