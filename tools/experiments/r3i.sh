#!/bin/bash
# advance: warp-cooperative survivor evaluation (k <= 10): parity, A/B, launch list
out=gpurun_out/${1:-r3i}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q -x > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
for r in 1 2; do
  bash tools/quickbench.sh new_$r >> $out/ab.txt
  bash tools/quickbench.sh prev_$r BKT_LIB_NAME=libbkt_prev.so >> $out/ab.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2>&1
python tools/launch_summary.py $out/launches.csv > $out/launches_summary.txt
timeout 900 python tools/configs.py cfg5 --m 1e7 --resident hbm --ks 10 --heights 8,11 > $out/cfg5_hbm.jsonl 2> $out/cfg5_hbm.err
echo done
