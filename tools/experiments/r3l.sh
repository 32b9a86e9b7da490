#!/bin/bash
# route: warp-uniform loop, register window counts, paired box/query loads; advance 3 vs 4 CTAs/SM
out=gpurun_out/${1:-r3l}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q -x > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
for r in 1 2; do
  bash tools/quickbench.sh a3_$r >> $out/ab.txt
  bash tools/quickbench.sh a4_$r BKT_LIB_NAME=libbkt_adv4.so >> $out/ab.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2>&1
python tools/launch_summary.py $out/launches.csv > $out/launches_summary.txt
BKT_BENCH_DEBUG=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu --check-rows 0 > $out/bench_e2e.jsonl 2> $out/bench_e2e.err
echo done
