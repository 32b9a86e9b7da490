#!/bin/bash
# fused advance+route (no per-leaf bucketing in split rounds): parity, bench, launch list
out=gpurun_out/${1:-r2o}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
bash tools/quickbench.sh new_1 >> $out/ab.txt
bash tools/quickbench.sh new_2 >> $out/ab.txt
BKT_VERBOSE=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --check-rows 0 > $out/verbose.jsonl 2> $out/verbose.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2>&1
python tools/launch_summary.py $out/launches.csv > $out/launches_summary.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"advance|place_kernel" -s 20 -c 2 -o $out/adv_place \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > $out/ncu.log 2>&1
python tools/ncu_summary.py $out/adv_place.ncu-rep > $out/ncu_adv_place.txt 2>&1
echo done
