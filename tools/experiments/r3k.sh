#!/bin/bash
out=gpurun_out/${1:-r3k}; mkdir -p $out
timeout 900 python bench.py > $out/bench.jsonl 2> $out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2>&1
python tools/launch_summary.py $out/launches.csv > $out/launches_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:splitscan -s 19 -c 1 -o $out/splitscan_full \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2>&1
python tools/ncu_summary.py $out/splitscan_full.ncu-rep > $out/ncu_splitscan_full.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:route -s 19 -c 1 -o $out/route_full \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2>&1
python tools/ncu_summary.py $out/route_full.ncu-rep > $out/ncu_route_full.txt 2>&1
echo done
