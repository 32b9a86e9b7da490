#!/bin/bash
out=gpurun_out/${1:-r2e}; mkdir -p $out
python -m paper_1512_02831_b200.build > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > $out/b.log 2>&1
python tools/launch_summary.py $out/launches.csv > $out/launches_summary.txt
echo done
