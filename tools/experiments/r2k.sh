#!/bin/bash
out=gpurun_out/${1:-r2k}; mkdir -p $out
python -m paper_1512_02831_b200.build > /dev/null 2>&1
for L in 2 20 40; do
  BKT_SPLIT_DEBUG=$L timeout 300 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2> $out/tl_$L.err
  python tools/split_timeline.py $out/tl_$L.err > $out/tl_$L.txt 2>&1
done
bash tools/quickbench.sh w4 >> $out/ab.txt
bash tools/quickbench.sh w8 BKT_SPLIT_W=8 >> $out/ab.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > $out/b.log 2>&1
python tools/launch_summary.py $out/launches.csv > $out/launches_summary.txt
echo done
