#!/bin/bash
# window width sweep on the current code
out=gpurun_out/${1:-r3m}; mkdir -p $out
for v in "BKT_SPLIT_W=4" "BKT_SPLIT_W=2" "BKT_SPLIT_W=8" "BKT_SPLIT_W=3"; do
  tag=$(echo $v | tr ' =' '_-')
  bash tools/quickbench.sh $tag $v >> $out/ab.txt
done
BKT_SPLIT_W=2 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_w2.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2>&1
python tools/launch_summary.py $out/launches_w2.csv > $out/launches_w2_summary.txt
echo done
