#!/bin/bash
# bench (pinned e2e inputs) + window sweep + advance/route ncu on the 3-CTA build
out=gpurun_out/${1:-r3q}; mkdir -p $out
timeout 900 python bench.py > $out/bench.jsonl 2> $out/bench.err
for v in "BKT_SPLIT_W=8" "BKT_SPLIT_W=2"; do
  tag=$(echo $v | tr ' =' '_-')
  bash tools/quickbench.sh $tag $v >> $out/ab.txt
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:advance -s 20 -c 1 -o $out/advance_full \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2>&1
python tools/ncu_summary.py $out/advance_full.ncu-rep > $out/ncu_advance_full.txt 2>&1
echo done
