#!/bin/bash
# new split scan: timelines + ncu full
out=gpurun_out/${1:-r3h}; mkdir -p $out
for Lc in 20; do
  BKT_SPLIT_DEBUG=$Lc timeout 300 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2> $out/tl_$Lc.err
  python tools/split_timeline.py $out/tl_$Lc.err > $out/tl_$Lc.txt 2>&1
  python tools/split_tile_gaps.py $out/tl_$Lc.err >> $out/tl_$Lc.txt 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:splitscan -s 19 -c 1 -o $out/splitscan_full \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2>&1
python tools/ncu_summary.py $out/splitscan_full.ncu-rep > $out/ncu_splitscan_full.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:advance -s 20 -c 1 -o $out/advance_full \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2>&1
python tools/ncu_summary.py $out/advance_full.ncu-rep > $out/ncu_advance_full.txt 2>&1
echo done
