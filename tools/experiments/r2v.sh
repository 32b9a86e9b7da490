#!/bin/bash
# L2 prefetch of split-scan windows (A/B), timelines, config 1 with the finisher from the start
out=gpurun_out/${1:-r2v}; mkdir -p $out
for r in 1 2; do
  bash tools/quickbench.sh pf0_$r BKT_LIB_NAME=libbkt_pf0.so >> $out/ab.txt
  bash tools/quickbench.sh pf1_$r BKT_LIB_NAME=libbkt_pf1.so >> $out/ab.txt
done
for L in 20; do
  BKT_LIB_NAME=libbkt_pf1.so BKT_SPLIT_DEBUG=$L timeout 300 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2> $out/tl_pf1_$L.err
  python tools/split_timeline.py $out/tl_pf1_$L.err > $out/tl_pf1_$L.txt 2>&1
done
for fa in default 70000; do
  for fc in 0 1; do
    if [ $fa = default ]; then e=""; else e="BKT_FINISH_AT=$fa BKT_FINISH_CTA=$fc"; fi
    env $e timeout 600 python tools/configs.py cfg1 > $out/cfg1_${fa}_$fc.jsonl 2> $out/cfg1_${fa}_$fc.err
  done
done
echo done
