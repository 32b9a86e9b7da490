#!/bin/bash
# timelines: split scan tile setup (new stamps), home-round TC scan
out=gpurun_out/${1:-r3d}; mkdir -p $out
L=paper_1512_02831_b200/_lib
for Lc in 20 40; do
  BKT_SPLIT_DEBUG=$Lc timeout 300 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2> $out/tl_$Lc.err
  python tools/split_timeline.py $out/tl_$Lc.err > $out/tl_$Lc.txt 2>&1
  python tools/split_tile_gaps.py $out/tl_$Lc.err >> $out/tl_$Lc.txt 2>&1
done
BKT_BUILD_DIAG=1 python -m paper_1512_02831_b200.build > /dev/null 2>&1 && cp $L/libbkt.so $L/libbkt_diag.so
python -m paper_1512_02831_b200.build > /dev/null 2>&1
BKT_LIB_NAME=libbkt_diag.so BKT_TC_DEBUG=0 timeout 300 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2> $out/tl_home.err
python tools/timeline.py $out/tl_home.err > $out/tl_home.txt 2>&1
echo done
