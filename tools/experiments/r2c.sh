#!/bin/bash
# round-2: per-chunk timeline of the current TC kernel (launch 3 and 19), stage-depth slope
out=gpurun_out/${1:-r2c}; mkdir -p $out
L=paper_1512_02831_b200/_lib
BKT_BUILD_DIAG=1 python -m paper_1512_02831_b200.build > /dev/null 2>&1 && cp $L/libbkt.so $L/libbkt_diag.so
for launch in 3 19 40; do
  BKT_LIB_NAME=libbkt_diag.so BKT_TC_DEBUG=$launch timeout 300 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2> $out/tl_$launch.err
  python tools/timeline.py $out/tl_$launch.err > $out/tl_$launch.txt 2>&1
done
BKT_BUILD_DEFS="-DBKT_TC_STAGES=3" python -m paper_1512_02831_b200.build > /dev/null 2>&1 && cp $L/libbkt.so $L/libbkt_s3.so
python -m paper_1512_02831_b200.build > /dev/null 2>&1
for r in 1 2; do
  bash tools/quickbench.sh s4_$r >> $out/ab.txt
  bash tools/quickbench.sh s3_$r BKT_LIB_NAME=libbkt_s3.so >> $out/ab.txt
done
echo done
