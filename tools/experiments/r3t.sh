#!/bin/bash
# home-round scan timeline (diag build)
out=gpurun_out/${1:-r3t}; mkdir -p $out
L=paper_1512_02831_b200/_lib
BKT_BUILD_DIAG=1 python -m paper_1512_02831_b200.build > /dev/null 2>&1 && cp $L/libbkt.so $L/libbkt_diag.so
python -m paper_1512_02831_b200.build > /dev/null 2>&1
BKT_LIB_NAME=libbkt_diag.so BKT_TC_DEBUG=0 timeout 300 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2> $out/tl_home.err
python tools/timeline.py $out/tl_home.err > $out/tl_home.txt 2>&1
BKT_LIB_NAME=libbkt_diag.so BKT_TC_COUNTERS=1 BKT_TRACE_ROUNDS=1 timeout 300 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2> $out/counters.err
echo done
