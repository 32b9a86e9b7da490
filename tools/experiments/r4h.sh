#!/bin/bash
# config 1: one tensor-core round scan under the per-chunk timestamp probe and ncu --set full
out=gpurun_out/${1:-r4h}; mkdir -p $out
BKT_TC_DEBUG=100 timeout 300 python tools/cfg1_trace.py > /dev/null 2> $out/tc_debug_round100.txt
BKT_TC_DEBUG=230 timeout 300 python tools/cfg1_trace.py > /dev/null 2> $out/tc_debug_round230.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:leafscan_tc -s 100 -c 1 -o $out/cfg1_tc_full python tools/cfg1_trace.py > /dev/null 2>&1
python tools/ncu_summary.py $out/cfg1_tc_full.ncu-rep > $out/ncu_cfg1_tc_full.txt 2>&1
echo done
