#!/bin/bash
# config 1: split vs leaf-level TC vs direct, launch lists
out=gpurun_out/${1:-r2w}; mkdir -p $out
timeout 600 python tools/configs.py cfg1 > $out/cfg1_default.jsonl 2> $out/cfg1_default.err
BKT_SPLIT=0 timeout 600 python tools/configs.py cfg1 > $out/cfg1_nosplit.jsonl 2> $out/cfg1_nosplit.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_cfg1.csv python tools/configs.py cfg1 > /dev/null 2>&1
python tools/launch_summary.py $out/launches_cfg1.csv > $out/launches_cfg1_summary.txt
BKT_SPLIT=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_cfg1_ns.csv python tools/configs.py cfg1 > /dev/null 2>&1
python tools/launch_summary.py $out/launches_cfg1_ns.csv > $out/launches_cfg1_ns_summary.txt
echo done
