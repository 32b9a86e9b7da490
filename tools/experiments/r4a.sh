#!/bin/bash
# session re-entry sanity: parity suite, bench line, config 1, host-resident h=14
out=gpurun_out/${1:-r4a}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
bash tools/quickbench.sh base > $out/qb.txt 2>&1
BKT_TRACE_ROUNDS=1 timeout 300 python tools/configs.py cfg1 > $out/cfg1.jsonl 2> $out/cfg1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_cfg1.csv python tools/configs.py cfg1 > /dev/null 2>&1
python tools/launch_summary.py $out/launches_cfg1.csv > $out/launches_cfg1_summary.txt
echo done
