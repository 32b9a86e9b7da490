#!/bin/bash
# fused plan+scatter: GPU suite, config 1 A/B, config 4 (d = 5 runs leaf-level rounds)
out=gpurun_out/${1:-r4g}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q -x > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
for r in 1 2; do
  python tools/configs.py cfg1 > $out/cfg1_fused_$r.jsonl 2>&1
  BKT_FUSED_PS=0 python tools/configs.py cfg1 > $out/cfg1_twolaunch_$r.jsonl 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_cfg1.csv python tools/configs.py cfg1 > /dev/null 2>&1
python tools/launch_summary.py $out/launches_cfg1.csv > $out/launches_cfg1_summary.txt
timeout 900 python tools/configs.py cfg4 > $out/cfg4.jsonl 2> $out/cfg4.err
echo done
