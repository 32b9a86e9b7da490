#!/bin/bash
# k = 50 breakdown: launch lists of config 5 h = 8 / 11 at k = 10 and 50 (HBM-resident, m = 2M)
out=gpurun_out/${1:-r4l}; mkdir -p $out
for k in 10 50; do for h in 8 11; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_h${h}_k$k.csv \
    python tools/configs.py cfg5 --m 2e6 --heights $h --ks $k --resident hbm > $out/cfg5_h${h}_k$k.jsonl 2>&1
  python tools/launch_summary.py $out/launches_h${h}_k$k.csv > $out/launches_h${h}_k${k}_summary.txt
done; done
echo done
