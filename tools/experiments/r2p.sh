#!/bin/bash
# route/advance micro-optimisations: parity, bench, launch list, split-scan timelines
out=gpurun_out/${1:-r2p}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
bash tools/quickbench.sh p_1 >> $out/ab.txt
bash tools/quickbench.sh p_2 >> $out/ab.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2>&1
python tools/launch_summary.py $out/launches.csv > $out/launches_summary.txt
for L in 2 20 40; do
  BKT_SPLIT_DEBUG=$L timeout 300 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2> $out/tl_$L.err
  python tools/split_timeline.py $out/tl_$L.err > $out/tl_$L.txt 2>&1
done
echo done
