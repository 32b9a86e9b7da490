#!/bin/bash
# warp-cooperative merge in advance; CUDA-graph split rounds (config 1)
out=gpurun_out/${1:-r2s}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
bash tools/quickbench.sh s_1 >> $out/ab.txt
bash tools/quickbench.sh s_2 >> $out/ab.txt
timeout 600 python tools/configs.py cfg1 > $out/cfg1_graph.jsonl 2> $out/cfg1_graph.err
BKT_GRAPH=0 timeout 600 python tools/configs.py cfg1 > $out/cfg1_eager.jsonl 2> $out/cfg1_eager.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2>&1
python tools/launch_summary.py $out/launches.csv > $out/launches_summary.txt
echo done
