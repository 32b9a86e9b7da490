#!/bin/bash
out=gpurun_out/${1:-r2j}; mkdir -p $out
python -m paper_1512_02831_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_parity.py -m gpu -x -q > $out/pytest.txt 2>&1; echo "rc=$?" >> $out/pytest.txt
BKT_VERBOSE=1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --check-rows 0 > $out/verbose.jsonl 2> $out/verbose.err
for v in "BKT_SPLIT_W=4" "BKT_SPLIT_W=2" "BKT_SPLIT_W=8"; do
  tag=$(echo $v | tr ' =' '_-')
  bash tools/quickbench.sh $tag $v >> $out/ab.txt
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > $out/b.log 2>&1
python tools/launch_summary.py $out/launches.csv > $out/launches_summary.txt
echo done
