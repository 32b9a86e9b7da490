#!/bin/bash
# home round on the split path (BKT_SEED_HOME=1: seed_kernel bound from the home block)
out=gpurun_out/${1:-r3x}; mkdir -p $out
BKT_SEED_HOME=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > $out/parity_seed.txt 2>&1; echo "rc=$?" >> $out/parity_seed.txt
for r in 1 2; do
  bash tools/quickbench.sh base_$r >> $out/ab.txt 2>&1
  bash tools/quickbench.sh seed_$r BKT_SEED_HOME=1 >> $out/ab.txt 2>&1
done
BKT_SEED_HOME=1 BKT_VERBOSE=1 BKT_TRACE_ROUNDS=1 timeout 300 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2> $out/trace_seed.err
BKT_VERBOSE=1 BKT_TRACE_ROUNDS=1 timeout 300 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2> $out/trace_base.err
BKT_SEED_HOME=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_seed.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2>&1
python tools/launch_summary.py $out/launches_seed.csv > $out/launches_seed_summary.txt
BKT_SEED_HOME=1 timeout 600 python -m pytest tests/test_gpu_scale_parity.py -q -x > $out/parity_seed_scale.txt 2>&1; echo "rc=$?" >> $out/parity_seed_scale.txt
echo done
