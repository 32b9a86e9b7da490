#!/bin/bash
# round-2 measurement of the committed code: tests, smoke, bench + reference arm,
# launch list, full ncu of the split-round scan and the home-round TC scan
out=gpurun_out/${1:-r2m}; mkdir -p $out
nvidia-smi -q -d CLOCK > $out/clocks.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1
timeout 900 python bench.py > $out/bench.jsonl 2> $out/bench.err
timeout 900 python bench.py --impl reference > $out/bench_reference.jsonl 2> $out/bench_reference.err
BKT_VERBOSE=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --check-rows 0 > $out/verbose.jsonl 2> $out/verbose.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2>&1
python tools/launch_summary.py $out/launches.csv > $out/launches_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:splitscan -s 10 -c 1 -o $out/splitscan_full \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > $out/ncu_split.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:leafscan_tc -s 0 -c 1 -o $out/leafscan_home_full \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > $out/ncu_home.log 2>&1
python tools/ncu_summary.py $out/splitscan_full.ncu-rep > $out/ncu_splitscan_full.txt 2>&1
python tools/ncu_summary.py $out/leafscan_home_full.ncu-rep > $out/ncu_leafscan_home_full.txt 2>&1
echo done
