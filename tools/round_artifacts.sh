#!/bin/bash
# Round-end measurement set (GPU box): parity tests, smoke, bench (+reference arm),
# ncu launch list, full captures of the split scan and the home-round scan, the
# split scan's DRAM bytes per pair, config sweeps, randomised parity sweep.
# usage: tools/round_artifacts.sh OUTDIR   (under gpurun_out/)
out=gpurun_out/$1; mkdir -p $out
nvidia-smi -q -d CLOCK > $out/clocks.txt 2>&1
lscpu > $out/lscpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > $out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1
timeout 900 python bench.py > $out/bench.jsonl 2> $out/bench.err
timeout 900 python bench.py --impl reference > $out/bench_reference.jsonl 2> $out/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2>&1
python tools/launch_summary.py $out/launches.csv > $out/launches_summary.txt
BKT_TRACE_ROUNDS=1 timeout 300 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2> $out/trace_rounds.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:splitscan -s 19 -c 1 -o $out/splitscan_full \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2>&1
python tools/ncu_summary.py $out/splitscan_full.ncu-rep > $out/ncu_splitscan_full.txt 2>&1
python tools/ncu_traffic.py $out/splitscan_full.ncu-rep $out/trace_rounds.err 20 2000000 512 > $out/ncu_traffic.json 2> $out/ncu_traffic.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_cfg4.csv python tools/configs.py cfg4 --m 2e6 > /dev/null 2>&1
python tools/launch_summary.py $out/launches_cfg4.csv > $out/launches_cfg4_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:leafscan_tc -s 0 -c 1 -o $out/leafscan_home_full \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2>&1
python tools/ncu_summary.py $out/leafscan_home_full.ncu-rep > $out/ncu_leafscan_home_full.txt 2>&1
for c in cfg1 cfg4 uniform2m; do timeout 900 python tools/configs.py $c > $out/$c.jsonl 2> $out/$c.err; done
timeout 1500 python tools/configs.py cfg5 --m 1e7 > $out/cfg5.jsonl 2> $out/cfg5.err
timeout 900 python tools/configs.py cfg3 --m 1e9 > $out/cfg3.jsonl 2> $out/cfg3.err
timeout 900 python tools/fuzz_parity.py --cases 3000 --seed 23 --seconds 720 > $out/fuzz_parity_seed23.jsonl 2> $out/fuzz.err
echo done
