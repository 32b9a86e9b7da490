#!/bin/bash
# Round-end measurement set (GPU box): parity tests, smoke, bench (+reference arm),
# ncu launch list and full capture of the leaf scan, config sweeps.
# usage: tools/round_artifacts.sh OUTDIR   (under gpurun_out/)
out=gpurun_out/$1; mkdir -p $out
nvidia-smi -q -d CLOCK > $out/clocks.txt 2>&1
lscpu > $out/lscpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1
timeout 900 python bench.py > $out/bench.jsonl 2> $out/bench.err
timeout 900 python bench.py --impl reference > $out/bench_reference.jsonl 2> $out/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
python tools/launch_summary.py $out/launches.csv > $out/launches_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:leafscan_tc -s 20 -c 1 -o $out/leafscan_full \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
python tools/ncu_summary.py $out/leafscan_full.ncu-rep > $out/ncu_leafscan_full.txt 2>&1
for c in cfg1 cfg4; do timeout 900 python tools/configs.py $c > $out/$c.jsonl 2> $out/$c.err; done
timeout 600 python tools/finish_sweep.py --at=-1,default > $out/finish_sweep.jsonl 2>&1
timeout 900 python tools/configs.py cfg3 --m 1e8 > $out/cfg3.jsonl 2> $out/cfg3.err
timeout 1200 python tools/configs.py cfg5 --m 1e6 > $out/cfg5.jsonl 2> $out/cfg5.err
echo done
