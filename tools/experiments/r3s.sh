#!/bin/bash
out=gpurun_out/${1:-r3s}; mkdir -p $out
timeout 600 python tools/e2e_probe2.py > $out/e2e_probe2.txt 2>&1
BKT_BENCH_DEBUG=1 timeout 900 python bench.py --no-cpu > $out/bench.jsonl 2> $out/bench.err
echo done
