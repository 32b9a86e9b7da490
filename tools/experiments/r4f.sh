#!/bin/bash
# full GPU suite after the drain, bench, config-1 round trace
out=gpurun_out/${1:-r4f}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
bash tools/quickbench.sh base > $out/qb.txt 2>&1
BKT_TRACE_ROUNDS=1 timeout 300 python tools/cfg1_trace.py > $out/cfg1_trace.json 2> $out/cfg1_trace.err
echo done
