#!/bin/bash
# round-2 probe: GPU tests, bench (new rank logic), reference arm, chunk-skip diagnostics
out=gpurun_out/${1:-probe}; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
timeout 600 python bench.py --steps 5 --warmup 3 > $out/bench.jsonl 2> $out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref.jsonl 2> $out/bench_ref.err
BKT_BUILD_DIAG=1 python -m paper_1512_02831_b200.build > $out/build_diag.txt 2>&1
BKT_TC_COUNTERS=1 BKT_TRACE_ROUNDS=1 BKT_TC_SKIPDIAG=1 timeout 600 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > $out/diag.jsonl 2> $out/diag.err
python -m paper_1512_02831_b200.build > /dev/null 2>&1
echo done
