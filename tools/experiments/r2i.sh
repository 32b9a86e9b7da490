#!/bin/bash
out=gpurun_out/${1:-r2i}; mkdir -p $out
python -m paper_1512_02831_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_parity.py -m gpu -x -q > $out/pytest.txt 2>&1; echo "rc=$?" >> $out/pytest.txt
BKT_VERBOSE=1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --check-rows 0 > $out/verbose.jsonl 2> $out/verbose.err
bash tools/quickbench.sh w4 >> $out/ab.txt
timeout 600 ncu --set full --import-source on --kernel-name regex:splitscan --launch-skip 19 --launch-count 1 -o $out/splitscan_full python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > $out/ncu.log 2>&1
echo done
