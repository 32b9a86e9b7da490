#!/bin/bash
# round-2: TMEM read ceiling + scale parity tests
out=gpurun_out/${1:-r2b}; mkdir -p $out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem_bw tools/tmem_bw.cu && timeout 120 /tmp/tmem_bw > $out/tmem_bw.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_scale_parity.py -m gpu -x -q --durations=30 > $out/pytest_scale.txt 2>&1; echo "rc=$?" >> $out/pytest_scale.txt
echo done
