#!/bin/bash
# tensor-core drain: parity, config 5 host-resident (k = 1 / 10 / 50, h = 8 / 11 / 14)
out=gpurun_out/${1:-r4e}; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "out_of_core or edge or run_engine" > $out/parity_ooc.txt 2>&1; echo "rc=$?" >> $out/parity_ooc.txt
timeout 900 python -m pytest tests/test_gpu_scale_parity.py -q -x -k "host4" > $out/parity_scale_host.txt 2>&1; echo "rc=$?" >> $out/parity_scale_host.txt
timeout 1500 python tools/configs.py cfg5 --m 1e7 --heights 8,11,14 --ks 1,10,50 --resident host > $out/cfg5_host.jsonl 2> $out/cfg5_host.err
echo done
