#!/bin/bash
# out-of-core drain schedule: parity, then config 5 host-resident drain vs rounds
out=gpurun_out/${1:-r4b}; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "out_of_core or edge or run_engine" > $out/parity_ooc.txt 2>&1; echo "rc=$?" >> $out/parity_ooc.txt
timeout 900 python -m pytest tests/test_gpu_scale_parity.py -q -x -k "host4" > $out/parity_scale_host.txt 2>&1; echo "rc=$?" >> $out/parity_scale_host.txt
BKT_VERBOSE=1 timeout 900 python tools/configs.py cfg5 --m 1e7 --heights 8,11,14 --ks 10 --resident host > $out/cfg5_drain.jsonl 2> $out/cfg5_drain.err
BKT_OOC_ROUNDS=1 timeout 900 python tools/configs.py cfg5 --m 1e7 --heights 14 --ks 10 --resident host > $out/cfg5_rounds.jsonl 2> $out/cfg5_rounds.err
timeout 900 python tools/configs.py cfg5 --m 1e7 --heights 8,11,14 --ks 10 --resident hbm > $out/cfg5_hbm.jsonl 2> $out/cfg5_hbm.err
echo done
