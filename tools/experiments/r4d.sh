#!/bin/bash
# drain + unit finisher: parity, config 5 host-resident, config-1 finisher sweep
out=gpurun_out/${1:-r4d}; mkdir -p $out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "out_of_core or edge or run_engine" > $out/parity_ooc.txt 2>&1; echo "rc=$?" >> $out/parity_ooc.txt
timeout 900 python -m pytest tests/test_gpu_scale_parity.py -q -x -k "host4" > $out/parity_scale_host.txt 2>&1; echo "rc=$?" >> $out/parity_scale_host.txt
timeout 900 python tools/configs.py cfg5 --m 1e7 --heights 8,11,14 --ks 10 --resident host > $out/cfg5_drain.jsonl 2> $out/cfg5_drain.err
BKT_FINISH_AT=-1 timeout 900 python tools/configs.py cfg5 --m 1e7 --heights 14 --ks 10 --resident host > $out/cfg5_drain_nofin.jsonl 2> $out/cfg5_drain_nofin.err
bash tools/experiments/r4c.sh ${1:-r4d}
