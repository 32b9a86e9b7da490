#!/bin/bash
# config 1 without split rounds / mirror fence; cfg5 HBM k sweep; cfg3 at 1e9
out=gpurun_out/${1:-r2x}; mkdir -p $out
timeout 600 python tools/configs.py cfg1 > $out/cfg1.jsonl 2> $out/cfg1.err
bash tools/quickbench.sh x_1 >> $out/ab.txt
timeout 1500 python tools/configs.py cfg5 --m 1e7 --resident hbm --ks 10,50 > $out/cfg5_hbm.jsonl 2> $out/cfg5_hbm.err
timeout 1500 python tools/configs.py cfg3 --m 1e9 > $out/cfg3_1e9.jsonl 2> $out/cfg3_1e9.err
echo done
