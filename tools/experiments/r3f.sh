#!/bin/bash
# one-window leaves on split rounds for k > 16 (cfg5 h=14), with/without
out=gpurun_out/${1:-r3f}; mkdir -p $out
timeout 900 python tools/configs.py cfg5 --m 1e7 --resident hbm --ks 10,50 --heights 14 > $out/cfg5_h14.jsonl 2> $out/cfg5_h14.err
BKT_SPLIT_NW1=1 timeout 900 python tools/configs.py cfg5 --m 1e7 --resident hbm --ks 10 --heights 14 > $out/cfg5_h14_nw1.jsonl 2> $out/cfg5_h14_nw1.err
BKT_SPLIT=0 timeout 900 python tools/configs.py cfg5 --m 1e7 --resident hbm --ks 50 --heights 14 > $out/cfg5_h14_nosplit.jsonl 2> $out/cfg5_h14_nosplit.err
timeout 900 python tools/configs.py cfg5 --m 1e7 --resident host --ks 10,50 --heights 8,11,14 > $out/cfg5_host.jsonl 2> $out/cfg5_host.err
echo done
