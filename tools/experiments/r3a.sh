#!/bin/bash
# fuzz failure repro (seed 11 case 68): TMEM load pipelining on/off
out=gpurun_out/${1:-r3a}; mkdir -p $out
timeout 300 python tools/fuzz_parity.py --seed 11 --only 68 --cases 69 > $out/repro_pipe1.txt 2>&1
BKT_LIB_NAME=libbkt_pipe0.so timeout 300 python tools/fuzz_parity.py --seed 11 --only 68 --cases 69 > $out/repro_pipe0.txt 2>&1
BKT_SPLIT=0 timeout 300 python tools/fuzz_parity.py --seed 11 --only 68 --cases 69 > $out/repro_nosplit.txt 2>&1
echo done
