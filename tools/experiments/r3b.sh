#!/bin/bash
out=gpurun_out/${1:-r3b}; mkdir -p $out
timeout 600 python tools/tc_repro.py > $out/tc_repro.jsonl 2> $out/tc_repro.err
BKT_TC_UNFUSED=1 timeout 600 python tools/tc_repro.py > $out/tc_repro_unfused.jsonl 2> $out/tc_repro_unfused.err
echo done
