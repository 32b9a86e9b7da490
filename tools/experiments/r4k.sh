#!/bin/bash
# randomised parity sweep including host-resident chunked plans (drain)
out=gpurun_out/${1:-r4k}; mkdir -p $out
timeout 900 python tools/fuzz_parity.py --cases 3000 --seed 29 --seconds 660 > $out/fuzz_parity_seed29.jsonl 2> $out/fuzz.err
grep -c '"chunks": [2-9]' $out/fuzz.err > $out/chunked_cases.txt
echo done
