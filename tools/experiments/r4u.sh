#!/bin/bash
# long randomised parity sweep of HEAD (chunked host-resident plans in 30% of cases)
out=gpurun_out/${1:-r4u}; mkdir -p $out
timeout 1500 python tools/fuzz_parity.py --cases 5000 --seed 37 --seconds 1200 > $out/fuzz_parity_seed37.jsonl 2> $out/fuzz.err
grep -c '"chunks": [2-9]' $out/fuzz.err > $out/chunked_cases.txt
echo done
