#!/bin/bash
# NR=64 stale-group fix; KB>=32 TC variants at 1 CTA/SM; full GPU tests; fuzz; cfg5 k=50
out=gpurun_out/${1:-r3c}; mkdir -p $out
timeout 600 python tools/tc_repro.py > $out/tc_repro.jsonl 2> $out/tc_repro.err
timeout 1200 python -m pytest tests -m gpu -q > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
bash tools/quickbench.sh c_1 >> $out/ab.txt
timeout 900 python tools/configs.py cfg5 --m 1e7 --resident hbm --ks 10,50 > $out/cfg5_hbm.jsonl 2> $out/cfg5_hbm.err
timeout 900 python tools/fuzz_parity.py --cases 3000 --seed 11 --seconds 840 > $out/fuzz_parity_seed11.jsonl 2> $out/fuzz.err
echo done
