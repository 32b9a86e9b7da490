#!/bin/bash
# parity incl. brute-on-engine; fuzz; cfg5 h=11 k=10/50 launch lists
out=gpurun_out/${1:-r2y}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
for k in 10 50; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_cfg5_h11_k$k.csv \
    python tools/configs.py cfg5 --m 1e7 --resident hbm --ks $k --heights 11 > $out/cfg5_h11_k$k.jsonl 2>&1
  python tools/launch_summary.py $out/launches_cfg5_h11_k$k.csv > $out/launches_cfg5_h11_k${k}_summary.txt
done
timeout 900 python tools/fuzz_parity.py --cases 2000 --seed 11 --seconds 720 > $out/fuzz_parity_seed11.jsonl 2> $out/fuzz.err
echo done
