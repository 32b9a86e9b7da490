#!/bin/bash
# cooperative merge (k > 10), warp-row rescan, even capw; fuzz; cfg5 k=50
out=gpurun_out/${1:-r2z}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q -x > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
bash tools/quickbench.sh z_1 >> $out/ab.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_cfg5_h11_k50.csv \
  python tools/configs.py cfg5 --m 1e7 --resident hbm --ks 50 --heights 11 > $out/cfg5_h11_k50.jsonl 2>&1
python tools/launch_summary.py $out/launches_cfg5_h11_k50.csv > $out/launches_cfg5_h11_k50_summary.txt
timeout 900 python tools/fuzz_parity.py --cases 2000 --seed 11 --seconds 720 > $out/fuzz_parity_seed11.jsonl 2> $out/fuzz.err
echo done
