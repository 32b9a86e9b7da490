#!/bin/bash
# packed per-query records in split rounds
out=gpurun_out/${1:-r2u}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -x -q > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
bash tools/quickbench.sh u_1 >> $out/ab.txt
bash tools/quickbench.sh u_2 >> $out/ab.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2>&1
python tools/launch_summary.py $out/launches.csv > $out/launches_summary.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"advance" -s 20 -c 1 -o $out/adv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > $out/ncu.log 2>&1
python tools/ncu_summary.py $out/adv.ncu-rep > $out/ncu_adv.txt 2>&1
echo done
