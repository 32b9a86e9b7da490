#!/bin/bash
# wide-path tests; eager query loads in the split scan (A/B); ncu of advance + route
out=gpurun_out/${1:-r2n}; mkdir -p $out
L=paper_1512_02831_b200/_lib
timeout 900 python -m pytest tests/test_gpu_wide.py -m gpu -x -q > $out/pytest_wide.txt 2>&1; echo "rc=$?" >> $out/pytest_wide.txt
for r in 1 2; do
  bash tools/quickbench.sh q0_$r BKT_LIB_NAME=libbkt_q0.so >> $out/ab.txt
  bash tools/quickbench.sh q1_$r BKT_LIB_NAME=libbkt_q1.so >> $out/ab.txt
done
timeout 600 ncu --set full --import-source on -k regex:"advance|route_kernel" -s 20 -c 2 -o $out/adv_route \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > $out/ncu.log 2>&1
python tools/ncu_summary.py $out/adv_route.ncu-rep > $out/ncu_adv_route.txt 2>&1
echo done
