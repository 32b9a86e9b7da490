#!/bin/bash
# advance_kernel query rows as float pairs (BKT_ADV_Q2 build define): parity + A/B
out=gpurun_out/${1:-r4w}; mkdir -p $out
for r in 1 2; do bash tools/quickbench.sh base_$r >> $out/ab.txt 2>&1; done
BKT_BUILD_DEFS="-DBKT_ADV_Q2=1" python -m paper_1512_02831_b200.build > $out/build_q2.txt 2>&1
for r in 1 2 3; do bash tools/quickbench.sh q2_$r >> $out/ab.txt 2>&1; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -q -x > $out/parity_q2.txt 2>&1; echo "rc=$?" >> $out/parity_q2.txt
echo done
