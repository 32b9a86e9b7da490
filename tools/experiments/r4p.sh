#!/bin/bash
# k = 50 home-round scan at two CTAs per SM (registers capped at 168, spills) vs one
out=gpurun_out/${1:-r4p}; mkdir -p $out
timeout 900 python tools/configs.py cfg5 --m 2e6 --heights 8,11 --ks 50 --resident hbm > $out/k50_base.jsonl 2>&1
BKT_BUILD_DEFS="-DBKT_TC_BIGK_MINB=2" python -m paper_1512_02831_b200.build > $out/build2.txt 2>&1
BKT_TC_BIGK_CTAS=2 timeout 900 python tools/configs.py cfg5 --m 2e6 --heights 8,11 --ks 50 --resident hbm > $out/k50_cta2.jsonl 2>&1
BKT_TC_BIGK_CTAS=2 timeout 900 python -m pytest tests/test_gpu_scale_parity.py -q -x -k "hbm and 50" > $out/parity_cta2.txt 2>&1; echo "rc=$?" >> $out/parity_cta2.txt
cuobjdump -res-usage paper_1512_02831_b200/_lib/obj/leafscan_tc_16_128_2_0.o 2>/dev/null | grep -A1 "Li64ELb0ELi128ELi2E" | head -4 > $out/res_usage.txt
echo done
