#!/bin/bash
# route early exit (BKT_ROUTE_EARLY=2/3) against the default build, + parity on the variants
out=gpurun_out/${1:-r3w}; mkdir -p $out
for r in 1 2 3; do
  for lib in libbkt.so libbkt_re2.so libbkt_re3.so; do
    bash tools/quickbench.sh ${lib%.so}_$r BKT_LIB_NAME=$lib >> $out/ab.txt 2>&1
  done
done
for lib in libbkt_re2.so libbkt_re3.so; do
  BKT_LIB_NAME=$lib timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale_parity.py -q -x > $out/parity_${lib%.so}.txt 2>&1
  echo "rc=$?" >> $out/parity_${lib%.so}.txt
done
# config 1: whole traversals per query from the start (warp / CTA finisher, wide path)
for v in "BKT_FINISH_AT=0" "BKT_FINISH_AT=8192 BKT_FINISH_CTA=0" "BKT_FINISH_AT=32768 BKT_FINISH_CTA=0" "BKT_FINISH_AT=65536 BKT_FINISH_CTA=0" \
         "BKT_FINISH_AT=65536 BKT_FINISH_CTA=1" "BKT_FORCE_WIDE=1"; do
  echo "== $v" >> $out/cfg1_sweep.txt
  env $v timeout 600 python tools/configs.py cfg1 >> $out/cfg1_sweep.txt 2>&1
done
echo done2
