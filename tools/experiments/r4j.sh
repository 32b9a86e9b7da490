#!/bin/bash
# home-round scan at three CTAs per SM under split rounds (BKT_HOME_CPS=3): parity + A/B
out=gpurun_out/${1:-r4j}; mkdir -p $out
BKT_HOME_CPS=3 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "config2 or golden" > $out/parity_home3.txt 2>&1; echo "rc=$?" >> $out/parity_home3.txt
for r in 1 2; do
  bash tools/quickbench.sh base_$r >> $out/ab.txt 2>&1
  bash tools/quickbench.sh home3_$r BKT_HOME_CPS=3 >> $out/ab.txt 2>&1
done
echo done
timeout 1200 python -m pytest tests -m gpu -q > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
python tools/configs.py cfg1 > $out/cfg1.jsonl 2>&1
BKT_TC_CPS=2 python tools/configs.py cfg1 > $out/cfg1_cps2.jsonl 2>&1
timeout 900 python tools/configs.py cfg4 > $out/cfg4.jsonl 2> $out/cfg4.err
BKT_TC_CPS=2 timeout 900 python tools/configs.py cfg4 > $out/cfg4_cps2.jsonl 2> $out/cfg4_cps2.err
echo done2
