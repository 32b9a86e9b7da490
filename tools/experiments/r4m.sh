#!/bin/bash
# final verification of HEAD: GPU suite, smoke, bench line, config 1
out=gpurun_out/${1:-r4m}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1
timeout 900 python bench.py > $out/bench.jsonl 2> $out/bench.err
python tools/configs.py cfg1 > $out/cfg1.jsonl 2>&1
echo done
