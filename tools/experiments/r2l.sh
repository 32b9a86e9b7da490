#!/bin/bash
out=gpurun_out/${1:-r2l}; mkdir -p $out
python -m paper_1512_02831_b200.build > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --kernel-name regex:"advance|route_kernel" --launch-skip 20 --launch-count 2 -o $out/adv_route python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > $out/ncu.log 2>&1
echo done
