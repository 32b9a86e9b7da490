#!/bin/bash
# ncu --set full of the round kernels of config 2 (advance, route, place, plan_split, scatter, rescan) at round 20
out=gpurun_out/${1:-r4r}; mkdir -p $out
for kn in advance_kernel route_kernel place_kernel scatter_kernel rescan_kernel; do
  timeout 600 ncu --set full --clock-control none -k regex:$kn -s 20 -c 1 -o $out/$kn \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --check-rows 0 > /dev/null 2>&1
  python tools/ncu_summary.py $out/$kn.ncu-rep > $out/ncu_$kn.txt 2>&1
done
echo done
