#!/bin/bash
# split scan: spinning instead of suspending on the MMA / epilogue barriers (build defines)
out=gpurun_out/${1:-r4v}; mkdir -p $out
for r in 1 2; do bash tools/quickbench.sh base_$r >> $out/ab.txt 2>&1; done
BKT_BUILD_DEFS="-DBKT_SPLIT_MMA_SPIN=1" python -m paper_1512_02831_b200.build > $out/build_mma.txt 2>&1
for r in 1 2; do bash tools/quickbench.sh mmaspin_$r >> $out/ab.txt 2>&1; done
BKT_BUILD_DEFS="-DBKT_SPLIT_EPI_SPIN=1" python -m paper_1512_02831_b200.build > $out/build_epi.txt 2>&1
for r in 1 2; do bash tools/quickbench.sh epispin_$r >> $out/ab.txt 2>&1; done
BKT_BUILD_DEFS="-DBKT_SPLIT_EPI_SPIN=1 -DBKT_SPLIT_MMA_SPIN=1" python -m paper_1512_02831_b200.build > $out/build_both.txt 2>&1
for r in 1 2; do bash tools/quickbench.sh bothspin_$r >> $out/ab.txt 2>&1; done
echo done
