#!/bin/bash
# ab.sh LIB_A LIB_B [reps]: alternate short bench runs of two builds of
# libbkt (paper_1512_02831_b200/_lib/<name>) on the same box
a=$1; b=$2; reps=${3:-2}
for r in $(seq $reps); do
  for lib in $a $b; do
    bash tools/quickbench.sh ${lib%.so}_$r BKT_LIB_NAME=$lib
  done
done
