#!/bin/bash
# round-2: split rounds -- parity, then split on/off bench
out=gpurun_out/${1:-r2d}; mkdir -p $out
python -m paper_1512_02831_b200.build > $out/build.txt 2>&1
timeout 300 python -c "
import numpy as np, paper_1512_02831_b200 as bkt
from oracle import oracle as O
rng=np.random.default_rng(3)
refs=rng.random((200000,10),dtype=np.float32); q=rng.random((20000,10),dtype=np.float32)
t=bkt.build_buffer_tree(refs,7); ot=O.build_tree(refs,7)
st=bkt.SearchStats()
r=bkt.lazy_search(t,q,bkt.SearchParams(k=10),stats=st)
w=O.knn_tree(ot,q,10,threads=8)
print('keys equal', np.array_equal(r.keys,w['keys']), 'visited equal', np.array_equal(st.visited_per_query,w['visited'].astype(np.int64)), 'pairs', st.pairs, w['pairs'], 'events', st.leaf_scan_events, int(w['visited'].sum()))
" > $out/quick.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_scale_parity.py tests/test_gpu_parity.py -m gpu -x -q > $out/pytest.txt 2>&1; echo "rc=$?" >> $out/pytest.txt
for r in 1 2; do
  bash tools/quickbench.sh split_$r >> $out/ab.txt
  bash tools/quickbench.sh nosplit_$r BKT_SPLIT=0 >> $out/ab.txt
done
BKT_TRACE_ROUNDS=1 timeout 300 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --check-rows 0 > /dev/null 2> $out/trace_split.err
echo done
