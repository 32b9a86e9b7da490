#!/bin/bash
# fine seam on device-resident slots: the seam / brute / CLI tests + full GPU suite
out=gpurun_out/${1:-r3v}; mkdir -p $out
timeout 1200 python -m pytest tests -m gpu -q > $out/pytest_gpu.txt 2>&1; echo "rc=$?" >> $out/pytest_gpu.txt
timeout 300 python -c "
import time, numpy as np, paper_1512_02831_b200 as bkt
rng = np.random.default_rng(1)
refs = rng.random((400000, 10), dtype=np.float32); q = rng.random((20000, 10), dtype=np.float32)
dev = bkt.device_init(bkt.DeviceSpec(cuda_device=0))
for nc in (1, 4, 8):
    t0 = time.perf_counter(); r = bkt.brute_knn(refs, q, bkt.SearchParams(k=10), device=dev, num_chunks=nc); t1 = time.perf_counter()
    print('brute num_chunks', nc, '%.1f ms' % (1e3 * (t1 - t0)), 'pairs/s %.3g' % (4e5 * 2e4 / (t1 - t0)))
" > $out/brute_timing.txt 2>&1
echo done
