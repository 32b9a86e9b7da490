BKT_BENCH_DEBUG=1 timeout 600 python bench.py --no-cpu 2>&1 | grep -E "e2e call|^\{" | cut -c1-120; timeout 300 python -m pytest tests -m gpu -q -k "pinned or pool" 2>&1 | tail -2
