for r in 1 2; do
bash tools/quickbench.sh base$r BKT_LIB_NAME=libbkt_base.so
bash tools/quickbench.sh qv$r
done
timeout 600 python -m pytest tests -m gpu -x -q -k "golden or tensor_core or config2 or mixture" 2>&1 | tail -2
