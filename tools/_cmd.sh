for r in 1 2; do
bash tools/quickbench.sh base$r BKT_LIB_NAME=libbkt_base.so
bash tools/quickbench.sh early$r
done
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
