for r in 1 2; do
bash tools/quickbench.sh base_nospin$r BKT_LIB_NAME=libbkt_base.so BKT_TC_SPIN=0
bash tools/quickbench.sh gmin$r
done
bash tools/quickbench.sh gmin_spin1 BKT_TC_SPIN=1
bash tools/quickbench.sh gmin_spin2 BKT_TC_SPIN=2
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
