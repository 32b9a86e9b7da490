python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 1 2; do
bash tools/quickbench.sh base$r BKT_LIB_NAME=libbkt_base.so
bash tools/quickbench.sh rank$r
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rank.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_rank.csv
