timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python tools/finish_sweep.py --at=-1,default
