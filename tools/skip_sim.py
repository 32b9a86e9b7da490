"""Driver for tools/skip_sim.c (design experiment): writes the config-2 tree
and a query sample, runs the simulation.  python tools/skip_sim.py [m] [k]"""
import subprocess, sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import oracle as O
from paper_1512_02831_b200.datasets import gen_mixture

m = int(float(sys.argv[1])) if len(sys.argv) > 1 else 200_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 10
n, h, d = 2_000_000, 9, 10
tmp = Path("/tmp/sim"); tmp.mkdir(exist_ok=True)
pts, _ = gen_mixture(n + m, d, seed=1)
refs = np.ascontiguousarray(pts.data[:n]); q = np.ascontiguousarray(pts.data[n:n + m])
t = O.build_tree(refs, h)
with open(tmp / "tree.bin", "wb") as f:
    np.array([h, d], np.int32).tofile(f); np.array([n], np.int64).tofile(f)
    np.asarray(t.split_values, np.float32).tofile(f); np.asarray(t.points, np.float32).tofile(f)
    np.asarray(t.original_index, np.int64).tofile(f); np.asarray(t.leaf_starts, np.int64).tofile(f)
with open(tmp / "q.bin", "wb") as f:
    np.array([m], np.int64).tofile(f); q.tofile(f)
exe = tmp / "skip_sim"
subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-pthread", "-o", str(exe), str(ROOT / "tools/skip_sim.c"), "-lm"], check=True)
subprocess.run([str(exe), str(tmp / "tree.bin"), str(tmp / "q.bin"), "120", "8", str(k)], check=True)
