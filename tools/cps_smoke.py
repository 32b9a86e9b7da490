"""Small exactness check of one TC variant (run with BKT_TC_CPS / BKT_TC_N set)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1512_02831_b200 as bkt  # noqa: E402
from oracle import oracle as O  # noqa: E402

rng = np.random.default_rng(1)
refs = rng.random((50000, 10), dtype=np.float32)
q = rng.random((20000, 10), dtype=np.float32)
tree = bkt.build_buffer_tree(refs, 7)
res = bkt.lazy_search(tree, q, bkt.SearchParams(k=10))
want = O.knn_tree(O.build_tree(refs, 7), q, 10, threads=8)
print("exact:", np.array_equal(res.keys, want["keys"]))
