"""Config 1 per-round trace (BKT_TRACE_ROUNDS=1 prints active queries and
leaf-scan ms per round of the last search to stderr)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1512_02831_b200 as bkt

refs, queries = bkt.datasets.config_inputs(1)
tree = bkt.build_buffer_tree(refs, 8)
dev = bkt.device_init(bkt.DeviceSpec(cuda_device=0))
dev.ensure_tree(tree)
dev.search(queries, 10)
keys, st, _ = dev.search(queries, 10, timing=True)
print(json.dumps({k: v for k, v in st.items() if isinstance(v, (int, float))}))
dev.close()
