"""Development aid: share of count items (w in adj(v), once per in-edge of v) whose
degree rank is in the top K (the hub zone), and the heavy/light split of those items."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import generators  # noqa: E402

scale = int(sys.argv[1])
g = generators.rmat_device(scale, 16, seed=0)
og, _ = tcb.preprocess_device(g)
g.free()
src, dst, off = og.edge_src, og.edge_dst, og.node_offsets
n = off.size - 1
outd = np.diff(off)
indeg = np.bincount(dst, minlength=n)
deg = outd + indeg
order = np.lexsort((np.arange(n), deg))
rank = np.empty(n, np.int64)
rank[order] = np.arange(n)
mult = indeg[src].astype(np.int64)  # adjacency entry (v -> w) is an item once per in-edge of v
tot = int(mult.sum())
rw = rank[dst]
out = {"scale": scale, "n": int(n), "items": tot, "top_k_item_share": {}}
for k in (1 << 14, 1 << 15, 1 << 16, 1 << 17, 1 << 18, 1 << 19, 1 << 20):
    out["top_k_item_share"][k] = round(float(mult[rw >= n - k].sum() / tot), 5)
# adjacency entries per source in the hub zone (bitmap fill) for heavy sources
print(json.dumps(out, indent=1))
