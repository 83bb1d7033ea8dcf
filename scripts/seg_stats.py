"""Development aid (GPU box): rank-space out-list sizes by segmented-sort class (lists,
elements, and padded elements of the power-of-two bitonic networks)."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import generators  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 26
g = generators.rmat_device(S, 16, seed=0)
og, _ = tcb.preprocess_device(g, rank_space=True)
g.free()
d = np.diff(og.node_offsets)
res = {}
edges = [0, 1, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 1 << 40]
for lo, hi in zip(edges[:-1], edges[1:]):
    b = (d > lo) & (d <= hi)
    p2 = np.where(d[b] > 0, 1 << np.ceil(np.log2(np.maximum(d[b], 1))).astype(np.int64), 0)
    res[f"{lo + 1}-{hi}"] = {"lists": int(b.sum()), "elements": int(d[b].sum()), "pow2_padded": int(p2.sum())}
print(json.dumps(res))
