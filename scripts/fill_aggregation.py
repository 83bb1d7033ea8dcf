"""Development aid (GPU box): how much a per-CTA aggregation of the v-major index fill by head
would save -- edges into the zone per distinct (chunk, head) pair for chunk sizes C."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from scripts.step import make  # noqa: E402

g = make(sys.argv[1] if len(sys.argv) > 1 else "rmat26")
og, _ = tcb.preprocess_device(g, rank_space=True)
g.free()
dst = og.edge_dst
n = og.node_offsets.size - 1
z0 = max(n - (1 << 20), 0)
e = np.nonzero(dst >= z0)[0]
v = dst[e].astype(np.uint64)
print("zone edges", e.size, flush=True)
for C in (1024, 4096, 16384):
    t = time.time()
    key = (e.astype(np.uint64) // C << np.uint64(21)) | (v - np.uint64(z0))
    u = np.unique(key).size
    print(C, "edges/distinct", round(e.size / u, 2), round(time.time() - t, 1), flush=True)
