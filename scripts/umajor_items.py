"""Development aid (GPU box): where the u-major item work of heavy sources goes at R-MAT
scale S, by head class (vectorised numpy, no sorts)."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from scripts.step import make  # noqa: E402

g = make(sys.argv[1] if len(sys.argv) > 1 else "rmat26")
og, _ = tcb.preprocess_device(g, rank_space=True)
g.free()
src = og.edge_src
dst = og.edge_dst
off = og.node_offsets
n = off.size - 1
outd = np.diff(off).astype(np.int64)
hz = max(n - (1 << 18), 0)
z0 = max(n - (1 << 20), 0)
du = outd[src]
dv = outd[dst]
e = np.arange(dst.size, dtype=np.int64)
suffix = off[1:][src] - e - 1
res = {"n": int(n), "m": int(dst.size)}
for name, sel in (("class0", (du > 32) & (du <= 512)), ("class1", (du > 512) & (du <= 2048)),
                  ("light", du <= 32)):
    below = sel & (dst < z0)
    lowbig = sel & (dst >= z0) & (dst < hz) & (dv > 512)
    res[name] = {"edges": int(sel.sum()),
                 "below_zone_edges": int(below.sum()), "below_zone_items": int(dv[below].sum()),
                 "below_zone_suffix": int(suffix[below].sum()),
                 "lowzone_big_edges": int(lowbig.sum()), "lowzone_big_items": int(dv[lowbig].sum()),
                 "lowzone_big_suffix": int(suffix[lowbig].sum())}
print(json.dumps(res, indent=1))
