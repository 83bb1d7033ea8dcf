"""Development aid (GPU box): where do the v-major suffix items of the hub heads come from?
Splits the suffix items of the edges the per-edge choice sends v-major (heavy sources, heads
in the hub zone) by head band n - v <= 2^k: a head in the top 2^16 ranks has every suffix
item in the top 2^16 too (16-bit offsets suffice)."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import generators  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 26
HUB, DENSE, F = 1 << 18, 1 << 17, 3
g = generators.rmat_device(S, 16, seed=0)
og, _ = tcb.preprocess_device(g, rank_space=True)
g.free()
src = og.edge_src
dst = og.edge_dst.astype(np.int64)
off = og.node_offsets
n, m = off.size - 1, dst.size
outd = np.diff(off)
hz = max(n - HUB, 0)
vt = max(n - DENSE, 0)
hwp = (((n - hz + 31) // 32) + 3) & ~3
e = np.arange(m, dtype=np.int64)
eu = off[1:][src]
suffix = eu - e - 1
du = outd[src]
del src, e
sel = (dst >= hz) & (du > 32) & (suffix > 0)
d, sfx = dst[sel], suffix[sel]
vs, ve = off[d], off[d + 1]
lb = ve - vs
dws = ((d + 1 - hz) >> 5) & ~3
dense = (d >= vt) & ((hwp - dws) < F * lb)
umaj = np.where(dense, (hwp - dws) * 4, np.where(lb > 0, ((ve - (vs & ~3) + 3) >> 2) * 16, 0))
pick = (4 * sfx + 8) < umaj
d, sfx = d[pick], sfx[pick]
top = n - d
res = {"scale": S, "n": int(n), "m": int(m), "vmajor_hub_edges": int(d.size),
       "vmajor_hub_items": int(sfx.sum()), "bands": {}}
prev = 0
for k in range(10, 19):
    b = (top > prev) & (top <= (1 << k))
    res["bands"][f"top_2^{k}"] = {"edges": int(b.sum()), "items": int(sfx[b].sum()),
                                  "items_frac": round(float(sfx[b].sum() / max(1, sfx.sum())), 4),
                                  "heads": int(np.unique(d[b]).size)}
    prev = 1 << k
print(json.dumps(res))
