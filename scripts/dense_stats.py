"""Development aid: share of items on edges (u, v) whose v ranks in the top T, and the
cost of the word-parallel alternative (bitmap AND over v's rank span, or testing each
element of adj(u) against v's bitmap)."""
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
deg = outd + np.bincount(dst, minlength=n)
order = np.lexsort((np.arange(n), deg))
rank = np.empty(n, np.int64)
rank[order] = np.arange(n)
rv = rank[dst]
dv = outd[dst].astype(np.int64)
du = outd[src].astype(np.int64)
tot = int(dv.sum())
res = {"scale": scale, "n": int(n), "items": tot}
for T in (1 << 12, 1 << 14, 1 << 15, 1 << 16):
    sel = rv >= n - T
    words = (n - 1 - rv[sel]) // 32 + 1
    best = np.minimum(np.minimum(words, du[sel]), dv[sel])
    res[T] = {"edge_share": round(float(sel.mean()), 4),
              "item_share": round(float(dv[sel].sum() / tot), 4),
              "and_words_over_items": round(float(words.sum() / max(dv[sel].sum(), 1)), 4),
              "min(words,du,dv)_over_items": round(float(best.sum() / max(dv[sel].sum(), 1)), 4),
              "bitmap_MB": round(float(T * T / 64 * 4 / 2**20), 1)}
print(json.dumps(res, indent=1))
