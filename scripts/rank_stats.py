"""Development aid: degree-rank statistics of the oriented R-MAT CSR (bitmap feasibility)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import generators  # noqa: E402

scale = int(sys.argv[1])
t = time.time()
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
du = outd[src]
dv = outd[dst].astype(np.int64)
span = n - 1 - rank[src]
tot = int(dv.sum())
out = {"scale": scale, "n": int(n), "m": int(dst.size), "items": tot, "max_out": int(outd.max())}
cov = {}
for kb in (8, 16, 32, 64, 96, 128, 160, 192, 224):
    sel = span <= kb * 8192
    heavy = du > 32
    cov[kb] = [round(float(dv[sel].sum() / tot), 4),
               round(float(dv[sel & heavy].sum() / max(dv[heavy].sum(), 1)), 4)]
out["bitmap_cover_items_all_heavy"] = cov
cls = {}
for lo, hi in ((1, 8), (9, 32), (33, 128), (129, 512), (513, 2048), (2049, 1 << 30)):
    sel = (du >= lo) & (du <= hi)
    cls[f"{lo}-{hi}"] = [round(float(dv[sel].sum() / tot), 4), round(float(sel.mean()), 4)]
out["items_edges_by_du"] = cls
# dense core: edges with both endpoints among the top-K ranks
rs, rd = rank[src], rank[dst]
core = {}
for K in (1 << 14, 1 << 15, 1 << 16, 1 << 17):
    sel = (rs >= n - K) & (rd >= n - K)
    words = ((n - 1 - rd[sel]) // 32 + 1).sum()
    core[K] = {"edge_frac": round(float(sel.mean()), 4), "item_frac": round(float(dv[sel].sum() / tot), 4),
               "and_words_vs_items": round(float(words / max(dv[sel].sum(), 1)), 4)}
out["core"] = core
out["secs"] = time.time() - t
print(json.dumps(out, indent=1))
