"""Development aid (CPU, oracle-based): where the rank-space count kernels' bytes go.

For R-MAT scale S: rank-space CSR (relabel by (degree, id)), then for every oriented edge
(u, v) with u in a heavy class, the bytes the hub kernel reads for v (dense words, hub
suffix items, non-hub prefix items, 16-byte chunk aligned), plus per-v totals to see how
much an L2-resident (persisting) window of the hottest v data could save.
"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402

S = int(sys.argv[1])
HUB = 1 << int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 18
DENSE = HUB // 2
F = 3
pairs = oracle.symmetrize(oracle.rmat_pairs(S, 16, seed=0))
n = int(pairs.max()) + 1
deg = np.bincount(pairs[:, 0], minlength=n).astype(np.int64)
order = np.lexsort((np.arange(n), deg))
rank = np.empty(n, np.int64)
rank[order] = np.arange(n)
ru, rv = rank[pairs[:, 0]], rank[pairs[:, 1]]
keep = ru < rv
ru, rv = ru[keep], rv[keep]
o = np.lexsort((rv, ru))
src, dst = ru[o], rv[o]
m = src.size
outd = np.bincount(src, minlength=n)
off = np.zeros(n + 1, np.int64)
np.cumsum(outd, out=off[1:])
hz = max(n - HUB, 0)
vt = max(n - DENSE, 0)
hwords = (n - hz + 31) // 32 + 1
hwp = (hwords + 3) & ~3
# hubstart[v] = first position in adj(v) with rank >= hz
is_hub_item = dst >= hz
nonhub_cnt = np.bincount(src[~is_hub_item], minlength=n)
hubstart = off[:-1] + nonhub_cnt
du = outd[src]
cls = np.select([du <= 32, du <= 512, du <= 2048, du <= 16384], [-1, 0, 1, 2], 3)
v = dst
vs, ve, hv = off[v], off[v + 1], hubstart[v]
dws = ((v + 1 - hz) >> 5) & ~3
dense = (v >= vt) & ((hwp - dws) < F * (ve - vs))
nh_u = (hubstart[src] - off[src]) > 0


def chunk_bytes(a, b):
    a4 = a & ~3
    return np.where(b > a, ((b - a4 + 3) >> 2) * 16, 0)


b_dense = np.where(dense, (hwp - dws) * 4, 0)
b_hub = np.where(dense, 0, chunk_bytes(hv, ve))
b_non = np.where(dense | ~nh_u, 0, chunk_bytes(vs, hv))
res = {"scale": S, "n": n, "m": int(m), "hub_ranks": HUB, "max_out": int(outd.max())}
for c in (-1, 0, 1, 2, 3):
    sel = cls == c
    if not sel.any():
        continue
    res[f"class{c}"] = {
        "edges": int(sel.sum()), "sources": int(np.unique(src[sel]).size),
        "dense_GB": round(b_dense[sel].sum() / 1e9, 3), "hub_items_GB": round(b_hub[sel].sum() / 1e9, 3),
        "nonhub_items_GB": round(b_non[sel].sum() / 1e9, 3),
        "dense_edges": int(dense[sel].sum()),
    }
heavy = cls >= 0
tot = (b_dense + b_hub + b_non)[heavy]
per_v = np.bincount(v[heavy], weights=tot, minlength=n)
reads_v = np.bincount(v[heavy], minlength=n)
# footprint of v's data: dense bitmap (if ever dense) + list bytes
foot = np.where(per_v > 0, per_v / np.maximum(reads_v, 1), 0)
ratio = np.where(foot > 0, per_v / np.maximum(foot, 1), 0)  # = reads
idx = np.argsort(-ratio)
cf = np.cumsum(foot[idx])
cs = np.cumsum(per_v[idx] - foot[idx])
total = per_v.sum()
res["heavy_total_GB"] = round(total / 1e9, 3)
for mb in (16, 32, 64, 96):
    k = np.searchsorted(cf, mb * 2**20)
    res[f"pin_{mb}MB_saves_frac"] = round(float(cs[k - 1] / total) if k else 0.0, 4)
# contiguity: are the hottest v's high ranks?
res["hot_top_ranks_frac"] = round(float((idx[:1000] >= n - HUB).mean()), 3)
print(json.dumps(res, indent=1))
