"""Development aid (GPU box): where the heavy (hub) count kernel's bytes go at R-MAT scale S.

Rank-space CSR from the device, then for every oriented edge (u, v) with a heavy source
(d+(u) > 32) the bytes k_count_hub reads for v (dense bitmap words or 16-byte item
chunks), grouped by the rank distance of v (and of u) from the top, with the footprint of
the distinct v data in each group -- reuse = bytes / footprint tells how much an
L2-blocked schedule could save."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import generators  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 26
HUB, DENSE, F = 1 << 18, 1 << 17, 3
t0 = time.time()
g = generators.rmat_device(S, 16, seed=0)
og, _ = tcb.preprocess_device(g, rank_space=True)
g.free()
src = og.edge_src.astype(np.int64)
dst = og.edge_dst.astype(np.int64)
off = og.node_offsets
n, m = off.size - 1, src.size
print("csr", n, m, round(time.time() - t0, 1), flush=True)
outd = np.diff(off)
hz = max(n - HUB, 0)
vt = max(n - DENSE, 0)
hwp = (((n - hz + 31) // 32) + 3) & ~3
nonhub = np.bincount(src[dst < hz], minlength=n)
hubstart = off[:-1] + nonhub
du = outd[src]
heavy = du > 32
hs, hd = src[heavy], dst[heavy]
del src
vs, ve, hv = off[hd], off[hd + 1], hubstart[hd]
dws = ((hd + 1 - hz) >> 5) & ~3
dense = (hd >= vt) & ((hwp - dws) < F * (ve - vs))


def chunk_bytes(a, b):
    return np.where(b > a, ((b - (a & ~3) + 3) >> 2) * 16, 0)


nh_u = nonhub[hs] > 0
cost = np.where(dense, (hwp - dws) * 4, chunk_bytes(hv, ve) + np.where(nh_u, chunk_bytes(vs, hv), 0))
print("costs", round(time.time() - t0, 1), flush=True)
res = {"scale": S, "n": int(n), "m": int(m), "heavy_edges": int(heavy.sum()),
       "heavy_bytes_GB": round(cost.sum() / 1e9, 2), "dense_edges": int(dense.sum()),
       "dense_bytes_GB": round(cost[dense].sum() / 1e9, 2)}
# per-v cost of a dense read / sparse read (footprint)
vb = np.floor(np.log2(n - hd)).astype(np.int64)
ub = np.floor(np.log2(n - hs)).astype(np.int64)
rows = []
for b in range(int(vb.max()) + 1):
    sel = vb == b
    if not sel.any():
        continue
    vv, first = np.unique(hd[sel], return_index=True)
    foot = cost[sel][first].sum()  # dense/sparse choice is per v: first edge's cost ~ per-v
    rows.append({"v_dist_log2": b, "edges": int(sel.sum()), "distinct_v": int(vv.size),
                 "bytes_GB": round(cost[sel].sum() / 1e9, 3), "footprint_MB": round(foot / 2**20, 2),
                 "dense_frac": round(float(dense[sel].mean()), 3)})
res["by_v"] = rows
rows = []
for b in range(int(ub.max()) + 1):
    sel = ub == b
    if not sel.any():
        continue
    rows.append({"u_dist_log2": b, "edges": int(sel.sum()), "sources": int(np.unique(hs[sel]).size),
                 "bytes_GB": round(cost[sel].sum() / 1e9, 3)})
res["by_u"] = rows
for K in (12, 13, 14, 15, 16):
    c0 = n - (1 << K)
    sel = hs >= c0
    res[f"u_in_top2^{K}_bytes_GB"] = round(cost[sel].sum() / 1e9, 3)
    res[f"core2^{K}_edges"] = int(((dst >= c0) & (og.edge_src >= c0)).sum())
print(json.dumps(res, indent=1), flush=True)
