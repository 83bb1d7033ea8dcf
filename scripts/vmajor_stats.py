"""Development aid (GPU box): cost of a v-major schedule for hub heads at R-MAT scale S.

For every oriented edge e = (u, v) with v in the hub zone (top 2^18 ranks), a v-major
kernel stages adj(v) as a shared-memory bitmap and streams the suffix of adj(u) after v
(off[u+1] - e - 1 items).  Compare its bytes with the current u-major costs."""
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
del src
inH = dst >= hz
res = {"scale": S, "n": int(n), "m": int(m), "edges_vH": int(inH.sum())}
vs, ve = off[dst], off[dst + 1]
lb = ve - vs
dws = ((dst + 1 - hz) >> 5) & ~3
dense = (dst >= vt) & ((hwp - dws) < F * lb)
and_b = np.where(dense, (hwp - dws) * 4, 0)
for name, sel in (("heavy_u", du > 32), ("light_u", du <= 32)):
    s2 = sel & inH
    res[name] = {
        "edges_vH": int(s2.sum()),
        "suffix_items_vH": int(suffix[s2].sum()),
        "suffix_GB": round(4 * suffix[s2].sum() / 1e9, 2),
        "v_items_vH_GB": round(4 * lb[s2].sum() / 1e9, 2),
        "dense_and_GB": round(and_b[s2].sum() / 1e9, 2),
        "distinct_v": int(np.unique(dst[s2]).size),
    }
# per-edge choice: v-major (4 * suffix) vs u-major (dense AND words or chunked items)
items_b = np.where(lb > 0, ((ve - (vs & ~3) + 3) >> 2) * 16, 0)
umaj = np.where(dense, and_b, items_b)
vmaj = 4 * suffix + 8
for name, sel in (("heavy_u", du > 32), ("light_u", du <= 32)):
    s2 = sel & inH
    pick_v = s2 & (vmaj < umaj)
    res[name]["choice_vmajor_edges"] = int(pick_v.sum())
    res[name]["choice_vmajor_GB"] = round(vmaj[pick_v].sum() / 1e9, 2)
    res[name]["choice_umajor_GB"] = round(umaj[s2 & ~pick_v].sum() / 1e9, 2)
    res[name]["umajor_all_GB"] = round(umaj[s2].sum() / 1e9, 2)
    for f in (2, 4, 8):
        pv = s2 & (vmaj * f < umaj)
        res[name][f"choice_f{f}_vmajor_GB"] = round(vmaj[pv].sum() / 1e9, 2)
        res[name][f"choice_f{f}_umajor_GB"] = round(umaj[s2 & ~pv].sum() / 1e9, 2)
        res[name][f"choice_f{f}_vmajor_edges"] = int(pv.sum())
# per-v in-degree within H (for CTA sizing) and bitmap words
vv = dst[inH]
indeg = np.bincount(vv - hz, minlength=n - hz)
res["indeg_vH"] = {"max": int(indeg.max()), "mean": float(indeg.mean()),
                   "p99": float(np.percentile(indeg, 99))}
res["adjH_edges"] = int((off[n] - off[hz]))
# suffix bytes by v bucket
vb = np.floor(np.log2(n - dst[inH])).astype(np.int64)
sf = suffix[inH]
res["suffix_GB_by_vdist"] = {int(b): round(4 * sf[vb == b].sum() / 1e9, 2) for b in np.unique(vb)}
print(json.dumps(res, indent=1), flush=True)
