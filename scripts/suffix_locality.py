"""Development aid (GPU): how concentrated are the v-major suffix streams in edge_dst?
v-major bytes by source window of the rank-space CSR (tc_shard_stats counter 8), sorted by
density: the fraction of all suffix bytes that the densest X MB of edge_dst would serve if
L2-resident (persisting window / blocked schedule candidates)."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import _lib  # noqa: E402
from scripts.step import make  # noqa: E402

g = make(sys.argv[1] if len(sys.argv) > 1 else "rmat26")
W = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
og, _ = tcb.preprocess_device(g, rank_space=True)
g.free()
h, m = og.device().handle, og.m_dir
b = np.linspace(0, m, W + 1).astype(np.int64)
out = np.zeros(9, np.uint64)
vb = np.zeros(W)
for i in range(W):
    _lib.check(_lib.lib().tc_shard_stats(h, int(b[i]), int(b[i + 1]), 0, 0, _lib.ptr(out)))
    vb[i] = float(out[8])
win_mb = 4.0 * (m / W) / 2**20
order = np.argsort(-vb)
cum = np.cumsum(vb[order]) / vb.sum()
res = {"windows": W, "window_MB": round(win_mb, 2), "total_vmajor_GB": round(vb.sum() / 1e9, 1)}
for mb in (32, 64, 96, 128, 256, 512, 1024):
    k = max(1, int(mb / win_mb))
    res[f"densest_{mb}MB"] = round(float(cum[min(k, W) - 1]), 3)
res["by_window_GB"] = [round(x / 1e9, 2) for x in vb[:: max(1, W // 64)]]
print(json.dumps(res))
