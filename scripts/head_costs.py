"""Development aid (GPU): v-major bytes and in-edges of single heads near the top of the
rank order vs the whole v-major side (is any head too big to be one shard's unit?)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import _lib  # noqa: E402
from scripts.step import make  # noqa: E402

g = make(sys.argv[1] if len(sys.argv) > 1 else "rmat26")
og, _ = tcb.preprocess_device(g, rank_space=True)
g.free()
h, n, m = og.device().handle, og.num_vertices, og.m_dir
out = np.zeros(9, np.uint64)
_lib.check(_lib.lib().tc_shard_stats(h, 0, 0, 0, n, _lib.ptr(out)))
tot_b, tot_e = int(out[5] + out[6]), int(out[7])
print("total v-major bytes", tot_b / 1e9, "GB, in-edges", tot_e)
rows = []
for lo, hi in [(n - 2 ** k, n - 2 ** (k - 1)) for k in range(22, 0, -1)] + [(n - 1, n)]:
    _lib.check(_lib.lib().tc_shard_stats(h, 0, 0, lo, hi, _lib.ptr(out)))
    rows.append((n - lo, int(out[5] + out[6]), int(out[7])))
    print(f"top heads [{n - lo:>8}..{n - hi:>8}): {rows[-1][1] / tot_b:7.4f} of v-major bytes, "
          f"{rows[-1][2] / tot_e:7.4f} of in-edges", flush=True)
for k in range(1, 9):
    _lib.check(_lib.lib().tc_shard_stats(h, 0, 0, n - k, n - k + 1, _lib.ptr(out)))
    print(f"head rank n-{k}: {int(out[5] + out[6]) / tot_b:.4f} of bytes, in-edges {int(out[7])}")
