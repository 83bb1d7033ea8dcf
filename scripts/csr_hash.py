"""Development aid: sha256 of the rank-space CSR (src|dst|offsets) for a few configs, to
compare preprocessing variants (e.g. TC_BUCKET=0 vs 1) byte for byte."""
import hashlib
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from scripts import devopts  # noqa: E402

devopts.apply()
from scripts.step import make  # noqa: E402

for cfg in sys.argv[1:]:
    g = make(cfg)
    og, _ = tcb.preprocess_device(g, rank_space=True)
    h = hashlib.sha256()
    for a in (og.edge_src, og.edge_dst, og.node_offsets):
        h.update(np.ascontiguousarray(a).tobytes())
    print(cfg, og.m_dir, h.hexdigest()[:16], flush=True)
    g.free()
