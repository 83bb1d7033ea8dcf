import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb
from scripts.step import make
for cfg in sys.argv[1:]:
    g = make(cfg)
    og, _ = tcb.preprocess_device(g, rank_space=True)
    g.free()
    src, dst = og.edge_src, og.edge_dst
    same = (src[1:] == src[:-1])
    dup = same & (dst[1:] == dst[:-1])
    unsorted = same & (dst[1:] < dst[:-1])
    print(cfg, "m", src.size, "dups", int(dup.sum()), "unsorted", int(unsorted.sum()), flush=True)
