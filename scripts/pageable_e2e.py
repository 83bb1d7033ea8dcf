"""Development aid: count_with_timings end to end from pinned vs pageable host pairs
(R-MAT scale S), wall clock per call."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import generators  # noqa: E402
from paper_1503_00576_b200.graph import EdgeArray  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 26
d = generators.rmat_device(S, 16, seed=0)
pinned = d.to_host(pinned=True)
d.free()
pageable = EdgeArray(np.array(pinned.edges), num_vertices=pinned.num_vertices)
for name, g in (("pinned", pinned), ("pageable", pageable)):
    for rep in range(3):
        t0 = time.perf_counter()
        tri, t = tcb.count_with_timings(g)
        print(f"{name} rep {rep}: wall {1e3 * (time.perf_counter() - t0):.1f} ms, pre(incl h2d) "
              f"{t.preprocess_ms:.1f}, count {t.count_ms:.1f}, tri {tri}", flush=True)
