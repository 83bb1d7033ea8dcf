"""Development aid (GPU box): per-call wall time vs the library's event time for a small
graph (ER 10^4 / 10^5, BASELINE configs[0]) -- the fixed host-side cost of one call."""
import math
import sys
import time

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import _lib, generators  # noqa: E402

g = generators.gnp(10_000, 100_000 / math.comb(10_000, 2), seed=0)
d = generators.to_device(g)
gp = d.to_host(pinned=True)
for name, arr in (("pageable", g), ("pinned", gp)):
    walls, evs = [], []
    for _ in range(12):
        t0 = time.perf_counter()
        tri, t = tcb.count_with_timings(arr)
        walls.append(1e3 * (time.perf_counter() - t0))
        evs.append(t.total_ms)
    print(name, tri, "wall ms", [round(x, 2) for x in walls[2:]], "event total ms", [round(x, 2) for x in evs[2:]])
t0 = time.perf_counter()
for _ in range(10):
    tcb.count_with_timings_device(d)
print("device-resident wall ms/call", round(100 * (time.perf_counter() - t0), 2))
