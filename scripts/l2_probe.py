"""Development aid: count time at scale S with the current env (TC_L2_PERSIST_MB etc.)."""
import os
import statistics
import sys

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import generators  # noqa: E402
from scripts import devopts  # noqa: E402

devopts.apply()

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
g = generators.rmat_device(scale, 16, seed=0)
ts = []
for _ in range(reps):
    tri, t = tcb.count_with_timings_device(g)
    ts.append(t)
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("TC_"))
print(f"[{tag}] s{scale} tri={tri} pre={statistics.median(x.preprocess_ms for x in ts):.1f} "
      f"count={statistics.median(x.count_ms for x in ts):.1f} heavy={statistics.median(x.heavy_ms for x in ts):.1f} "
      f"light={statistics.median(x.light_ms for x in ts):.1f}", flush=True)
