"""Development aid: one fused preprocess+count step (count_with_timings on device pairs)."""
import sys

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import generators  # noqa: E402
from scripts import devopts  # noqa: E402

devopts.apply()

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
g = generators.rmat_device(scale, 16, seed=0)
for _ in range(reps):
    tri, t = tcb.count_with_timings_device(g)
    print(tri, {k: round(v, 3) for k, v in t.as_dict().items()})
