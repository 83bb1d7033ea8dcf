"""Quick device timing probe (development aid): generate rmat(scale) on the device,
preprocess + count a few times, print event timings."""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import _lib, generators  # noqa: E402
from scripts import devopts  # noqa: E402

devopts.apply()

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
t0 = time.time()
g = generators.rmat_device(scale, 16, seed=0)
gen_s = time.time() - t0
out = {"scale": scale, "npairs": g.npairs, "n": g.num_vertices, "gen_s": gen_s}
for r in range(reps):
    og, tp = tcb.preprocess_device(g)
    tri, tc = tcb.count_device(og)
    out[f"rep{r}"] = {"pre_ms": tp.preprocess_ms, "count": tc.as_dict(), "tri": tri}
tri_m, tm = tcb.count_device(og, algo=_lib.ALGO_MERGE_THREAD)
out["merge_thread"] = {"tri": tri_m, "ms": tm.count_ms}
out["W"] = tcb.merge_work(og)
out["max_out"] = og.device().max_out
print(json.dumps(out, indent=1))
