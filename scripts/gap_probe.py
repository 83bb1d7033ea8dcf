"""Development aid: does holding an extra preprocessed graph slow the fused step?"""
import sys
import time

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import generators  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
g = generators.rmat_device(scale, 16, seed=0)
for i in range(2):
    t0 = time.time(); tri, t = tcb.count_with_timings_device(g)
    print("plain", i, round(t.preprocess_ms, 1), round(t.count_ms, 1), round((time.time() - t0) * 1e3, 1), flush=True)
og, _ = tcb.preprocess_device(g)
W = tcb.merge_work(og)
for i in range(3):
    t0 = time.time(); tri, t = tcb.count_with_timings_device(g)
    print("with og", i, round(t.preprocess_ms, 1), round(t.count_ms, 1), round((time.time() - t0) * 1e3, 1), flush=True)
del og
import gc; gc.collect()
for i in range(2):
    t0 = time.time(); tri, t = tcb.count_with_timings_device(g)
    print("og freed", i, round(t.preprocess_ms, 1), round(t.count_ms, 1), round((time.time() - t0) * 1e3, 1), flush=True)
