"""Development aid (GPU box): median rank-space preprocess time (no count) of a config,
e.g. for diagnostic library variants whose index would not be countable:
    TC_LIB_PATH=variants/lib_x.so python scripts/pre_probe.py rmat26 5"""
import statistics
import sys

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from scripts.step import make  # noqa: E402

g = make(sys.argv[1])
ms = []
for _ in range(int(sys.argv[2]) + 1):
    og, t = tcb.preprocess_device(g, rank_space=True)
    ms.append(t.preprocess_ms)
    del og
print(sys.argv[1], "preprocess_ms median", round(statistics.median(ms[1:]), 3), [round(x, 2) for x in ms], flush=True)
