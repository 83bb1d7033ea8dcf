"""Development aid (GPU): per-shard count time of the work-balanced edge ranges on one GPU
(the multi-GPU schedule's load balance, measured serially): python scripts/shard_balance.py CFG P"""
import json
import statistics
import sys

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import _lib  # noqa: E402
from scripts import devopts  # noqa: E402

devopts.apply()
from scripts.step import make  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "rmat26"
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8
g = make(cfg)
og, _ = tcb.preprocess_device(g, rank_space=True)
g.free()
from paper_1503_00576_b200.count import count_shard, shard_plan  # noqa: E402

from paper_1503_00576_b200.distributed import ShardPlanner  # noqa: E402

planner = ShardPlanner.from_device(og.device(), P)
eb, hb = planner.bounds()
full = statistics.median(tcb.count_device(og)[1].count_ms for _ in range(3))
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 0
for it in range(iters + 1):
    times, tris, phases, edge_ms, head_ms = [], 0, [], [], []
    for p in range(P):
        args = (og, eb[p], eb[p + 1], hb[p], hb[p + 1])
        with _lib.options(count_stats=1):
            count_shard(*args)
            ts = [count_shard(*args) for _ in range(3)]
        tris += ts[0][0]
        times.append(statistics.median(t[1].count_ms for t in ts))
        vm = statistics.median(t[1].vmajor_ms for t in ts)
        rest = statistics.median(t[1].count_ms - t[1].vmajor_ms for t in ts)
        phases.append([round(vm, 2), round(rest, 2)])
        head_ms.append(vm)
        edge_ms.append(rest)
    print(json.dumps({"config": cfg, "P": P, "refinement": it, "full_ms": round(full, 2),
                      "shard_ms": [round(t, 2) for t in times],
                      "max_over_mean": round(max(times) / statistics.mean(times), 3),
                      "speedup_bound": round(full / max(times), 2), "sum_over_full": round(sum(times) / full, 3),
                      "triangles": tris, "phases_head_edge": phases, "edge_bounds": [int(x) for x in eb],
                      "head_bounds": [int(x) for x in hb]}), flush=True)
    eb, hb = planner.refine(edge_ms, head_ms)
