"""Development aid (GPU): per-shard cost features (tc_shard_stats) beside the measured
per-phase times of tc_count_shard, over several shard plans of the R-MAT rank-space CSR --
the data the shard plan's class weights are fitted to.
    python scripts/shard_calib.py rmat26 > gpurun_out/shard_calib.jsonl"""
import json
import statistics
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import _lib  # noqa: E402
from paper_1503_00576_b200.count import count_shard, shard_plan  # noqa: E402
from scripts import devopts  # noqa: E402

devopts.apply()
from scripts.step import make  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "rmat26"
g = make(cfg)
og, _ = tcb.preprocess_device(g, rank_space=True)
g.free()
h = og.device().handle
plans = []
for P, wl, wv, we in ((8, 16, 6, 0), (8, 32, 4, 64), (8, 4, 8, 256), (4, 16, 4, 64), (16, 8, 4, 0)):
    with _lib.options(shard_wlight=wl, shard_wvlow4=wv, shard_wvedge=we):
        plans.append((f"P{P}_wl{wl}_wv{wv}_we{we}",) + shard_plan(og, P))
for name, eb, hb in plans:
    for p in range(len(eb) - 1):
        a = (og, eb[p], eb[p + 1], hb[p], hb[p + 1])
        out = np.zeros(9, np.uint64)
        _lib.check(_lib.lib().tc_shard_stats(h, int(eb[p]), int(eb[p + 1]), int(hb[p]), int(hb[p + 1]),
                                             _lib.ptr(out)))
        with _lib.options(count_stats=1):
            count_shard(*a)
            ts = [count_shard(*a)[1] for _ in range(3)]
        rec = {"plan": name, "p": p, "stats": [int(x) for x in out],
               "ms": statistics.median(t.count_ms for t in ts),
               "vmajor_ms": statistics.median(t.vmajor_ms for t in ts),
               "heavy_ms": statistics.median(t.heavy_ms for t in ts),
               "light_ms": statistics.median(t.light_ms for t in ts),
               "classify_ms": statistics.median(t.classify_ms for t in ts)}
        print(json.dumps(rec), flush=True)
