"""Development aid (GPU): per-shard count times beside the shard's schedule bytes by class,
for several partitions of the R-MAT rank-space CSR -- the data the rank-space shard cost
model is fitted to.  python scripts/shard_calib.py CFG > gpurun_out/shard_calib.jsonl"""
import ctypes
import json
import statistics
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import _lib  # noqa: E402
from scripts import devopts  # noqa: E402

devopts.apply()
from scripts.step import make  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "rmat26"
g = make(cfg)
og, _ = tcb.preprocess_device(g, rank_space=True)
g.free()
m = og.m_dir
h = og.device().handle
src = og.edge_src  # host copy for per-shard source counts
plans = {"even16": np.linspace(0, m, 17).astype(np.int64),
         "model0_16": np.array(tcb.PartitionPlan.work_balanced(og, 16).bounds, np.int64),
         "even8": np.linspace(0, m, 9).astype(np.int64)}
for name, b in plans.items():
    for p in range(len(b) - 1):
        lo, hi = int(b[p]), int(b[p + 1])
        out = np.zeros(5, np.uint64)
        _lib.check(_lib.lib().tc_schedule_bytes_range(h, lo, hi, _lib.ptr(out)))
        with _lib.options(count_stats=1):
            tcb.count_device(og, lo, hi)
            ts = [tcb.count_device(og, lo, hi)[1] for _ in range(3)]
        rec = {"plan": name, "p": p, "lo": lo, "hi": hi, "edges": hi - lo,
               "sources": int(src[hi - 1]) - int(src[lo]) + 1,
               "bytes": [int(x) for x in out],
               "ms": statistics.median(t.count_ms for t in ts),
               "vmajor_ms": statistics.median(t.vmajor_ms for t in ts),
               "heavy_ms": statistics.median(t.heavy_ms for t in ts),
               "light_ms": statistics.median(t.light_ms for t in ts)}
        print(json.dumps(rec), flush=True)
