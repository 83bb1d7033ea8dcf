"""Per-config device timings (development aid): fused preprocess+count on device pairs."""
import json
import math
import statistics
import sys

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import generators  # noqa: E402
from scripts import devopts  # noqa: E402

devopts.apply()


def run(name, dev, reps=5):
    tcb.count_with_timings_device(dev)
    ts = [tcb.count_with_timings_device(dev) for _ in range(reps)]
    tri = {t[0] for t in ts}
    pre = statistics.median(t[1].preprocess_ms for t in ts)
    cnt = statistics.median(t[1].count_ms for t in ts)
    hv = statistics.median(t[1].heavy_ms for t in ts)
    lt = statistics.median(t[1].light_ms for t in ts)
    vm = statistics.median(t[1].vmajor_ms for t in ts)
    m = dev.npairs // 2
    print(json.dumps({"config": name, "m": m, "triangles": sorted(tri), "preprocess_ms": round(pre, 3),
                      "count_ms": round(cnt, 3), "heavy_ms": round(hv, 3), "light_ms": round(lt, 3), "vmajor_ms": round(vm, 3), "edges_per_s": m / ((pre + cnt) / 1e3)}), flush=True)


which = sys.argv[1:] or ["rmat20", "ba1e7", "rmat22"]
for w in which:
    if w.startswith("rmat"):
        run(w, generators.rmat_device(int(w[4:]), 16, seed=0))
    elif w == "ba1e7":
        run(w, generators.barabasi_albert_device(10_000_000, 9, seed=0))
    elif w == "ba1e6":
        run(w, generators.barabasi_albert_device(1_000_000, 9, seed=0))
    elif w.startswith("rgg"):  # rgg2e7 -> n = 2*10^7, avg degree 32
        run(w, generators.random_geometric_device(int(float(w[3:])), 32.0, seed=0))
