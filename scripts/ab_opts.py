"""Development aid (GPU box): A/B of schedule options on one workload in one process.

    python scripts/ab_opts.py rmat26 6 "" "vin_overlap=0" "seg_k16=0,vin_grid=4"

Each option set (comma-separated name=value; "" = defaults) runs `reps` fused
count_with_timings steps on the same device edge array; prints the median phase times
and checks every count equals the first one."""
import json
import statistics
import sys

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import _lib  # noqa: E402
from scripts.step import make  # noqa: E402

g = make(sys.argv[1])
reps = int(sys.argv[2])
want = None
for spec in sys.argv[3:] or [""]:
    kv = dict(x.split("=") for x in spec.split(",") if x)
    with _lib.options(**{k: int(v) for k, v in kv.items()}):
        rows = []
        for _ in range(reps + 1):
            tri, t = tcb.count_with_timings_device(g)
            want = tri if want is None else want
            if tri != want:
                raise SystemExit(f"{spec}: count {tri} != {want}")
            rows.append(t.as_dict())
        rows = rows[1:]
        med = {k: round(statistics.median(r[k] for r in rows), 3) for k in rows[0]}
        print(json.dumps({"opts": spec or "defaults", "triangles": tri, **med}), flush=True)
