"""Development aid: fused preprocess+count steps on device pairs for any config
(rmatS, ba1e7, ba1e6, rgg2e7, ...): python scripts/step.py CONFIG [reps]."""
import sys

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import generators  # noqa: E402
from scripts import devopts  # noqa: E402

devopts.apply()


def make(w):
    if w.startswith("rmat"):
        return generators.rmat_device(int(w[4:]), 16, seed=0)
    if w.startswith("ba"):
        return generators.barabasi_albert_device(int(float(w[2:])), 9, seed=0)
    if w.startswith("rgg"):
        return generators.random_geometric_device(int(float(w[3:])), 32.0, seed=0)
    raise SystemExit(f"unknown config {w}")


if __name__ == "__main__":
    g = make(sys.argv[1])
    for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
        tri, t = tcb.count_with_timings_device(g)
        print(tri, {k: round(v, 3) for k, v in t.as_dict().items()}, flush=True)
