"""R-MAT s23 / s24 goldens produced by the reference package itself.

s23 (m = 2^27) is the smallest R-MAT on which the default count schedule turns the
v-major in-edge index on (tc_count.cu: m >= 2^27 and max out-degree > 256), so these two
records pin that schedule -- the one bench.py times at s26 -- against the reference's own
``preprocess`` + ``count_triangles`` (reference generators.py:203-284, preprocess.py:74-84,
count.py:162-178).  Run ONCE in the build container (the reference does not exist on the
GPU box); ~20 GB RAM peak at s24:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_huge.py 23 24

Output: tests/golden/golden_huge.json (same record layout as golden_big.json).
"""
from __future__ import annotations

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from make_golden import HERE, csr_record  # noqa: E402
from tricount.generators import rmat  # noqa: E402


def main(scales) -> None:
    path = os.path.join(HERE, "golden_huge.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for scale in scales:
        t = time.time()
        key = f"rmat_{scale}_16_0"
        out[key] = dict(csr_record(rmat(scale, 16, seed=0), workers=os.cpu_count()),
                        gen="rmat", scale=scale, edge_factor=16, seed=0,
                        reference_seconds=round(time.time() - t, 1))
        print(scale, out[key], flush=True)
        with open(path, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [23, 24])
