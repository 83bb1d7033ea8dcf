"""Golden counts for the random geometric graph (BASELINE config 5).

The reference has no RGG generator, so parity here means: the graph
is defined by oracle.rgg_pairs (numpy default_rng(seed).random((n, 2)) points; edge iff
squared distance < r^2), checked against a direct numpy evaluation of that definition on
the small case, and the triangles are counted by the REFERENCE counter
(tricount.preprocess + count_triangles).

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_rgg_golden.py
    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_rgg_golden.py --full
        (adds BASELINE config 5 at full size, n = 2*10^7: the reference counter on the
        6.4*10^8-pair oracle-generated graph, ~30 GB RAM, a few minutes on 8 cores)
"""
from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from tricount.count import count_triangles  # noqa: E402
from tricount.graph import EdgeArray  # noqa: E402
from tricount.preprocess import preprocess  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def brute(n, seed, r):
    p = np.random.default_rng(seed).random((n, 2))
    out = []
    for i0 in range(0, n, 2048):
        blk = p[i0:i0 + 2048]
        d = (blk[:, None, 0] - p[None, :, 0]) ** 2 + (blk[:, None, 1] - p[None, :, 1]) ** 2
        d[np.arange(blk.shape[0]), np.arange(i0, i0 + blk.shape[0])] = np.inf
        i, j = np.nonzero(d < r * r)
        out.append(np.stack([i + i0, j], 1))
    return np.concatenate(out).astype(np.uint32)


def main(full: bool):
    path = os.path.join(HERE, "golden_rgg.json")
    if full:
        cases = json.load(open(path))["rgg"]
        params = ((20_000_000, 32.0, 0),)
    else:
        cases = []
        params = ((2_000, 32.0, 3), (20_000, 32.0, 0), (200_000, 32.0, 0), (2_000_000, 32.0, 0),
                  (50_000, 200.0, 1))
    for n, k, seed in params:
        r = math.sqrt(k / (math.pi * n))
        pairs = oracle.rgg_pairs(n, k, seed)
        if n <= 50_000:
            assert np.array_equal(pairs, brute(n, seed, r)), n
        g = EdgeArray(pairs)
        del pairs
        t = count_triangles(preprocess(g), os.cpu_count())
        pairs = g.edges
        cases.append({"n": n, "avg_degree": k, "seed": seed, "radius": r, "pairs": int(pairs.shape[0]),
                      "num_vertices": int(g.num_vertices), "edges_sha256": sha(pairs), "triangles": int(t)})
        print(cases[-1], file=sys.stderr)
    with open(path, "w") as fh:
        json.dump({"rgg": cases}, fh, indent=1)


if __name__ == "__main__":
    main("--full" in sys.argv)
