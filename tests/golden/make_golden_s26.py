"""Golden record for the headline config (BASELINE.json configs[3]): R-MAT scale 26, edge
factor 16, seed 0 -- produced entirely by the CPU oracle, which restates the reference
(oracle/tricount_oracle.c: generators.py:203-284 rmat, preprocess.py:74-84, count.py:162-178)
and is itself pinned bit-for-bit against reference-generated goldens up to s24
(tests/test_oracle.py).  Nothing from the product package is imported.

The reference's own numpy/numba path needs ~45 min and ~180 GB for s26,
so this runs on the GPU box's host (CPU only; ~60 GB RAM, all cores):

    python tests/golden/make_golden_s26.py [scale]   -> tests/golden/golden_s<scale>.json

The record doubles as the one full, unsampled CPU run of the headline workload that
calibrates bench.py's sampled CPU baseline (every phase is timed).
"""
from __future__ import annotations

import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        if a.size == 0:
            continue
        mv = memoryview(a).cast("B")
        for i in range(0, len(mv), 1 << 28):
            h.update(mv[i:i + (1 << 28)])
    return h.hexdigest()


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main(scale: int) -> None:
    threads = os.cpu_count() or 1
    rec = {"gen": "rmat", "scale": scale, "edge_factor": 16, "seed": 0,
           "produced_by": "oracle (CPU restatement of the reference; no product code)",
           "host": {"cpu": cpu_model(), "threads": threads}}
    t = time.time()
    pairs = oracle.rmat_edges(scale, 16, seed=0, threads=threads)
    rec["generate_s"] = round(time.time() - t, 2)
    rec["pairs"] = int(pairs.shape[0])
    rec["n"] = int(pairs.max()) + 1
    rec["edges_sha256"] = sha(pairs)
    print("generated", rec, flush=True)
    t = time.time()
    src, dst, off = oracle.preprocess(pairs, num_vertices=rec["n"], threads=threads)
    rec["preprocess_s"] = round(time.time() - t, 2)
    del pairs
    rec["m"] = int(dst.shape[0])
    rec["csr_sha256"] = sha(src, dst, off)
    deg = np.diff(off)
    rec["max_out_degree"] = int(deg.max())
    rec["merge_work"] = oracle.merge_work(src, dst, off)
    print("preprocessed", rec, flush=True)
    t = time.time()
    rec["triangles"] = oracle.count(src, dst, off, workers=threads)
    rec["count_s"] = round(time.time() - t, 2)
    rec["edges_per_s_full_run"] = rec["m"] / (rec["preprocess_s"] + rec["count_s"])
    print("counted", rec, flush=True)
    with open(os.path.join(HERE, f"golden_s{scale}.json"), "w") as fh:
        json.dump(rec, fh, indent=1)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 26)
