"""Generate the golden vectors that pin the oracle and the GPU path.

Run ONCE in a container that has the reference mounted (it is not needed at test
time, and it does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--big]

Everything here is produced by the reference package ``tricount`` itself
(generators, preprocess, count_triangles); nothing from this repo is imported.
Outputs: tests/golden/golden.json (+ golden_big.json with --big).
"""
from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time

import numpy as np

from tricount.count import count_triangles, intersect_count
from tricount.generators import barabasi_albert, gnp, rmat
from tricount.graph import EdgeArray, OrientedGraph, edge_array_from_undirected, normalize
from tricount.preprocess import preprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def csr_record(g: EdgeArray, with_arrays: bool = False, workers: int = 8) -> dict:
    og = preprocess(g)
    deg = np.diff(og.node_offsets)
    work = int((deg[og.edge_src].astype(np.int64) + deg[og.edge_dst]).sum()) if og.m_dir else 0
    rec = {
        "n": g.num_vertices,
        "pairs": int(g.edges.shape[0]),
        "m": og.m_dir,
        "edges_sha256": sha(g.edges),
        "csr_sha256": sha(og.edge_src, og.edge_dst, og.node_offsets),
        "triangles": count_triangles(og, workers),
        "merge_work": work,
        "max_out_degree": int(deg.max()) if deg.size else 0,
    }
    if with_arrays:
        rec["edge_src"] = og.edge_src.tolist()
        rec["edge_dst"] = og.edge_dst.tolist()
        rec["node_offsets"] = og.node_offsets.tolist()
    return rec


def pairs_of(n):  # complete graph K_n as canonical pairs
    return [(i, j) for i in range(n) for j in range(i + 1, n)]


def ea(pairs):
    return edge_array_from_undirected(np.asarray(pairs, dtype=np.int64).reshape(-1, 2))


def small_cases() -> list[dict]:
    cases = []

    def add(name, g, tri=True):
        rec = csr_record(g, with_arrays=True)
        rec["name"] = name
        rec["input"] = g.edges.tolist()
        cases.append(rec)

    add("empty", EdgeArray([]))
    add("K3", ea(pairs_of(3)))
    add("K5", ea(pairs_of(5)))
    add("single_edge", ea([(0, 1)]))
    add("isolated_interior", ea([(0, 2)]))
    add("star4", ea([(0, i) for i in range(1, 5)]))
    add("path3", ea([(0, 1), (1, 2)]))
    add("petersen", ea(sorted({(min(u, v), max(u, v)) for u, v in
                               [(i, (i + 1) % 5) for i in range(5)]
                               + [(5 + i, 5 + (i + 2) % 5) for i in range(5)]
                               + [(i, 5 + i) for i in range(5)]})))
    # arbitrary raw inputs (hypothesis-style, reference test_preprocess.py:141-154)
    rng = np.random.default_rng(1234)
    for i in range(40):
        raw = rng.integers(0, 41, size=(int(rng.integers(0, 150)), 2))
        add(f"normalized_{i}", normalize(raw))
    # shuffled-order input (the contract allows any order)
    for i, seed in enumerate((3, 8, 21)):
        g = gnp(64, 0.3, seed=seed)
        perm = np.random.default_rng(100 + i).permutation(g.edges.shape[0])
        add(f"gnp64_shuffled_{seed}", EdgeArray(g.edges[perm]))
    # the 200-vertex id-gap case: isolated ids in the middle and at the top
    add("id_gaps", ea([(0, 7), (7, 100), (0, 100), (3, 250), (250, 251)]))
    return cases


def corpus(count: int, seed: int) -> list[tuple[int, float, int]]:
    """reference test_acceptance.py:48-55 parameter stream."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        n = int(rng.integers(2, 65))
        p = float(rng.choice((0.05, 0.1, 0.3, 0.7)))
        out.append((n, p, int(rng.integers(0, 2**31))))
    return out


def corpus_records(params) -> list[dict]:
    recs = []
    for n, p, s in params:
        rec = csr_record(gnp(n, p, seed=s))
        rec.update({"gen": "gnp", "n_param": n, "p": p, "seed": s})
        recs.append(rec)
    return recs


def main(big: bool) -> None:
    t0 = time.time()
    out = {
        "generated_by": "reference tricount (PYTHONPATH=/root/reference/pkg/src), numpy "
                        + np.__version__,
        "csr_sha256_recipe": "sha256(edge_src.u32 || edge_dst.u32 || node_offsets.i64)",
        "small": small_cases(),
        "intersect_handmade": {
            # reference test_count.py:39-45
            "edge_src": [0, 0, 0, 0, 1, 1, 1],
            "edge_dst": [2, 4, 6, 8, 4, 8, 9],
            "node_offsets": [0, 4, 7, 7, 7, 7, 7, 7, 7, 7, 7],
            "intersect_0_1": intersect_count(
                OrientedGraph(np.array([0, 0, 0, 0, 1, 1, 1], np.uint32),
                              np.array([2, 4, 6, 8, 4, 8, 9], np.uint32),
                              np.array([0, 4, 7, 7, 7, 7, 7, 7, 7, 7, 7], np.int64)), 0, 1),
        },
        "corpora": {
            "C1_20240615": corpus_records(corpus(200, 20240615)),
            "C3_77": corpus_records(corpus(20, 77)),
        },
        "graphs": {},
    }
    g = gnp(10_000, 100_000 / math.comb(10_000, 2), seed=0)
    out["graphs"]["er_1e4"] = dict(csr_record(g), gen="gnp", n_param=10_000,
                                   p=100_000 / math.comb(10_000, 2), seed=0)
    for scale, ef, seed in ((8, 4, 1), (10, 8, 7), (12, 16, 99), (16, 76, 20240616)):
        out["graphs"][f"rmat_{scale}_{ef}_{seed}"] = dict(
            csr_record(rmat(scale, ef, seed=seed)), gen="rmat", scale=scale, edge_factor=ef,
            seed=seed)
    for n, m_att, seed in ((1000, 3, 5), (100_000, 9, 0)):
        out["graphs"][f"ba_{n}_{m_att}_{seed}"] = dict(
            csr_record(barabasi_albert(n, m_att, seed=seed)), gen="barabasi_albert", n_param=n,
            m_attach=m_att, seed=seed)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=0)
    print(f"golden.json written in {time.time() - t0:.1f}s", flush=True)

    if big:
        big_out = {}
        for scale in (20, 21, 22):
            t = time.time()
            big_out[f"rmat_{scale}_16_0"] = dict(csr_record(rmat(scale, 16, seed=0)),
                                                gen="rmat", scale=scale, edge_factor=16, seed=0)
            print(scale, time.time() - t, big_out[f"rmat_{scale}_16_0"], flush=True)
            with open(os.path.join(HERE, "golden_big.json"), "w") as fh:
                json.dump(big_out, fh, indent=1)
        for n in (1_000_000, 10_000_000):
            t = time.time()
            big_out[f"ba_{n}_9_0"] = dict(csr_record(barabasi_albert(n, 9, seed=0)),
                                         gen="barabasi_albert", n_param=n, m_attach=9, seed=0)
            print(n, time.time() - t, big_out[f"ba_{n}_9_0"], flush=True)
            with open(os.path.join(HERE, "golden_big.json"), "w") as fh:
                json.dump(big_out, fh, indent=1)


if __name__ == "__main__":
    main("--big" in sys.argv)
