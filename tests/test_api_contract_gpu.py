"""Contract tests of the C ABI through the Python mirror (GPU): concurrency (reference
SPEC.md:294 -- "safe to invoke concurrently on different graphs"), hand-built and
non-forward-oriented graphs, argument validation on upload, pools, and the shared-memory
staging limit.  Every count is checked against the oracle (CPU restatement of reference
count.py:63-99) -- bit-exact integers."""
from __future__ import annotations

import threading

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

tcb = pytest.importorskip("paper_1503_00576_b200")
from paper_1503_00576_b200 import _lib, generators  # noqa: E402
from paper_1503_00576_b200.graph import EdgeArray, OrientedGraph  # noqa: E402


def _graphs():
    """Four different graphs with their oracle counts."""
    out = []
    for scale, ef, seed in ((12, 16, 99), (13, 8, 1), (14, 16, 3), (11, 32, 5)):
        pairs = oracle.symmetrize(oracle.rmat_pairs(scale, ef, seed=seed))
        out.append((EdgeArray(pairs), oracle.count(*oracle.preprocess(pairs))))
    return out


def test_concurrent_calls_on_different_graphs():
    """8 Python threads (ctypes releases the GIL) count 4 different graphs at the same time
    through every counting entry point; every result must be the oracle's."""
    graphs = _graphs()
    ogs = [tcb.preprocess(g) for g, _ in graphs]
    errors, results = [], []
    start = threading.Barrier(8)

    def worker(k):
        try:
            start.wait()
            for rep in range(6):
                i = (k + rep) % 4
                g, want = graphs[i]
                which = (k + rep) % 4
                if which == 0:
                    got = tcb.count_triangles(ogs[i])
                elif which == 1:
                    got = tcb.count_with_timings(g)[0]
                elif which == 2:
                    got = tcb.count_partitioned(ogs[i], tcb.PartitionPlan.even(3, ogs[i].m_dir), 2)
                else:  # a fresh graph per call: the lazy rank-space copy is built concurrently
                    got = tcb.count_triangles(tcb.preprocess(g))
                results.append((i, which, got, want))
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(8)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    assert len(results) == 48
    bad = [r for r in results if r[2] != r[3]]
    assert not bad, bad


def test_concurrent_rank_copy_of_one_graph():
    """Many threads trigger the first full count (and the rank-space copy) of ONE graph."""
    g, want = _graphs()[2]
    og = tcb.preprocess(g)
    got = []
    threads = [threading.Thread(target=lambda: got.append(tcb.count_triangles(og))) for _ in range(8)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert got == [want] * 8


def test_hand_built_graph_not_forward_by_degree():
    """An OrientedGraph built by hand in id order (advisor case): 0->{1..5}, 1->{2,6}.  Its
    edges do not all point to a higher (out+in degree, id) rank, so full counts must stay
    on the original-id kernels; the reference counts 1 (triangle 0-1-2)."""
    src = np.array([0, 0, 0, 0, 0, 1, 1], np.uint32)
    dst = np.array([1, 2, 3, 4, 5, 2, 6], np.uint32)
    off = np.array([0, 5, 7, 7, 7, 7, 7, 7], np.int64)
    og = OrientedGraph(src, dst, off)
    want = oracle.count(src, dst, off)
    assert want == 1
    assert tcb.count_triangles(og) == want
    assert tcb.count_device(og, algo=_lib.ALGO_MERGE_THREAD)[0] == want
    assert tcb.count_partitioned(og, tcb.PartitionPlan.even(3, og.m_dir), 1) == want
    assert sum(tcb.count_device(og, lo, hi)[0] for lo, hi in ((0, 3), (3, 7))) == want


def test_preprocess_of_non_symmetric_pairs_all_paths_agree():
    """preprocess() orients by first-column degree; on a non-symmetric array that differs
    from out+in degree, so the two-call path must not take the rank-space shortcut blindly.
    count_triangles(preprocess(g)), count_with_timings(g) and ranged counts all equal the
    oracle on the same array."""
    rng = np.random.default_rng(7)
    for scale in (10, 14):
        p = oracle.symmetrize(oracle.rmat_pairs(scale, 16, seed=scale))
        p = np.ascontiguousarray(p[rng.random(p.shape[0]) < 0.7])
        want = oracle.count(*oracle.preprocess(p))
        g = EdgeArray(p)
        og = tcb.preprocess(g)
        assert tcb.count_triangles(og) == want
        assert tcb.count_with_timings(g)[0] == want
        half = og.m_dir // 2
        assert tcb.count_device(og, 0, half)[0] + tcb.count_device(og, half, og.m_dir)[0] == want


def test_random_dags_match_oracle():
    """Random hand-built DAG CSRs (sorted lists, arbitrary orientation): full, ranged and
    merge-thread counts equal the oracle."""
    rng = np.random.default_rng(11)
    for n, m in ((50, 400), (300, 6000), (2000, 30000)):
        a = rng.integers(0, n, m)
        b = rng.integers(0, n, m)
        keep = a != b
        perm = rng.permutation(n)  # random orientation: by a random vertex order
        u = np.where(perm[a] < perm[b], a, b)[keep]
        v = np.where(perm[a] < perm[b], b, a)[keep]
        keys = np.unique((u.astype(np.uint64) << np.uint64(32)) | v.astype(np.uint64))
        src = (keys >> np.uint64(32)).astype(np.uint32)
        dst = (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        off = np.zeros(n + 1, np.int64)
        np.cumsum(np.bincount(src, minlength=n), out=off[1:])
        og = OrientedGraph(src, dst, off)
        want = oracle.count(src, dst, off)
        assert tcb.count_triangles(og) == want
        assert tcb.count_device(og, algo=_lib.ALGO_MERGE_THREAD)[0] == want
        assert tcb.count_partitioned(og, tcb.PartitionPlan.even(4, og.m_dir), 1) == want


def test_upload_rejects_bad_offsets():
    src = np.array([0, 0, 1], np.uint32)
    dst = np.array([1, 2, 2], np.uint32)
    for off in ([1, 2, 3, 3], [0, 2, 3, 4], [0, 3, 2, 3]):
        og = OrientedGraph(src, dst, np.array(off, np.int64))
        with pytest.raises(ValueError):
            tcb.count_triangles(og)
    og = OrientedGraph(src, np.array([1, 2, 7], np.uint32), np.array([0, 2, 3, 3], np.int64))
    with pytest.raises(ValueError):
        tcb.count_triangles(og)
    # the library is still healthy afterwards
    ok = OrientedGraph(src, dst, np.array([0, 2, 3, 3], np.int64))
    assert tcb.count_triangles(ok) == 1


def test_count_with_timings_pools(golden):
    """reference test_count.py:152-156: count_with_timings(g, 2, pools=4)."""
    rec = golden["graphs"]["rmat_12_16_99"]
    g = generators.rmat(12, 16, seed=99)
    for pools in (1, 2, 4, 7):
        tri, t = tcb.count_with_timings(g, 2, pools=pools)
        assert tri == rec["triangles"]
        assert t.preprocess_ms > 0 and t.count_ms > 0
        assert t.total_ms >= t.count_ms
    with pytest.raises(ValueError):
        tcb.count_with_timings(g, 2, pools=0)


def test_out_degree_beyond_shared_memory_staging():
    """A hand-built source with 60,000 out-edges (above the 51,200-entry shared-memory
    staging limit) is counted by the thread-per-edge merge instead of failing:
    0 -> {1..60000} and i -> i+1 close 59,999 triangles."""
    k = 60_000
    src = np.concatenate([np.zeros(k, np.uint32), np.arange(1, k, dtype=np.uint32)])
    dst = np.concatenate([np.arange(1, k + 1, dtype=np.uint32), np.arange(2, k + 1, dtype=np.uint32)])
    off = np.zeros(k + 2, np.int64)
    np.cumsum(np.bincount(src, minlength=k + 1), out=off[1:])
    og = OrientedGraph(src, dst, off)
    assert tcb.count_triangles(og) == k - 1
    assert tcb.count_device(og, 0, k)[0] == k - 1


def test_options_api():
    assert _lib.get_option("vmajor") == -1
    with _lib.options(vmajor=0, light=2):
        assert _lib.get_option("vmajor") == 0 and _lib.get_option("light") == 2
    assert _lib.get_option("vmajor") == -1 and _lib.get_option("light") == -1
    with pytest.raises(ValueError):
        _lib.set_option("no_such_option", 1)


def test_foreign_oriented_graph_objects():
    """An object carrying the reference OrientedGraph's arrays (a tricount.graph.OrientedGraph
    handed over by reference code, graph.py:146-193) is accepted by every counting entry
    point; its device copy lives as long as the object (reference test_count.py:39-45)."""
    import gc

    class RefOG:  # duck-typed stand-in: frozen arrays + m_dir / num_vertices
        def __init__(self, src, dst, off):
            self.edge_src, self.edge_dst, self.node_offsets = src, dst, off
            self.m_dir, self.num_vertices = int(dst.size), int(off.size) - 1

    src = np.array([0, 0, 0, 0, 1, 1, 1], np.uint32)
    dst = np.array([2, 4, 6, 8, 4, 8, 9], np.uint32)
    off = np.array([0, 4, 7, 7, 7, 7, 7, 7, 7, 7, 7], np.int64)
    for _ in range(3):
        og = RefOG(src, dst, off)
        assert tcb.intersect_count(og, 0, 1) == 2
        assert tcb.count_triangles(og) == 0
        assert tcb.count_partitioned(og, tcb.PartitionPlan.even(2, og.m_dir), 1) == 0
        del og
        gc.collect()
    pairs = oracle.symmetrize(oracle.rmat_pairs(10, 8, seed=7))
    s, d, o = oracle.preprocess(pairs)
    og = RefOG(s, d, o)
    assert tcb.count_triangles(og) == oracle.count(s, d, o)
    assert sum(tcb.intersect_count(og, int(u), int(v)) for u, v in zip(s[:200], d[:200])) == \
        sum(oracle.intersect_count(d, o, int(u), int(v)) for u, v in zip(s[:200], d[:200]))


def test_chunked_copy_with_overlapped_degrees(golden_big):
    """Host pairs are copied in 256 MB chunks (pinned) or 128 MB staged chunks (pageable)
    while the degree histogram of each landed chunk runs on the compute stream.  R-MAT s21
    (537 MB of pairs: several chunks of either kind) through count_with_timings and the
    two-call path equals the reference golden; an out-of-range id placed in the last chunk
    is still reported as ValueError by both entry points."""
    d = generators.rmat_device(21, 16, seed=0)
    pinned = d.to_host(pinned=True)
    d.free()
    want = golden_big["rmat_21_16_0"]["triangles"]
    pageable = EdgeArray(np.array(pinned.edges), num_vertices=pinned.num_vertices)
    for g in (pinned, pageable):
        assert tcb.count_with_timings(g)[0] == want
        assert tcb.count_triangles(tcb.preprocess(g)) == want
    bad = np.array(pinned.edges)
    bad[-1, 0] = pinned.num_vertices  # id == num_vertices: out of range
    with pytest.raises(ValueError):
        tcb.count_with_timings(EdgeArray(bad, num_vertices=pinned.num_vertices))
    with pytest.raises(ValueError):
        tcb.preprocess(EdgeArray(bad, num_vertices=pinned.num_vertices))
