"""GPU parity: the sm_100a path (through the C ABI) against the oracle and the golden
vectors produced by the reference.  Integer work: every comparison is bit-exact."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from conftest import sha

pytestmark = pytest.mark.gpu

tcb = pytest.importorskip("paper_1503_00576_b200")
from paper_1503_00576_b200 import _lib, generators  # noqa: E402
from paper_1503_00576_b200.graph import EdgeArray, OrientedGraph, validate_oriented_graph  # noqa: E402


def _csr(og):
    return og.edge_src, og.edge_dst, og.node_offsets


def _count_all_ways(og, expected):
    assert tcb.count_triangles(og) == expected
    assert tcb.count_device(og, algo=_lib.ALGO_MERGE_THREAD)[0] == expected
    for pools in (2, 3, 5):
        assert tcb.count_partitioned(og, tcb.PartitionPlan.even(pools, og.m_dir), 1) == expected


def test_small_cases(golden):
    for case in golden["small"]:
        g = EdgeArray(np.asarray(case["input"], dtype=np.uint32).reshape(-1, 2))
        og = tcb.preprocess(g)
        assert og.edge_src.tolist() == case["edge_src"], case["name"]
        assert og.edge_dst.tolist() == case["edge_dst"], case["name"]
        assert og.node_offsets.tolist() == case["node_offsets"], case["name"]
        if og.m_dir:
            _count_all_ways(og, case["triangles"])
        else:
            assert tcb.count_triangles(og) == 0
        t, timings = tcb.count_with_timings(g)
        assert t == case["triangles"]


def test_intersect_handmade(golden):
    h = golden["intersect_handmade"]
    og = OrientedGraph(np.array(h["edge_src"], np.uint32), np.array(h["edge_dst"], np.uint32),
                       np.array(h["node_offsets"], np.int64))
    assert tcb.intersect_count(og, 0, 1) == 2
    assert tcb.count_triangles(og) == 0


@pytest.mark.parametrize("corpus", ["C1_20240615", "C3_77"])
def test_corpora(golden, corpus):
    for i, rec in enumerate(golden["corpora"][corpus]):
        pairs = oracle.gnp_pairs(rec["n_param"], rec["p"], rec["seed"])
        og = tcb.preprocess(EdgeArray(pairs))
        assert sha(*_csr(og)) == rec["csr_sha256"]
        assert tcb.count_triangles(og, 1 + i % 8) == rec["triangles"]


@pytest.mark.parametrize("name", ["rmat_8_4_1", "rmat_10_8_7", "rmat_12_16_99",
                                  "rmat_16_76_20240616"])
def test_rmat_generator_and_pipeline(golden, name):
    rec = golden["graphs"][name]
    g = generators.rmat(rec["scale"], rec["edge_factor"], seed=rec["seed"])
    assert sha(g.edges) == rec["edges_sha256"], "device rmat must equal reference rmat"
    assert g.num_vertices == rec["n"]
    og = tcb.preprocess(g)
    assert sha(*_csr(og)) == rec["csr_sha256"]
    assert og.device().max_out == rec["max_out_degree"]
    assert tcb.merge_work(og) == rec["merge_work"]
    _count_all_ways(og, rec["triangles"])


def test_er_config(golden):
    rec = golden["graphs"]["er_1e4"]
    pairs = oracle.gnp_pairs(rec["n_param"], rec["p"], rec["seed"])
    assert sha(pairs) == rec["edges_sha256"]
    og = tcb.preprocess(EdgeArray(pairs))
    assert sha(*_csr(og)) == rec["csr_sha256"]
    _count_all_ways(og, rec["triangles"])
    assert rec["triangles"] == 1343


def test_shuffled_input_same_csr():
    pairs = oracle.symmetrize(oracle.rmat_pairs(12, 16, seed=99))
    ref = tcb.preprocess(EdgeArray(pairs))
    perm = np.random.default_rng(1).permutation(pairs.shape[0])
    shuf = tcb.preprocess(EdgeArray(pairs[perm]))
    assert ref == shuf
    validate_oriented_graph(shuf)


def test_substeps_match_oracle(golden):
    rec = golden["graphs"]["rmat_12_16_99"]
    pairs = oracle.symmetrize(oracle.rmat_pairs(12, 16, seed=99))
    perm = np.random.default_rng(2).permutation(pairs.shape[0])
    g = EdgeArray(pairs[perm])
    s = tcb.sort_edges(g)
    assert np.array_equal(s.edges, pairs)
    off_all = tcb.build_node_array(s, g.num_vertices)
    assert np.array_equal(off_all, oracle.build_node_array(pairs[:, 0], g.num_vertices))
    deg = tcb.DegreeOrder(np.diff(off_all))
    directed = tcb.orient_and_compact(s, deg)
    src, dst, off = oracle.preprocess(pairs)
    assert np.array_equal(directed[:, 0], src) and np.array_equal(directed[:, 1], dst)
    assert np.array_equal(tcb.build_node_array(directed[:, 0], g.num_vertices), off)


def test_upload_path_and_partitions(golden):
    rec = golden["graphs"]["rmat_12_16_99"]
    src, dst, off = oracle.preprocess(oracle.symmetrize(oracle.rmat_pairs(12, 16, seed=99)))
    og = OrientedGraph(src, dst, off)
    _count_all_ways(og, rec["triangles"])
    for pools in (1, 2, 4, 8):
        plan = tcb.PartitionPlan.work_balanced(og, pools)
        plan.check_covers(og.m_dir)
        assert tcb.count_partitioned(og, plan, 2) == rec["triangles"]
        # every single pool agrees with the oracle's count over the same edge range
        for p in range(pools):
            lo, hi = plan.pool_range(p)
            assert tcb.count_device(og, lo, hi)[0] == _range_oracle(src, dst, off, lo, hi)


def _range_oracle(src, dst, off, lo, hi):
    lib = oracle.lib()
    return int(lib.or_count_strided(oracle._c32(src), oracle._c32(dst), oracle._c64(off), lo, hi, 0, 1))


def test_range_counts_match_oracle():
    src, dst, off = oracle.preprocess(oracle.symmetrize(oracle.rmat_pairs(12, 16, seed=99)))
    og = OrientedGraph(src, dst, off)
    rng = np.random.default_rng(7)
    for _ in range(20):
        lo, hi = sorted(int(x) for x in rng.integers(0, og.m_dir + 1, size=2))
        assert tcb.count_device(og, lo, hi)[0] == _range_oracle(src, dst, off, lo, hi)


def test_rejects_bad_arguments():
    og = tcb.preprocess(EdgeArray([(0, 1), (1, 0)]))
    with pytest.raises(ValueError):
        tcb.count_triangles(og, 0)
    with pytest.raises(ValueError):
        tcb.count_partitioned(og, tcb.PartitionPlan(2, (0, 1, 2)), 1)
    with pytest.raises(ValueError):
        tcb.count_device(og, 0, 5)


def test_big_rmat_s20(golden_big):
    rec = golden_big.get("rmat_20_16_0")
    if rec is None:
        pytest.skip("s20 golden not generated")
    g = generators.rmat_device(20, 16, seed=0)
    h = g.to_host()
    assert sha(h.edges) == rec["edges_sha256"]
    og, _ = tcb.preprocess_device(g)
    assert sha(*_csr(og)) == rec["csr_sha256"]
    assert tcb.count_triangles(og) == rec["triangles"] == 490_084_299
    assert tcb.count_device(og, algo=_lib.ALGO_MERGE_THREAD)[0] == rec["triangles"]
    t, _ = tcb.count_with_timings_device(g)
    assert t == rec["triangles"]


@pytest.mark.parametrize("scale", [21, 22])
def test_big_rmat_counts(golden_big, scale):
    rec = golden_big.get(f"rmat_{scale}_16_0")
    if rec is None:
        pytest.skip(f"s{scale} golden not generated")
    g = generators.rmat_device(scale, 16, seed=0)
    og, _ = tcb.preprocess_device(g)
    assert sha(*_csr(og)) == rec["csr_sha256"]
    assert tcb.count_triangles(og) == rec["triangles"]


def _default_schedule_pin(rec, scale):
    """Device generator, reference-id CSR and the DEFAULT count schedule (the one bench.py
    times: rank-space preprocess, v-major in-edge index auto-on for m >= 2^27) against a
    record that the reference (s23, s24) or the full oracle run (s26) produced."""
    g = generators.rmat_device(scale, 16, seed=0)
    assert g.npairs == rec["pairs"] and g.num_vertices == rec["n"]
    h = g.to_host(pinned=True)
    assert sha(h.edges) == rec["edges_sha256"], "device rmat must equal the reference rmat"
    del h
    with _lib.options(count_stats=1):
        tri, t = tcb.count_with_timings_device(g)
    assert tri == rec["triangles"]
    assert t.vmajor_ms > 0, "the default schedule at m >= 2^27 runs the v-major kernels"
    og, _ = tcb.preprocess_device(g)
    g.free()
    assert sha(*_csr(og)) == rec["csr_sha256"]
    assert tcb.merge_work(og) == rec["merge_work"]
    assert og.device().max_out == rec["max_out_degree"]
    assert tcb.count_triangles(og) == rec["triangles"]  # two-call path (relabelled copy)
    plan = tcb.PartitionPlan.work_balanced(og, 8)
    assert tcb.count_partitioned(og, plan, 1) == rec["triangles"]


@pytest.mark.parametrize("scale", [23, 24])
def test_huge_rmat_default_schedule(golden_huge, scale):
    rec = golden_huge.get(f"rmat_{scale}_16_0")
    if rec is None:
        pytest.skip(f"s{scale} golden not generated")
    _default_schedule_pin(rec, scale)


def test_headline_rmat_s26(golden_s26):
    """BASELINE.json configs[3], the bench workload: bit-exact input, CSR and count against
    the full oracle run (51,563,396,809 triangles if the r01 device count was right)."""
    _default_schedule_pin(golden_s26, 26)


@pytest.mark.parametrize("name", ["ba_1000_3_5", "ba_100000_9_0"])
def test_ba_generator_and_pipeline(golden, name):
    rec = golden["graphs"][name]
    g = generators.barabasi_albert(rec["n_param"], rec["m_attach"], seed=rec["seed"])
    assert sha(g.edges) == rec["edges_sha256"], "device-symmetrised BA must equal reference BA"
    og = tcb.preprocess(g)
    assert sha(*_csr(og)) == rec["csr_sha256"]
    _count_all_ways(og, rec["triangles"])
    assert tcb.count_with_timings(g)[0] == rec["triangles"]


@pytest.mark.parametrize("n", [1_000_000, 10_000_000])
def test_big_ba(golden_big, n):
    """BA config 3 (n = 10^7, m = 9): bit-identical input, CSR and count."""
    rec = golden_big.get(f"ba_{n}_9_0")
    if rec is None:
        pytest.skip("BA golden not generated")
    d = generators.barabasi_albert_device(n, 9, seed=0)
    h = d.to_host()
    assert sha(h.edges) == rec["edges_sha256"]
    og, _ = tcb.preprocess_device(d)
    assert sha(*_csr(og)) == rec["csr_sha256"]
    assert tcb.count_triangles(og) == rec["triangles"]
    assert tcb.count_with_timings_device(d)[0] == rec["triangles"]
    assert tcb.count_device(og, algo=_lib.ALGO_MERGE_THREAD)[0] == rec["triangles"]


def _complete_pairs(k: int) -> np.ndarray:
    """K_k, both directions, lexicographically sorted (reference complete_graph)."""
    iu = np.triu_indices(k, k=1)
    a = np.stack([iu[0], iu[1]], axis=1).astype(np.uint32)
    both = np.concatenate([a, a[:, ::-1]])
    return both[np.lexsort((both[:, 1], both[:, 0]))]


@pytest.mark.parametrize("k", [34, 600, 3000, 17000])
def test_complete_graphs_every_size_class(k):
    """Closed form C(k, 3) through every count path: the hub classes (d+ up to 16384),
    the sorted-array class (d+ > 16384: K_17000), the window path (K_34 light part),
    the fused rank-space path and the reference-id ranged kernels."""
    import math
    g = EdgeArray(_complete_pairs(k))
    want = math.comb(k, 3)
    assert tcb.count_with_timings(g)[0] == want
    og = tcb.preprocess(g)
    assert og.device().max_out == k - 1
    assert tcb.count_triangles(og) == want
    half = og.m_dir // 2
    assert tcb.count_device(og, 0, half)[0] + tcb.count_device(og, half, og.m_dir)[0] == want
    if k <= 3000:
        assert tcb.count_device(og, algo=_lib.ALGO_MERGE_THREAD)[0] == want


def _golden_rgg():
    import json
    import os
    from conftest import GOLDEN_DIR
    with open(os.path.join(GOLDEN_DIR, "golden_rgg.json")) as fh:
        return json.load(fh)["rgg"]


@pytest.mark.parametrize("case", [c for c in _golden_rgg() if c["n"] < 20_000_000],
                         ids=lambda c: f"n{c['n']}_k{int(c['avg_degree'])}")
def test_rgg_generator_and_count(case):
    """RGG (config 5): device generator == oracle definition (sha), count == reference."""
    d = generators.random_geometric_device(case["n"], case["avg_degree"], seed=case["seed"])
    assert d.npairs == case["pairs"] and d.num_vertices == case["num_vertices"]
    assert sha(d.to_host().edges) == case["edges_sha256"]
    assert tcb.count_with_timings_device(d)[0] == case["triangles"]
    og, _ = tcb.preprocess_device(d)
    assert tcb.count_triangles(og) == case["triangles"]
    assert tcb.count_device(og, algo=_lib.ALGO_MERGE_THREAD)[0] == case["triangles"]


def test_rgg_config5_full_size():
    """n = 2*10^7, avg degree 32 (BASELINE config 5): generator == oracle restatement bit for
    bit, and every count path == the REFERENCE counter's count of that graph (golden_rgg.json,
    make_rgg_golden.py --full: tricount.preprocess + count_triangles)."""
    rec = next((c for c in _golden_rgg() if c["n"] == 20_000_000), None)
    if rec is None:
        pytest.skip("full-size RGG golden not generated")
    n = 20_000_000
    d = generators.random_geometric_device(n, 32.0, seed=0)
    host = d.to_host()
    ref = oracle.rgg_pairs(n, 32.0, seed=0)
    assert np.array_equal(host.edges, ref)
    t, _ = tcb.count_with_timings_device(d)
    assert t == rec["triangles"] == 2_000_002_911
    og, _ = tcb.preprocess_device(d)
    assert tcb.count_triangles(og) == t
    assert tcb.count_partitioned(og, tcb.PartitionPlan.work_balanced(og, 3), 1) == t


def _rank_csr_numpy(pairs: np.ndarray, n: int):
    """Rank-space CSR restated in numpy: vertices relabelled by (degree, id) rank (the
    reference orientation order, preprocess.py:49-62), oriented low -> high rank, sorted."""
    deg = np.bincount(pairs[:, 0], minlength=n)
    order = np.lexsort((np.arange(n), deg))
    rank = np.empty(n, np.int64)
    rank[order] = np.arange(n)
    ru, rv = rank[pairs[:, 0]], rank[pairs[:, 1]]
    keep = ru < rv
    ru, rv = ru[keep], rv[keep]
    o = np.lexsort((rv, ru))
    off = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(ru, minlength=n), out=off[1:])
    return ru[o].astype(np.uint32), rv[o].astype(np.uint32), off


@pytest.mark.parametrize("case", ["rmat14", "ba", "k600_shuffled", "k5000"])
def test_rank_space_csr_matches_numpy(case):
    """The count-ready rank-space CSR (bucket scatter + size-class segmented sort: register,
    warp, CTA and global-radix classes) is byte-identical to a numpy restatement."""
    if case == "rmat14":
        pairs = oracle.symmetrize(oracle.rmat_pairs(14, 16, seed=3))
    elif case == "ba":
        pairs = generators.barabasi_albert(20000, 9, seed=1, pinned=False).edges
    elif case == "k600_shuffled":
        pairs = _complete_pairs(600)
        pairs = pairs[np.random.default_rng(5).permutation(pairs.shape[0])]
    else:
        pairs = _complete_pairs(5000)  # lists of 4999: the global-radix class
    pairs = np.ascontiguousarray(pairs, dtype=np.uint32)
    n = int(pairs.max()) + 1
    og, _ = tcb.preprocess_device(EdgeArray(pairs, num_vertices=n), rank_space=True)
    src, dst, off = _rank_csr_numpy(pairs, n)
    assert np.array_equal(og.edge_src, src)
    assert np.array_equal(og.edge_dst, dst)
    assert np.array_equal(og.node_offsets, off)


@pytest.mark.parametrize("opts", [
    {"vmajor": 1},                                   # hub-zone heads v-major
    {"vmajor": 1, "vzone_log2": 19, "vlow_all": 1},  # + heads below the hub zone
    {"vmajor": 1, "vm_bias": 1},                     # (almost) every hub-head edge v-major
    {"vmajor": 1, "vm_bias": 4, "vzone_log2": 22},   # round-1 defaults: neutral bias, 2^22 zone
    {"vmajor": 1, "midwarp": 0, "light": 2},         # CTA mid class, warp light kernel
    {"vmajor": 0, "light": 0},                       # u-major only, CTA-window light kernel
    {"vmajor": 0, "light_vec": 1, "hub_unroll": 2},  # vector light loads, 2-way hub unroll
    {"bucket": 0},                                   # rank-space preprocess by global key sort
    {"vmajor": 1, "hubpack": 1},                     # hub suffixes from the 18-bit packed copy
    {"vmajor": 1, "hubpack": 2},                     # packed reads, 4-byte cost model
    {"vmajor": 1, "vhub": 0},                        # hub heads on the masked-sweep CTA kernel
    {"vmajor": 1, "vin_overlap": 0, "seg_k16": 0},   # in-edge index serial; 1024-wide sorts
    {"vmajor": 1, "vhub_blocks": 8, "seg_w2k": 1},   # source-blocked top-band tasks; warp 2K sorts
    {"vmajor": 1, "vhub_unroll": 1},                 # unpipelined-width sweep
    {"vmajor": 1, "vix": 0},                         # index built at count time (k_vin_pass)
], ids=lambda o: ",".join(f"{k}={v}" for k, v in o.items()))
def test_count_schedules_agree(opts, golden_big):
    """Every count schedule (v-major on/off and its zone, the per-edge bias, the light and
    mid-class kernels, the preprocess variant) gives the golden count, for full and ranged
    counts.  Options are set through the explicit ABI call tc_set_option (the library never
    reads the environment)."""
    want = {14: None, 18: None, 20: golden_big["rmat_20_16_0"]["triangles"]}
    with _lib.options(**opts):
        for scale in (14, 18, 20):
            g = generators.rmat_device(scale, 16, seed=0)
            tri, _ = tcb.count_with_timings_device(g)
            og, _ = tcb.preprocess_device(g, rank_space=True)
            third = og.m_dir // 3
            parts = [tcb.count_device(og, 0, third)[0], tcb.count_device(og, third, og.m_dir)[0]]
            full = tcb.count_device(og)[0]
            g.free()
            ref = want[scale] or oracle.count(*oracle.preprocess(oracle.symmetrize(
                oracle.rmat_pairs(scale, 16, seed=0))))
            assert [tri, sum(parts), full] == [ref, ref, ref], (scale, opts)
        # a non-symmetric array (10 % of the pairs dropped): the v-major capacity layout
        # must notice and recount
        p = oracle.symmetrize(oracle.rmat_pairs(16, 16, seed=4))
        p = np.ascontiguousarray(p[np.random.default_rng(2).random(p.shape[0]) < 0.9])
        assert tcb.count_with_timings(EdgeArray(p))[0] == oracle.count(*oracle.preprocess(p))


def test_prebuilt_vmajor_index():
    """The rank-space preprocess fills the v-major in-edge index inside its segmented sorts
    (option vix) when full counts will run v-major; a full count reuses it only when its
    split equals the one the index was filled with.  Same count for: the reused index
    (twice), a count under a different split (index rebuilt), the index turned off, and
    ranged counts (always rebuilt over the range)."""
    pairs = oracle.symmetrize(oracle.rmat_pairs(15, 16, seed=11))
    want = oracle.count(*oracle.preprocess(pairs))
    g = EdgeArray(np.ascontiguousarray(pairs, dtype=np.uint32))
    got = []
    with _lib.options(vmajor=1):
        og = tcb.preprocess(g)
        got += [tcb.count_triangles(og), tcb.count_triangles(og)]
        with _lib.options(vmajor=1, vm_bias=2):
            got.append(tcb.count_triangles(og))
        half = og.m_dir // 2
        got.append(tcb.count_partitioned(og, tcb.PartitionPlan(2, (0, half, og.m_dir)), 1))
        got.append(tcb.count_with_timings(g)[0])
    with _lib.options(vmajor=1, vix=0):
        got.append(tcb.count_with_timings(g)[0])
    assert got == [want] * len(got), got


def test_forced_vmajor_without_hubs(golden_big):
    """v-major forced on graphs without hubs (BA 10^7, RGG 2*10^7: the zone lies below the
    hub zone, thousands of small warp tasks, cuckoo tables at load 1/3 -- RGG produced key
    sets on which 32 cuckoo seeds failed, now a binary-search fallback): same counts as
    the default schedule."""
    got = {}
    for vm in (1, 0):
        with _lib.options(vmajor=vm):
            out = {}
            g = generators.barabasi_albert_device(10_000_000, 9, seed=0)
            out["ba1e7"] = tcb.count_with_timings_device(g)[0]
            g.free()
            g = generators.random_geometric_device(20_000_000, 32.0, seed=0)
            out["rgg2e7"] = tcb.count_with_timings_device(g)[0]
            g.free()
            got[vm] = out
    assert got[1] == got[0], got
    assert got[0]["ba1e7"] == golden_big["ba_10000000_9_0"]["triangles"]


@pytest.mark.parametrize("name", ["rmat23", "rmat16_forced", "rgg2e6"])
def test_shard_plan_covers_every_edge_once(golden_huge, name):
    """The multi-GPU shard plan (edge ranges for u-major/light work, head ranges for v-major
    work): for P = 1..8 the shard counts sum to the full count, including empty shards."""
    from paper_1503_00576_b200.count import count_shard, shard_plan
    opts = {"vmajor": 1} if name == "rmat16_forced" else {}
    with _lib.options(**opts):
        if name == "rmat23":
            g = generators.rmat_device(23, 16, seed=0)
            want = golden_huge["rmat_23_16_0"]["triangles"]
        elif name == "rmat16_forced":
            g = generators.rmat_device(16, 16, seed=0)
            want = None
        else:
            g = generators.random_geometric_device(2_000_000, 32.0, seed=0)
            want = next(c for c in _golden_rgg() if c["n"] == 2_000_000)["triangles"]
        og, _ = tcb.preprocess_device(g, rank_space=True)
        full = tcb.count_device(og)[0]
        if want is not None:
            assert full == want
        for P in (1, 2, 3, 8):
            eb, hb = shard_plan(og, P)
            assert eb[0] == 0 and eb[-1] == og.m_dir and hb[0] == 0 and hb[-1] == og.num_vertices
            assert all(eb[i] <= eb[i + 1] for i in range(P)) and all(hb[i] <= hb[i + 1] for i in range(P))
            parts = [count_shard(og, eb[r], eb[r + 1], hb[r], hb[r + 1])[0] for r in range(P)]
            assert sum(parts) == full, (name, P, parts)
        # degenerate shards: everything in one shard, nothing in the other
        m, n = og.m_dir, og.num_vertices
        assert count_shard(og, 0, m, 0, n)[0] == full
        assert count_shard(og, 0, 0, 0, 0)[0] == 0
        assert count_shard(og, 0, m, 0, 0)[0] + count_shard(og, m, m, 0, n)[0] == full
        g.free()
