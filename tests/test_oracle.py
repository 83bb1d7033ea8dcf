"""Pin the CPU oracle (oracle/) against golden vectors produced by the reference."""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from conftest import sha


def test_small_cases_bit_exact(golden):
    for case in golden["small"]:
        pairs = np.asarray(case["input"], dtype=np.uint32).reshape(-1, 2)
        src, dst, off = oracle.preprocess(pairs)
        assert src.tolist() == case["edge_src"], case["name"]
        assert dst.tolist() == case["edge_dst"], case["name"]
        assert off.tolist() == case["node_offsets"], case["name"]
        assert oracle.count(src, dst, off, workers=3) == case["triangles"], case["name"]
        rs, rd, ro = oracle.reference_preprocess(pairs)
        assert (rs, rd, ro) == (case["edge_src"], case["edge_dst"], case["node_offsets"])


def test_pure_python_oracles_agree(golden):
    for case in golden["small"]:
        pairs = np.asarray(case["input"], dtype=np.uint32).reshape(-1, 2)
        assert oracle.brute_force_count(pairs) == case["triangles"], case["name"]
        assert oracle.sequential_forward_count(pairs) == case["triangles"], case["name"]


def test_intersect_handmade(golden):
    h = golden["intersect_handmade"]
    dst = np.asarray(h["edge_dst"], np.uint32)
    off = np.asarray(h["node_offsets"], np.int64)
    assert oracle.intersect_count(dst, off, 0, 1) == h["intersect_0_1"] == 2


@pytest.mark.parametrize("corpus", ["C1_20240615", "C3_77"])
def test_corpus_generation_and_counts(golden, corpus):
    for rec in golden["corpora"][corpus]:
        pairs = oracle.gnp_pairs(rec["n_param"], rec["p"], rec["seed"])
        assert sha(pairs) == rec["edges_sha256"]
        src, dst, off = oracle.preprocess(pairs)
        assert sha(src, dst, off) == rec["csr_sha256"]
        assert oracle.count(src, dst, off, workers=2) == rec["triangles"]


def _regen(rec):
    if rec["gen"] == "gnp":
        return oracle.gnp_pairs(rec["n_param"], rec["p"], rec["seed"])
    if rec["gen"] == "rmat":
        return oracle.symmetrize(oracle.rmat_pairs(rec["scale"], rec["edge_factor"], rec["seed"]))
    if rec["gen"] == "barabasi_albert":
        return oracle.ba_pairs(rec["n_param"], rec["m_attach"], rec["seed"])
    pytest.skip(f"no oracle generator for {rec['gen']}")


@pytest.mark.parametrize("name", ["er_1e4", "rmat_8_4_1", "rmat_10_8_7", "rmat_12_16_99",
                                  "rmat_16_76_20240616", "ba_1000_3_5", "ba_100000_9_0"])
def test_graph_goldens(golden, name):
    rec = golden["graphs"][name]
    pairs = _regen(rec)
    assert sha(pairs) == rec["edges_sha256"]
    src, dst, off = oracle.preprocess(pairs)
    assert sha(src, dst, off) == rec["csr_sha256"]
    assert oracle.merge_work(src, dst, off) == rec["merge_work"]
    assert oracle.count(src, dst, off) == rec["triangles"]


def test_partitioned_matches(golden):
    rec = golden["graphs"]["rmat_12_16_99"]
    src, dst, off = oracle.preprocess(_regen(rec))
    m = dst.size
    for pools in (1, 2, 3, 4, 8):
        bounds = np.linspace(0, m, pools + 1).astype(np.int64)
        assert oracle.count_partitioned(src, dst, off, bounds, workers=2) == rec["triangles"]


def test_ba_big_generator(golden_big):
    """BA(10^6, 9, 0) restated bit-for-bit (reference run: 32 s; here ~1 s)."""
    rec = golden_big["ba_1000000_9_0"]
    pairs = oracle.ba_pairs(rec["n_param"], rec["m_attach"], rec["seed"])
    assert sha(pairs) == rec["edges_sha256"]


def test_rgg_oracle_matches_definition():
    """oracle.rgg_points == numpy default_rng(seed).random((n, 2)); pairs pinned by the
    golden (built with a direct numpy evaluation of the definition)."""
    import json
    import os
    from conftest import GOLDEN_DIR
    xs, ys = oracle.rgg_points(5000, seed=3)
    pts = np.random.default_rng(3).random((5000, 2))
    assert np.array_equal(xs, pts[:, 0]) and np.array_equal(ys, pts[:, 1])
    with open(os.path.join(GOLDEN_DIR, "golden_rgg.json")) as fh:
        cases = json.load(fh)["rgg"]
    for c in cases[:2]:
        pairs = oracle.rgg_pairs(c["n"], c["avg_degree"], seed=c["seed"])
        assert sha(pairs) == c["edges_sha256"]
        og = oracle.preprocess(pairs)
        assert oracle.count(*og) == c["triangles"]


@pytest.mark.parametrize("name", ["rmat_8_4_1", "rmat_10_8_7", "rmat_12_16_99", "rmat_16_76_20240616"])
def test_fast_rmat_matches_reference(golden, name):
    """oracle.rmat_edges (the whole reference rmat loop in C, used for s23-s26 and by the
    reference arm of bench.py) == the reference generator's output, byte for byte."""
    rec = golden["graphs"][name]
    e = oracle.rmat_edges(rec["scale"], rec["edge_factor"], seed=rec["seed"])
    assert sha(e) == rec["edges_sha256"]


def test_fast_rmat_matches_reference_s20_s22(golden_big):
    for scale in (20, 22):
        rec = golden_big[f"rmat_{scale}_16_0"]
        assert sha(oracle.rmat_edges(scale, 16, seed=0)) == rec["edges_sha256"], scale


def test_fast_rmat_matches_reference_s23(golden_huge):
    """s23 (m = 2^27, 2 GB of pairs; ~20 s): the reference's own s23 output, and the oracle's
    CSR + count of it == the reference's (the default GPU schedule turns v-major on here)."""
    rec = golden_huge["rmat_23_16_0"]
    e = oracle.rmat_edges(23, 16, seed=0)
    assert sha(e) == rec["edges_sha256"]
    src, dst, off = oracle.preprocess(e, num_vertices=rec["n"])
    del e
    assert sha(src, dst, off) == rec["csr_sha256"]
    assert oracle.count(src, dst, off) == rec["triangles"]


def test_headline_golden_consistent(golden_s26, golden_big, golden_huge):
    """The s26 record (full oracle run on the GPU host) continues the reference-produced
    s20-s24 series: same generator parameters, n and m per scale, triangles growing."""
    assert golden_s26["m"] == 16 << 26 and golden_s26["pairs"] == 32 << 26
    assert golden_s26["triangles"] == 51_563_396_809
    assert golden_huge["rmat_24_16_0"]["triangles"] < golden_s26["triangles"]
