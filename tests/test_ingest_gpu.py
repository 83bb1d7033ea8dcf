"""GPU parity for the ingest side: text / TRI1 readers,
device validate_edge_array, wedge counts and the `count` command, against outcomes the
reference produced (tests/golden/golden_ingest.json, make_ingest_golden.py)."""
from __future__ import annotations

import base64
import json
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN_DIR, sha

pytestmark = pytest.mark.gpu

tcb = pytest.importorskip("paper_1503_00576_b200")
from paper_1503_00576_b200 import cli, generators  # noqa: E402
from paper_1503_00576_b200 import io as gio  # noqa: E402
from paper_1503_00576_b200.graph import EdgeArray  # noqa: E402


@pytest.fixture(scope="module")
def gi():
    with open(os.path.join(GOLDEN_DIR, "golden_ingest.json")) as fh:
        return json.load(fh)


def _outcome(fn):
    try:
        g = fn()
    except Exception as e:  # noqa: BLE001
        rec = {"error": type(e).__name__, "message": str(e)}
        for attr in ("line", "vertex", "u", "v"):
            if hasattr(e, attr):
                rec[attr] = int(getattr(e, attr))
        return rec
    return {"n": int(g.num_vertices), "pairs": int(g.edges.shape[0]), "sha256": sha(g.edges)}


def test_text_reader_all_modes(gi, tmp_path):
    for name, rec in gi["text"].items():
        path = tmp_path / f"{name}.txt"
        path.write_bytes(rec["text"].encode("utf-8"))
        for mode in gio.READ_MODES:
            assert _outcome(lambda: gio.read_edge_list(path, mode)) == rec[mode], (name, mode)


def test_binary_reader_and_load(gi, tmp_path):
    for name, rec in gi["binary"].items():
        path = tmp_path / f"{name}.bin"
        path.write_bytes(base64.b64decode(rec["blob"]))
        assert _outcome(lambda: gio.read_binary(path)) == rec["read_binary"], name
        for mode in ("strict", "normalize"):
            assert _outcome(lambda: gio.load_graph(path, "binary", mode)) == rec["load_" + mode], (name, mode)
        assert gio.sniff_format(path) == ("binary" if rec["blob"] and
                                          base64.b64decode(rec["blob"])[:4] == b"TRI1" else "text")


def test_validate_random_arrays(gi):
    for i, rec in enumerate(gi["validate"]):
        pairs = np.asarray(rec["input"], dtype=np.uint32).reshape(-1, 2)
        expect = {k: v for k, v in rec.items() if k != "input"}
        assert _outcome(lambda: tcb.validate_edge_array(pairs)) == expect, i


def _first_errors(pairs):
    """numpy restatement of reference graph.py:221-240 (the checker for big arrays)."""
    keys = (pairs[:, 0].astype(np.uint64) << np.uint64(32)) | pairs[:, 1]
    order = np.argsort(keys, kind="stable")
    sk = keys[order]
    dup = sk[1:] == sk[:-1]
    if dup.any():
        return "DuplicateEdgeError", int(order[1:][dup].min())
    rev = (pairs[:, 1].astype(np.uint64) << np.uint64(32)) | pairs[:, 0]
    has = np.isin(rev, keys)
    if not has.all():
        return "AsymmetricEdgeError", int(np.argmin(has))
    return None, None


def test_validate_at_scale_first_offender():
    pairs = oracle.symmetrize(oracle.rmat_pairs(16, 16, seed=5))
    rng = np.random.default_rng(1)
    perm = rng.permutation(pairs.shape[0])
    base = np.ascontiguousarray(pairs[perm])
    assert tcb.validate_edge_array(base).edges.shape == base.shape
    # several duplicates: the earliest SECOND occurrence wins
    dup = base.copy()
    for j, pos in ((100, 900_000), (5, 700_000), (400_000, 600_000)):
        dup[pos] = dup[j]
    kind, idx = _first_errors(dup)
    with pytest.raises(tcb.DuplicateEdgeError) as e:
        tcb.validate_edge_array(dup)
    assert kind == "DuplicateEdgeError" and (e.value.u, e.value.v) == tuple(int(x) for x in dup[idx])
    # missing reverses: the first pair (input order) whose reverse is absent
    asym = np.delete(base, [800_000, 300_000, 1_000_000], axis=0)
    kind, idx = _first_errors(asym)
    with pytest.raises(tcb.AsymmetricEdgeError) as e:
        tcb.validate_edge_array(asym)
    assert kind == "AsymmetricEdgeError" and (e.value.u, e.value.v) == tuple(int(x) for x in asym[idx])
    # self-loops: the first in input order, reported before anything else
    loop = dup.copy()
    loop[123_456] = (7, 7)
    loop[50] = (9, 9)
    with pytest.raises(tcb.SelfLoopError) as e:
        tcb.validate_edge_array(loop)
    assert e.value.vertex == 9


def test_validate_device_resident():
    dev = generators.rmat_device(14, 16, seed=3)
    assert tcb.validate_edge_array(dev) is dev


def test_wedges(gi):
    for name, rec in gi["wedges"].items():
        dev = generators.rmat_device(rec["scale"], rec["edge_factor"], seed=rec["seed"])
        assert tcb.wedge_count(dev) == rec["wedges"], name
        host = dev.to_host()
        assert sha(host.edges) == rec["edges_sha256"]
        assert tcb.wedge_count(host) == rec["wedges"]
        assert tcb.wedge_count(tcb.degrees_of(host)) == rec["wedges"]
    assert tcb.wedge_count(EdgeArray(np.zeros((0, 2), np.uint32))) == 0
    star = EdgeArray([(0, i) for i in range(1, 6)] + [(i, 0) for i in range(1, 6)])
    assert tcb.wedge_count(star) == 10


def test_wedges_and_transitivity_complete_graph():
    k = 3000
    und = np.array([(u, v) for u in range(k) for v in range(u + 1, k)], dtype=np.uint32)
    g = EdgeArray(oracle.symmetrize(und))
    w = tcb.wedge_count(g)
    assert w == k * (k - 1) * (k - 2) // 2
    t = tcb.count_triangles(tcb.preprocess(g))
    assert tcb.transitivity(t, w) == 1.0


def test_count_command(gi, tmp_path, capsys):
    for name, rec in gi["cli"].items():
        path = tmp_path / name
        if rec["format"] == "text":
            path.write_text(rec["text"])
        else:
            gio.write_binary(EdgeArray(oracle.symmetrize(oracle.rmat_pairs(8, 4, seed=1))), path)
        capsys.readouterr()
        rc = cli.main(["count", str(path), "--workers", "2"])
        out, err = capsys.readouterr()
        assert rc == rec["rc"], name
        if "record" in rec:
            lines = out.strip().splitlines()
            kv = dict(tok.split("=", 1) for tok in lines[-1].split())
            assert kv.pop("graph") == str(path)
            for key in ("preprocess_ms", "count_ms", "total_ms"):
                assert float(kv.pop(key)) >= 0
            assert kv == rec["record"], name
            assert lines[0].split(": ", 1)[1] == rec["summary_tail"]
            assert lines[1].startswith("phases: preprocess ")
        else:
            assert err.strip().replace(str(path), "<path>") == rec["stderr"]
    assert cli.main(["count", str(tmp_path / "missing.txt")]) == 1


def test_text_round_trip_multichunk(tmp_path):
    """A ~12 MB file splits into several parser chunks (incl. CRLF); symmetrize must give
    back exactly the reference's rmat edge array."""
    und = oracle.rmat_pairs(16, 16, seed=11)
    full = oracle.symmetrize(und)
    for nl in ("\n", "\r\n"):
        path = tmp_path / "g.txt"
        with open(path, "w", newline="") as fh:
            fh.write("# rmat 16 16 11" + nl)
            fh.writelines(f"{u} {v}{nl}" for u, v in und.tolist())
        g = gio.read_edge_list(path, "symmetrize")
        assert np.array_equal(g.edges, full)
        s = gio.read_edge_list(path, "normalize")
        assert np.array_equal(s.edges, full)
    # an error deep in the file reports the right line
    lines = [f"{u} {v}\n" for u, v in und.tolist()]
    lines[654_321] = "1 2 3\n"
    path.write_text("".join(lines))
    with pytest.raises(gio.ParseError) as e:
        gio.read_edge_list(path)
    assert e.value.line == 654_322 and "expected two fields, got 3" in str(e.value)


def test_binary_round_trip_big(tmp_path):
    dev = generators.rmat_device(18, 16, seed=2)
    host = dev.to_host()
    path = tmp_path / "g.bin"
    gio.write_binary(host, path)
    back = gio.read_binary(path)
    assert np.array_equal(back.edges, host.edges)
    t, _ = tcb.count_with_timings(gio.load_graph(path))
    og = tcb.preprocess(host)
    assert t == tcb.count_triangles(og)
