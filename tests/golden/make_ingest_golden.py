"""Golden outcomes for the ingest side of the path.

Run in a container with the reference mounted (not needed at test time):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_ingest_golden.py

For every case the reference itself (tricount.io / graph / metrics / cli) decides the
outcome: either the resulting edge array (sha256 + vertex count) or the exception class,
message and attributes.  Cases: text edge lists in all three read modes (comments, CR /
CRLF, signs, underscores, ranges, field counts ...), TRI1 blobs (bad magic, truncation,
trailing bytes, invalid contents), random pair arrays for validate_edge_array, wedge
counts, and the `count` command's key=value record (timing fields dropped).
Output: tests/golden/golden_ingest.json.
"""
from __future__ import annotations

import base64
import contextlib
import hashlib
import io as pyio
import json
import os
import sys
import tempfile

import numpy as np

from tricount import cli
from tricount import io as gio
from tricount.generators import rmat
from tricount.graph import degrees_of, validate_edge_array
from tricount.metrics import wedge_count

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def outcome(fn):
    try:
        g = fn()
    except Exception as e:  # noqa: BLE001 - recording the reference's behaviour
        rec = {"error": type(e).__name__, "message": str(e)}
        for attr in ("line", "vertex", "u", "v"):
            if hasattr(e, attr):
                rec[attr] = int(getattr(e, attr))
        return rec
    return {"n": int(g.num_vertices), "pairs": int(g.edges.shape[0]), "sha256": sha(g.edges)}


TEXT_CASES = {
    "k3_once": "0 1\n1 2\n0 2\n",
    "k3_both": "0 1\n1 0\n1 2\n2 1\n0 2\n2 0\n",
    "comments_blank": "# header\n\n% also a comment\n0 1\n   \n1 2 \n\t2 0\n",
    "crlf": "0 1\r\n1 2\r\n2 0\r\n",
    "lone_cr": "0 1\r1 2\r2 0\r",
    "no_trailing_newline": "0 1\n1 2\n2 0",
    "tabs_spaces": "0\t1\n1   2\n  2 \t 0  \n",
    "plus_sign": "+0 1\n1 +2\n",
    "underscore": "1_0 2\n2 3\n",
    "bad_underscore": "1__0 2\n",
    "trailing_underscore": "10_ 2\n",
    "minus_zero": "-0 1\n1 2\n",
    "negative": "0 1\n-1 2\n",
    "too_big": "0 1\n4294967296 2\n",
    "max_id": "0 4294967295\n",
    "three_fields": "0 1\n1 2 3\n",
    "one_field": "0 1\n7\n",
    "not_int": "0 1\n1 x\n",
    "float": "0 1.0\n",
    "hex": "0x1 2\n",
    "syntax_beats_range": "99999999999 abc\n",
    "empty": "",
    "only_comments": "# nothing\n% here\n",
    "self_loop": "0 1\n2 2\n",
    "duplicate_once": "0 1\n1 2\n0 1\n",
    "reverse_listed": "0 1\n1 0\n",
    "sparse_ids": "5 1000\n1000 77\n",
    "unit_separator_ws": "0\x1f1\n1 2\n",
    "comment_after_ws": "   # indented comment\n0 1\n",
    "hash_inside": "0 1 # trailing\n",
    "crlf_error_line": "0 1\r\n\r\n1 x\r\n",
    "mixed_breaks_error": "0 1\r1 2\n\r\n3 y\n",
}


def text_cases():
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for name, body in TEXT_CASES.items():
            path = os.path.join(d, name + ".txt")
            with open(path, "w", encoding="utf-8", newline="") as fh:
                fh.write(body)
            rec = {"text": body}
            for mode in gio.READ_MODES:
                rec[mode] = outcome(lambda: gio.read_edge_list(path, mode))
            out[name] = rec
    return out


def tri1(pairs, count=None, magic=b"TRI1", extra=b"", cut=None) -> bytes:
    arr = np.asarray(pairs, dtype="<u4").reshape(-1, 2)
    blob = magic + np.uint64(arr.shape[0] if count is None else count).tobytes() + arr.tobytes() + extra
    return blob if cut is None else blob[:cut]


def binary_cases():
    k3 = [(0, 1), (1, 0), (1, 2), (2, 1), (0, 2), (2, 0)]
    blobs = {
        "k3": tri1(k3),
        "empty": tri1([]),
        "bad_magic": tri1(k3, magic=b"TRI2"),
        "short_header": b"TRI1\x01\x00",
        "truncated": tri1(k3, cut=12 + 8 * 5 + 3),
        "trailing": tri1(k3, extra=b"\x00"),
        "count_too_big": tri1(k3, count=7),
        "self_loop": tri1([(0, 1), (1, 0), (3, 3)]),
        "duplicate": tri1([(0, 1), (1, 0), (0, 1)]),
        "asymmetric": tri1([(0, 1), (1, 0), (1, 2)]),
        "unsorted_valid": tri1([(2, 0), (0, 1), (1, 2), (0, 2), (1, 0), (2, 1)]),
        "dup_loops_for_normalize": tri1([(0, 1), (0, 1), (1, 1), (2, 0)]),
    }
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for name, blob in blobs.items():
            path = os.path.join(d, name + ".bin")
            with open(path, "wb") as fh:
                fh.write(blob)
            rec = {"blob": base64.b64encode(blob).decode()}
            rec["read_binary"] = outcome(lambda: gio.read_binary(path))
            for mode in ("strict", "normalize"):
                rec["load_" + mode] = outcome(lambda: gio.load_graph(path, "binary", mode))
            out[name] = rec
    return out


def validation_cases(seed: int = 20261017, count: int = 300):
    """Random small pair arrays, biased towards each failure kind."""
    rng = np.random.default_rng(seed)
    out = []
    for i in range(count):
        n = int(rng.integers(2, 12))
        k = int(rng.integers(1, 10))
        und = rng.integers(0, n, size=(k, 2))
        und = und[und[:, 0] != und[:, 1]]
        pairs = np.concatenate([und, und[:, ::-1]]) if und.size else np.zeros((0, 2), np.int64)
        kind = i % 5
        if kind == 1 and pairs.size:  # drop a random entry -> asymmetric
            pairs = np.delete(pairs, int(rng.integers(0, pairs.shape[0])), axis=0)
        elif kind == 2:  # self-loop somewhere
            v = int(rng.integers(0, n))
            pos = int(rng.integers(0, pairs.shape[0] + 1))
            pairs = np.insert(pairs, pos, [v, v], axis=0)
        elif kind == 3 and pairs.size:  # duplicate an entry later in the array
            j = int(rng.integers(0, pairs.shape[0]))
            pos = int(rng.integers(j + 1, pairs.shape[0] + 1))
            pairs = np.insert(pairs, pos, pairs[j], axis=0)
        perm = rng.permutation(pairs.shape[0])
        pairs = pairs[perm].astype(np.uint32)
        if pairs.size == 0:
            continue
        rec = outcome(lambda: validate_edge_array(pairs))
        rec["input"] = pairs.tolist()
        out.append(rec)
    return out


def wedge_cases():
    out = {}
    for name, (s, ef, sd) in {"rmat_10_8_7": (10, 8, 7), "rmat_14_16_3": (14, 16, 3)}.items():
        g = rmat(s, ef, seed=sd)
        out[name] = {"scale": s, "edge_factor": ef, "seed": sd, "n": g.num_vertices,
                     "edges_sha256": sha(g.edges), "wedges": wedge_count(degrees_of(g))}
    return out


def cli_cases():
    """`count` record minus timing fields, for text and binary inputs."""
    out = {}
    graphs = {
        "k5.txt": ("text", "".join(f"{u} {v}\n" for u in range(5) for v in range(u + 1, 5))),
        "path.txt": ("text", "0 1\n1 2\n2 3\n"),
        "empty.txt": ("text", "# no edges\n"),
        "tri_plus_tail.txt": ("text", "0 1\n1 2\n2 0\n2 3\n3 4\n"),
        "selfloop.txt": ("text", "0 1\n1 1\n"),
        "rmat8.bin": ("binary", None),
    }
    with tempfile.TemporaryDirectory() as d:
        for name, (fmt, body) in graphs.items():
            path = os.path.join(d, name)
            if fmt == "text":
                with open(path, "w", encoding="utf-8") as fh:
                    fh.write(body)
            else:
                gio.write_binary(rmat(8, 4, seed=1), path)
            stdout, stderr = pyio.StringIO(), pyio.StringIO()
            with contextlib.redirect_stdout(stdout), contextlib.redirect_stderr(stderr):
                rc = cli.main(["count", path, "--workers", "2"])
            rec = {"format": fmt, "text": body, "rc": rc}
            lines = stdout.getvalue().strip().splitlines()
            if lines:
                kv = dict(tok.split("=", 1) for tok in lines[-1].split())
                for key in ("preprocess_ms", "count_ms", "total_ms", "graph"):
                    kv.pop(key, None)
                rec["record"] = kv
                rec["summary_tail"] = lines[0].split(": ", 1)[1]
            else:
                rec["stderr"] = stderr.getvalue().strip().replace(path, "<path>")
            out[name] = rec
    return out


def main() -> None:
    golden = {
        "text": text_cases(),
        "binary": binary_cases(),
        "validate": validation_cases(),
        "wedges": wedge_cases(),
        "cli": cli_cases(),
    }
    with open(os.path.join(HERE, "golden_ingest.json"), "w") as fh:
        json.dump(golden, fh, indent=1, sort_keys=True)
    kinds = {}
    for rec in golden["validate"]:
        kinds[rec.get("error", "ok")] = kinds.get(rec.get("error", "ok"), 0) + 1
    print("validation outcomes:", kinds, file=sys.stderr)


if __name__ == "__main__":
    main()
