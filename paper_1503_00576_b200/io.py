"""Edge-list files on either side of the hot path (reference io.py).

Same formats, modes and errors as the reference:

* text -- "u v" lines, '#'/'%' comments; modes strict / symmetrize / normalize
  (io.py:51-99).  Parsed by a multi-threaded native parser straight into pinned host
  memory (tc_parse_edge_list); validation and the mode's sort run on the device.
* TRI1 binary -- "TRI1" + u64 count + u32 pairs, little endian (io.py:18-33,127-152),
  read by the library into pinned memory (tc_read_tri1) so the H2D copy that follows
  runs at full PCIe rate.

Returned EdgeArrays are ordinary (read-only) numpy-backed arrays over pinned memory.
"""
from __future__ import annotations

import ctypes
import struct
from pathlib import Path

import numpy as np

from . import _lib
from .generators import pinned_adopt
from .graph import EdgeArray, validate_edge_array
from .preprocess import sort_edges

__all__ = [
    "MAGIC", "READ_MODES", "ParseError", "BadMagicError", "TruncatedFileError",
    "read_edge_list", "write_edge_list", "read_binary", "write_binary", "sniff_format",
    "load_graph", "normalize",
]

MAGIC = b"TRI1"
_HEADER = struct.Struct("<4sQ")

READ_MODES = ("strict", "symmetrize", "normalize")


class ParseError(ValueError):
    def __init__(self, line: int, message: str):
        self.line = line
        super().__init__(f"line {line}: {message}")


class BadMagicError(ValueError):
    pass


class TruncatedFileError(ValueError):
    pass


def _pairs_from(p: int, npairs: int) -> np.ndarray:
    arr = pinned_adopt(p, (npairs, 2), np.uint32)
    arr.flags.writeable = False
    return arr


def _line_message(path, lineno: int) -> str:
    """Rebuild the reference's ParseError text for the failing line (io.py:79-87)."""
    with open(path, "r", encoding="utf-8") as fh:
        for i, raw in enumerate(fh, start=1):
            if i == lineno:
                line = raw.strip()
                tokens = line.split()
                if len(tokens) != 2:
                    return f"expected two fields, got {len(tokens)}"
                try:
                    int(tokens[0]), int(tokens[1])
                except ValueError:
                    return f"not an integer pair: {line!r}"
                return f"vertex id out of unsigned 32-bit range: {line!r}"
    return "parse error"


def _parse_text(path) -> np.ndarray:
    p, n = ctypes.c_void_p(), ctypes.c_uint64()
    line, kind = ctypes.c_uint64(), ctypes.c_int()
    rc = _lib.lib().tc_parse_edge_list(str(path).encode(), ctypes.byref(p), ctypes.byref(n),
                                       ctypes.byref(line), ctypes.byref(kind))
    if rc == -7:
        raise ParseError(int(line.value), _line_message(path, int(line.value)))
    _lib.check(rc)
    return _pairs_from(p.value, int(n.value))


def normalize(edges) -> EdgeArray:
    """Drop self-loops and duplicates, add missing reverses; lexicographic order
    (reference graph.py:245-268).  The sort runs on the device."""
    g = edges if isinstance(edges, EdgeArray) else EdgeArray(edges)
    arr = g.edges
    if arr.size == 0:
        return g
    arr = arr[arr[:, 0] != arr[:, 1]]
    if arr.size == 0:
        return EdgeArray(np.zeros((0, 2), dtype=np.uint32))
    both = np.concatenate([arr, arr[:, ::-1]])
    s = sort_edges(EdgeArray(both)).edges
    keep = np.ones(s.shape[0], dtype=bool)
    keep[1:] = np.any(s[1:] != s[:-1], axis=1)
    return EdgeArray(np.ascontiguousarray(s[keep]))


def read_edge_list(source, mode: str = "symmetrize") -> EdgeArray:
    """Parse a text edge list (reference io.py:51-99): strict keeps file order and
    validates; symmetrize adds reverses, validates, sorts; normalize cleans up."""
    if mode not in READ_MODES:
        raise ValueError(f"unknown mode {mode!r} (choose from {', '.join(READ_MODES)})")
    if not isinstance(source, (str, Path)):
        import os
        import tempfile
        with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False, encoding="utf-8") as fh:
            fh.write(source.read())
        try:
            return read_edge_list(fh.name, mode)
        finally:
            os.unlink(fh.name)
    pairs = _parse_text(source)
    if mode == "strict":
        return validate_edge_array(pairs)
    if mode == "symmetrize":
        if pairs.size == 0:
            return EdgeArray(pairs)
        doubled = np.concatenate([pairs, pairs[:, ::-1]])
        g = validate_edge_array(doubled)
        return sort_edges(g)
    return normalize(pairs)


def write_edge_list(g: EdgeArray, dest, both_directions: bool = False) -> None:
    """Write "u v" lines: u < v once per edge, or every directed pair (io.py:102-118)."""
    if isinstance(dest, (str, Path)):
        with open(dest, "w", encoding="utf-8") as fh:
            write_edge_list(g, fh, both_directions)
            return
    rows = g.edges if both_directions else g.edges[g.edges[:, 0] < g.edges[:, 1]]
    dest.writelines(f"{u} {v}\n" for u, v in rows.tolist())


def write_binary(g: EdgeArray, dest) -> None:
    """Serialize to TRI1 (io.py:127-134); round trips bit-exactly."""
    if isinstance(dest, (str, Path)):
        with open(dest, "wb") as fh:
            write_binary(g, fh)
            return
    dest.write(_HEADER.pack(MAGIC, g.edges.shape[0]))
    dest.write(np.ascontiguousarray(g.edges, dtype="<u4").tobytes())


def read_binary(source) -> EdgeArray:
    """Deserialize a TRI1 file (io.py:137-152) into pinned host memory."""
    if not isinstance(source, (str, Path)):
        data = source.read()
        if len(data) < _HEADER.size:
            raise TruncatedFileError(f"file shorter than the {_HEADER.size}-byte header")
        magic, count = _HEADER.unpack_from(data)
        if magic != MAGIC:
            raise BadMagicError(f"expected magic {MAGIC!r}, got {magic!r}")
        expected = _HEADER.size + 8 * count
        if len(data) != expected:
            raise TruncatedFileError(f"expected {expected} bytes for {count} pairs, got {len(data)}")
        return EdgeArray(np.frombuffer(data, dtype="<u4", offset=_HEADER.size).reshape(-1, 2))
    p, n = ctypes.c_void_p(), ctypes.c_uint64()
    rc = _lib.lib().tc_read_tri1(str(source).encode(), ctypes.byref(p), ctypes.byref(n))
    if rc in (-5, -6):
        with open(source, "rb") as fh:  # re-raise with the reference's exact message
            return read_binary(fh)
    _lib.check(rc)
    return EdgeArray(_pairs_from(p.value, int(n.value)))


def sniff_format(path) -> str:
    """'binary' if the file starts with the TRI1 magic, else 'text' (io.py:155-159)."""
    with open(path, "rb") as fh:
        return "binary" if fh.read(4) == MAGIC else "text"


def load_graph(path, fmt: str = "auto", mode: str = "symmetrize") -> EdgeArray:
    """Read either format (io.py:162-178); binary pairs are validated as stored unless
    mode is normalize."""
    if fmt == "auto":
        fmt = sniff_format(path)
    if fmt == "text":
        return read_edge_list(path, mode)
    if fmt == "binary":
        g = read_binary(path)
        return normalize(g) if mode == "normalize" else validate_edge_array(g)
    raise ValueError(f"unknown format {fmt!r}")
