"""EdgeArray -> OrientedGraph on the B200 (reference preprocess.py:1-84).

``preprocess`` runs the whole pipeline on the device (tc_preprocess): degree histogram,
orientation by (degree, id) with the reverse copy dropped, a hand-written LSD radix sort
of the oriented (u, v) keys whose last pass writes edge_src / edge_dst directly, and the
node-array build.  The result stays in HBM.  The sub-steps the reference exposes
(sort_edges, build_node_array, orient_and_compact, unzip) are available individually
with the reference's host-array signatures; each runs its own kernel(s).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .graph import DegreeOrder, DeviceGraph, EdgeArray, OrientedGraph, _pair_array

__all__ = ["preprocess", "sort_edges", "build_node_array", "orient_and_compact", "unzip",
           "preprocess_with_timings"]


def preprocess_with_timings(g: EdgeArray):
    """preprocess(g) plus the library's event-timed phases (h2d_ms, preprocess_ms)."""
    L = _lib.lib()
    edges = g.edges
    h = ctypes.c_void_p()
    t = _lib.TcTimes()
    _lib.check(L.tc_preprocess(_lib.ptr(edges), edges.shape[0], g.num_vertices, 0,
                               ctypes.byref(h), ctypes.byref(t)))
    return OrientedGraph._from_device(DeviceGraph(h.value)), t


def preprocess(g: EdgeArray) -> OrientedGraph:
    """Full pipeline on a valid EdgeArray (reference preprocess.py:74-84)."""
    return preprocess_with_timings(g)[0]


def sort_edges(g: EdgeArray) -> EdgeArray:
    """Pairs in lexicographic (first, second) order (reference preprocess.py:23-33)."""
    k = g.edges.shape[0]
    if k == 0:
        return g
    out = np.empty((k, 2), dtype=np.uint32)
    _lib.check(_lib.lib().tc_sort_edges(_lib.ptr(g.edges), k, g.num_vertices, _lib.ptr(out)))
    return EdgeArray(out, num_vertices=g.num_vertices)


def build_node_array(sorted_edges, num_vertices: int) -> np.ndarray:
    """offsets[i] = first index whose first vertex is >= i (reference preprocess.py:36-46).

    Accepts a sorted EdgeArray, a (k, 2) pair array or a bare first-vertex column.
    """
    if hasattr(sorted_edges, "edges"):  # an EdgeArray (ours or the reference's)
        sorted_edges = sorted_edges.edges
    arr = np.asarray(sorted_edges)
    firsts = np.ascontiguousarray(arr[:, 0] if arr.ndim == 2 else arr, dtype=np.uint32)
    out = np.empty(int(num_vertices) + 1, dtype=np.int64)
    _lib.check(_lib.lib().tc_build_node_array(_lib.ptr(firsts), firsts.size, int(num_vertices),
                                              _lib.ptr(out)))
    return out


def orient_and_compact(g: EdgeArray, d: DegreeOrder) -> np.ndarray:
    """Pairs with (deg u, u) < (deg v, v), order preserved (reference preprocess.py:49-62)."""
    edges = g.edges
    if edges.size == 0:
        return edges
    degrees = np.ascontiguousarray(d.degrees, dtype=np.int64)
    out = np.empty_like(edges)
    kept = ctypes.c_uint64()
    _lib.check(_lib.lib().tc_orient_and_compact(_lib.ptr(edges), edges.shape[0], _lib.ptr(degrees),
                                                degrees.size, _lib.ptr(out), ctypes.byref(kept)))
    return out[: kept.value]


def unzip(directed) -> tuple[np.ndarray, np.ndarray]:
    """(k, 2) pairs -> contiguous source and destination columns (preprocess.py:65-71).

    A host-side layout change of the caller's host array (the device pipeline fuses
    this into the sort's last pass)."""
    arr = _pair_array(directed) if np.asarray(directed).size else np.zeros((0, 2), np.uint32)
    return np.ascontiguousarray(arr[:, 0]), np.ascontiguousarray(arr[:, 1])
