"""Wedge count and global transitivity (reference metrics.py:1-33).

``wedge_count`` of an edge array runs on the device: the first-column degree histogram
and sum_v C(deg v, 2) in one pass each (tc_wedge_count).  A host ``DegreeOrder`` (what
the reference passes) is accepted too; its degrees are already on the host, so the sum
is exact host integer arithmetic over that array.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .graph import DegreeOrder, EdgeArray

__all__ = ["CountOverflowError", "InconsistentCountsError", "wedge_count", "transitivity"]

_U64_MAX = 2**64 - 1


class CountOverflowError(ArithmeticError):
    """Wedge total exceeds 64 bits; reported instead of wrapping (metrics.py:9-10)."""


class InconsistentCountsError(ValueError):
    """3 * triangles > wedges: the counts cannot come from the same graph (metrics.py:13-14)."""


def _check_u64(total: int, approx: float) -> int:
    if approx >= 2.0**64 * (1 - 1e-12) or total > _U64_MAX:
        raise CountOverflowError(f"wedge count {int(approx) if approx >= 2.0**64 else total} exceeds 64 bits")
    return total


def wedge_count(d) -> int:
    """Number of two-edge paths: sum over vertices of C(deg, 2) (metrics.py:17-24).

    ``d`` is a DegreeOrder (as in the reference), an EdgeArray or a DeviceEdges.
    """
    if isinstance(d, DegreeOrder):
        deg = d.degrees.astype(np.uint64)
        dm1 = deg - (deg > 0)
        c2 = np.where(deg % 2 == 0, (deg // 2) * dm1, deg * (dm1 // 2))  # no u64 wrap
        approx = float(np.sum(deg.astype(np.float64) * dm1.astype(np.float64) * 0.5))
        if approx >= 2.0**63:
            return _check_u64(sum(int(x) * (int(x) - 1) // 2 for x in d.degrees.tolist()), approx)
        return _check_u64(int(c2.sum(dtype=np.uint64)), approx)
    out, approx = ctypes.c_uint64(), ctypes.c_double()
    if hasattr(d, "ptr"):
        _lib.check(_lib.lib().tc_wedge_count(ctypes.c_void_p(d.ptr), d.npairs, d.num_vertices, 1,
                                             ctypes.byref(out), ctypes.byref(approx)))
    else:
        g = d if isinstance(d, EdgeArray) else EdgeArray(d)
        _lib.check(_lib.lib().tc_wedge_count(_lib.ptr(g.edges), g.edges.shape[0], g.num_vertices, 0,
                                             ctypes.byref(out), ctypes.byref(approx)))
    return _check_u64(int(out.value), approx.value)


def transitivity(triangles: int, wedges: int) -> float:
    """Fraction of wedges closed into triangles: 3t / w, 0 when w = 0 (metrics.py:27-33)."""
    if 3 * triangles > wedges:
        raise InconsistentCountsError(f"3 * {triangles} > {wedges}")
    if wedges == 0:
        return 0.0
    return 3 * triangles / wedges
