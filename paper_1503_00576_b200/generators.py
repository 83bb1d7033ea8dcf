"""Synthetic inputs for the parity tests and the bench (input production, not timed).

``rmat`` reproduces reference generators.py:203-284 bit-for-bit on the device
(tc_gen_rmat: PCG64 stream positions are jumped to directly, first-occurrence
de-duplication via a stable key/value radix sort); the same seed gives the same
EdgeArray as ``tricount.generators.rmat`` (pinned by sha256 in tests/golden).
Host buffers handed back are pinned (cudaHostAlloc) so the timed host->device copy
in count_with_timings runs at PCIe speed.
"""
from __future__ import annotations

import ctypes
import math
import weakref

import numpy as np

from . import _lib
from .graph import EdgeArray

RMAT_DEFAULT_PROBS = (0.57, 0.19, 0.19, 0.05)
RMAT_DEFAULT_EDGE_FACTOR = 16


def _pcg64_words(seed: int):
    """numpy default_rng(seed)'s PCG64 (state, inc) as (hi, lo) uint64 words."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m = (1 << 64) - 1
    return (s >> 64, s & m), (inc >> 64, inc & m)


class DeviceEdges:
    """An edge array resident in HBM: npairs (u, v) uint32 pairs at ``ptr``."""

    def __init__(self, ptr: int, npairs: int, num_vertices: int):
        self.ptr = int(ptr)
        self.npairs = int(npairs)
        self.num_vertices = int(num_vertices)
        self._fin = weakref.finalize(self, _lib.lib().tc_device_free, ctypes.c_void_p(self.ptr))

    @property
    def nbytes(self) -> int:
        return self.npairs * 8

    def to_host(self, pinned: bool = True) -> EdgeArray:
        arr = pinned_empty((self.npairs, 2), np.uint32) if pinned else np.empty((self.npairs, 2), np.uint32)
        if self.npairs:
            _lib.check(_lib.lib().tc_memcpy(_lib.ptr(arr), ctypes.c_void_p(self.ptr), self.nbytes, 1))
        return EdgeArray(arr, num_vertices=self.num_vertices)

    def free(self) -> None:
        self._fin()


class DeviceEdgesView:
    """Pairs [lo, hi) of a DeviceEdges (a rank's shard); keeps the parent alive, owns nothing."""

    def __init__(self, parent: DeviceEdges, lo: int, hi: int):
        if not 0 <= lo <= hi <= parent.npairs:
            raise ValueError(f"bad shard [{lo}, {hi}) of {parent.npairs} pairs")
        self.parent = parent
        self.ptr = parent.ptr + 8 * int(lo)
        self.npairs = int(hi - lo)
        self.num_vertices = parent.num_vertices

    @property
    def nbytes(self) -> int:
        return self.npairs * 8


class _PinnedOwner:
    def __init__(self, p: int):
        self.p = p
        self._fin = weakref.finalize(self, _lib.lib().tc_host_free, ctypes.c_void_p(p))


def pinned_empty(shape, dtype) -> np.ndarray:
    """numpy array over page-locked host memory (freed with the array)."""
    dtype = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dtype.itemsize
    p = ctypes.c_void_p()
    _lib.check(_lib.lib().tc_host_alloc(max(nbytes, 16), ctypes.byref(p)))
    return pinned_adopt(p.value, shape, dtype)


def pinned_adopt(p: int, shape, dtype) -> np.ndarray:
    """Wrap a library-allocated pinned buffer (tc_host_free'd with the array)."""
    dtype = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dtype.itemsize
    owner = _PinnedOwner(p)
    buf = (ctypes.c_byte * max(nbytes, 16)).from_address(p)
    arr = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)
    # tie the owner's lifetime to the array through the ctypes buffer object
    buf._owner = owner
    return arr


def rmat_device(scale: int, edge_factor: int = RMAT_DEFAULT_EDGE_FACTOR, *,
                probs=RMAT_DEFAULT_PROBS, seed: int = 0) -> DeviceEdges:
    """reference rmat(scale, edge_factor, probs, seed), generated and kept on the device."""
    if not 1 <= scale <= 30:
        raise ValueError(f"scale: must be in 1..30, got {scale}")
    if edge_factor < 1:
        raise ValueError(f"edge_factor: must be >= 1, got {edge_factor}")
    a, b, c, d = (float(x) for x in probs)
    if min(a, b, c, d) < 0 or abs(a + b + c + d - 1.0) > 1e-9:
        raise ValueError(f"probs: must be nonnegative and sum to 1, got {probs}")
    (sh, sl), (ih, il) = _pcg64_words(seed)
    pr = (ctypes.c_double * 4)(a, b, c, d)
    state = (ctypes.c_uint64 * 2)(sh, sl)
    inc = (ctypes.c_uint64 * 2)(ih, il)
    p = ctypes.c_void_p()
    npairs, nverts = ctypes.c_uint64(), ctypes.c_uint64()
    _lib.check(_lib.lib().tc_gen_rmat(int(scale), int(edge_factor), pr, state, inc, ctypes.byref(p),
                                      ctypes.byref(npairs), ctypes.byref(nverts)))
    return DeviceEdges(p.value, npairs.value, nverts.value)


def rmat(scale: int, edge_factor: int = RMAT_DEFAULT_EDGE_FACTOR, *,
         probs=RMAT_DEFAULT_PROBS, seed: int = 0, pinned: bool = True) -> EdgeArray:
    """Host EdgeArray of reference rmat(...) (device-generated, copied back once)."""
    dev = rmat_device(scale, edge_factor, probs=probs, seed=seed)
    try:
        return dev.to_host(pinned=pinned)
    finally:
        dev.free()


def barabasi_albert_device(n: int, m_attach: int, seed: int = 0) -> DeviceEdges:
    """reference barabasi_albert(n, m_attach, seed) (generators.py:287-322), bit-identical;
    the sampling loop is sequential by construction and runs on the host."""
    if n < 2:
        raise ValueError(f"n: must be >= 2, got {n}")
    if not 1 <= m_attach < n:
        raise ValueError(f"m_attach: must satisfy 1 <= m_attach < n, got {m_attach}")
    (sh, sl), (ih, il) = _pcg64_words(seed)
    state = (ctypes.c_uint64 * 2)(sh, sl)
    inc = (ctypes.c_uint64 * 2)(ih, il)
    p = ctypes.c_void_p()
    npairs, nverts = ctypes.c_uint64(), ctypes.c_uint64()
    _lib.check(_lib.lib().tc_gen_ba(int(n), int(m_attach), state, inc, ctypes.byref(p),
                                    ctypes.byref(npairs), ctypes.byref(nverts)))
    return DeviceEdges(p.value, npairs.value, nverts.value)


def rgg_radius(n: int, avg_degree: float = 32.0) -> float:
    """Radius giving expected degree ``avg_degree`` away from the border: sqrt(k / (pi n))."""
    return math.sqrt(avg_degree / (math.pi * n))


def random_geometric_device(n: int, avg_degree: float = 32.0, seed: int = 0,
                            radius: float | None = None) -> DeviceEdges:
    """2-D random geometric graph (BASELINE config 5; SURVEY.md §8(d) recipe).

    Points are numpy ``default_rng(seed).random((n, 2))`` (row i = point i); vertices i, j
    are adjacent iff (xi-xj)**2 + (yi-yj)**2 < radius**2 in float64, radius defaulting to
    sqrt(avg_degree / (pi n)).  No torus wrap.  Pairs in both directions, sorted (the
    reference generators' layout).  The reference has no RGG generator; parity is the
    oracle restatement (oracle.rgg_pairs) and the reference counter on its output.
    """
    if n < 1 or n >= 2**32:
        raise ValueError(f"n: must be in [1, 2^32), got {n}")
    r = rgg_radius(n, avg_degree) if radius is None else float(radius)
    if not 0 < r < 2:
        raise ValueError(f"radius: must be in (0, 2), got {r}")
    (sh, sl), (ih, il) = _pcg64_words(seed)
    state = (ctypes.c_uint64 * 2)(sh, sl)
    inc = (ctypes.c_uint64 * 2)(ih, il)
    p = ctypes.c_void_p()
    npairs, nverts = ctypes.c_uint64(), ctypes.c_uint64()
    _lib.check(_lib.lib().tc_gen_rgg(int(n), r, state, inc, ctypes.byref(p), ctypes.byref(npairs),
                                     ctypes.byref(nverts)))
    return DeviceEdges(p.value or 0, npairs.value, nverts.value)


def random_geometric(n: int, avg_degree: float = 32.0, seed: int = 0, radius: float | None = None,
                     pinned: bool = True) -> EdgeArray:
    """Host EdgeArray of :func:`random_geometric_device`."""
    dev = random_geometric_device(n, avg_degree, seed, radius)
    try:
        return dev.to_host(pinned=pinned)
    finally:
        dev.free()


def barabasi_albert(n: int, m_attach: int, seed: int = 0, pinned: bool = True) -> EdgeArray:
    """Host EdgeArray of reference barabasi_albert(n, m_attach, seed)."""
    dev = barabasi_albert_device(n, m_attach, seed)
    try:
        return dev.to_host(pinned=pinned)
    finally:
        dev.free()


def gnp(n: int, p: float, seed: int = 0) -> EdgeArray:
    """Reference generators.py:186-200 (G(n, p) row by row from numpy default_rng(seed)):
    for every u, the hits of rng.random(n - u - 1) < p are u's higher neighbours; both
    directions, lexicographically sorted.  Host-side input production (BASELINE config 1 is
    G(n = 10^4, p = 10^5 / C(n, 2))); the sort of the symmetrised pairs runs on the device."""
    if n < 0 or not 0.0 <= p <= 1.0:
        raise ValueError("gnp: n >= 0 and 0 <= p <= 1 required")
    rng = np.random.default_rng(seed)
    rows = []
    for u in range(n - 1):
        hits = np.flatnonzero(rng.random(n - u - 1) < p)
        if hits.size:
            rows.append(np.stack([np.full(hits.size, u, np.uint32), (hits + u + 1).astype(np.uint32)], axis=1))
    if not rows:
        return EdgeArray(np.zeros((0, 2), np.uint32), num_vertices=0)
    canon = np.concatenate(rows)
    both = np.ascontiguousarray(np.concatenate([canon, canon[:, ::-1]]))
    from .preprocess import sort_edges
    return sort_edges(EdgeArray(both))


def to_device(g: EdgeArray) -> DeviceEdges:
    """Copy a host edge array into library-owned HBM (untimed input staging)."""
    e = np.ascontiguousarray(g.edges)
    p = ctypes.c_void_p()
    _lib.check(_lib.lib().tc_device_alloc(max(e.nbytes, 16), ctypes.byref(p)))
    if e.size:
        _lib.check(_lib.lib().tc_memcpy(p, _lib.ptr(e), e.nbytes, 0))
    return DeviceEdges(p.value, e.shape[0], g.num_vertices)
