"""Exact triangle counting on the B200 (reference count.py:1-229).

Same entry points, argument meaning and errors as the reference:
``count_triangles(og, num_workers)``, ``count_partitioned(og, plan, workers_per_pool)``,
``count_with_timings(g, num_workers, pools)``, ``intersect_count(og, u, v)``,
``PartitionPlan`` and ``PhaseTimings``.  ``num_workers`` is validated exactly as the
reference does (ValueError below 1) but does not change the device schedule -- the
count is worker-invariant by construction, as in the reference.  Pools are contiguous
edge ranges, each counted by the device kernels restricted to that range; with
torch.distributed initialised, ``paper_1503_00576_b200.distributed`` maps pools to GPUs.
"""
from __future__ import annotations

import ctypes
import os
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .graph import EdgeArray, OrientedGraph

__all__ = ["PhaseTimings", "PartitionPlan", "count_triangles", "count_partitioned",
           "count_with_timings", "intersect_count", "warm_kernel", "default_workers",
           "count_device", "merge_work", "schedule_bytes", "shard_plan", "count_shard"]


@dataclass(frozen=True)
class PhaseTimings:
    """Split between preprocessing (incl. the host->device copy) and counting, in ms."""

    preprocess_ms: float
    count_ms: float
    total_ms: float


@dataclass(frozen=True)
class PartitionPlan:
    """Contiguous split of the oriented edge array into pools (count.py:35-60)."""

    num_pools: int
    bounds: tuple[int, ...]

    @classmethod
    def even(cls, num_pools: int, num_edges: int) -> "PartitionPlan":
        if num_pools < 1:
            raise ValueError("num_pools must be >= 1")
        cuts = np.linspace(0, num_edges, num_pools + 1).astype(np.int64)
        return cls(num_pools, tuple(int(c) for c in cuts))

    @classmethod
    def work_balanced(cls, og: OrientedGraph, num_pools: int) -> "PartitionPlan":
        """Cuts at k/P of the estimated work sum(d+(u) + d+(v) + c)."""
        if num_pools < 1:
            raise ValueError("num_pools must be >= 1")
        dev = _device(og)
        bounds = np.zeros(num_pools + 1, dtype=np.int64)
        _lib.check(_lib.lib().tc_work_bounds(dev.handle, num_pools, _lib.ptr(bounds)))
        return cls(num_pools, tuple(int(b) for b in bounds))

    def pool_range(self, pool: int) -> tuple[int, int]:
        return self.bounds[pool], self.bounds[pool + 1]

    def check_covers(self, num_edges: int) -> None:
        b = self.bounds
        ok = (len(b) == self.num_pools + 1 and b[0] == 0 and b[-1] == num_edges
              and all(x <= y for x, y in zip(b, b[1:])))
        if not ok:
            raise ValueError(f"plan {b} does not cover [0, {num_edges})")


def default_workers() -> int:
    return max(1, os.cpu_count() or 1)


def _resolve_workers(num_workers: int | None) -> int:
    if num_workers is None:
        return default_workers()
    w = int(num_workers)
    if w < 1:
        raise ValueError("num_workers must be >= 1")
    return w


def warm_kernel() -> None:
    """Bind the GPU, create the stream and memory pool outside any timed region
    (the reference JIT-compiles its numba kernel here, count.py:143-150)."""
    _lib.lib()


_foreign = weakref.WeakKeyDictionary()


def _device(og):
    """The device graph of an OrientedGraph -- ours (cached on it), or any object with the
    reference OrientedGraph's arrays (graph.py:146-193), e.g. a tricount.graph.OrientedGraph
    handed over by reference code: uploaded once and cached for the object's lifetime
    (its arrays are read-only).  Callers keep the returned handle alive for the call."""
    if isinstance(og, OrientedGraph):
        return og.device()
    try:
        dev = _foreign.get(og)
    except TypeError:  # not weak-referenceable: upload for this call only
        dev = None
    if dev is None:
        dev = _upload_foreign(og)
        try:
            _foreign[og] = dev
        except TypeError:
            pass
    return dev


def _upload_foreign(og):
    from .graph import DeviceGraph
    src = np.ascontiguousarray(og.edge_src, dtype=np.uint32)
    dst = np.ascontiguousarray(og.edge_dst, dtype=np.uint32)
    off = np.ascontiguousarray(og.node_offsets, dtype=np.int64)
    if src.shape[0] != dst.shape[0]:
        raise ValueError("edge_src and edge_dst lengths differ")
    return DeviceGraph.upload(src, dst, off)


def _count_bounds(og: OrientedGraph, bounds, algo: int):
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    out = ctypes.c_uint64()
    t = _lib.TcTimes()
    dev = _device(og)  # keeps the device graph alive across the call
    _lib.check(_lib.lib().tc_count_partitioned(dev.handle, _lib.ptr(b), b.size - 1, algo,
                                               ctypes.byref(out), ctypes.byref(t)))
    return int(out.value), t


def count_device(og: OrientedGraph, lo: int = 0, hi: int | None = None,
                 algo: int = _lib.ALGO_AUTO):
    """Triangles over oriented edges [lo, hi) plus the library's kernel timings."""
    hi = og.m_dir if hi is None else int(hi)
    out = ctypes.c_uint64()
    t = _lib.TcTimes()
    dev = _device(og)
    _lib.check(_lib.lib().tc_count(dev.handle, int(lo), hi, algo, ctypes.byref(out),
                                   ctypes.byref(t)))
    return int(out.value), t


def count_triangles(g: OrientedGraph, num_workers: int | None = None) -> int:
    """Exact triangle count, identical for every worker count (count.py:162-178)."""
    _resolve_workers(num_workers)
    if g.m_dir == 0:
        return 0
    return count_device(g)[0]


def count_partitioned(g: OrientedGraph, plan: PartitionPlan,
                      workers_per_pool: int | None = None) -> int:
    """Sum of per-pool counts over a covering plan (count.py:181-204)."""
    _resolve_workers(workers_per_pool)
    plan.check_covers(g.m_dir)
    if g.m_dir == 0:
        return 0
    return _count_bounds(g, plan.bounds, _lib.ALGO_AUTO)[0]


def intersect_count(g: OrientedGraph, u: int, v: int) -> int:
    """|adj(u) ∩ adj(v)| over the oriented lists (count.py:102-136)."""
    out = ctypes.c_uint64()
    dev = _device(g)
    _lib.check(_lib.lib().tc_intersect_count(dev.handle, int(u), int(v), ctypes.byref(out)))
    return int(out.value)


def merge_work(g: OrientedGraph) -> int:
    """W = sum over oriented edges of d+(u) + d+(v) (SURVEY.md §8(d) roofline numerator)."""
    out = ctypes.c_uint64()
    dev = _device(g)
    _lib.check(_lib.lib().tc_merge_work(dev.handle, ctypes.byref(out)))
    return int(out.value)


def shard_plan(g: OrientedGraph, parts: int):
    """Multi-GPU shard plan of a full count (tc_shard_plan): (edge_bounds, head_bounds) of the
    rank-space copy.  Shard r = non-v-major edges in its edge range + v-major edges whose
    head is in its head range; count_shard(g, r-th bounds) summed over r is the count."""
    if parts < 1:
        raise ValueError("parts must be >= 1")
    eb = np.zeros(parts + 1, dtype=np.int64)
    hb = np.zeros(parts + 1, dtype=np.int64)
    dev = _device(g)
    _lib.check(_lib.lib().tc_shard_plan(dev.handle, int(parts), _lib.ptr(eb), _lib.ptr(hb)))
    return eb, hb


def count_shard(g: OrientedGraph, lo: int, hi: int, head_lo: int, head_hi: int):
    """One shard of a shard_plan (triangles, library timings)."""
    out = ctypes.c_uint64()
    t = _lib.TcTimes()
    dev = _device(g)
    _lib.check(_lib.lib().tc_count_shard(dev.handle, int(lo), int(hi), int(head_lo), int(head_hi),
                                         ctypes.byref(out), ctypes.byref(t)))
    return int(out.value), t


def schedule_bytes(g: OrientedGraph) -> dict:
    """Compulsory HBM bytes of the full-count schedule, by kernel class (tc_schedule_bytes)."""
    out = np.zeros(5, dtype=np.uint64)
    dev = _device(g)
    _lib.check(_lib.lib().tc_schedule_bytes(dev.handle, _lib.ptr(out)))
    keys = ("vmajor", "umajor_heavy", "light", "per_edge", "heavy_staging")
    return {k: int(v) for k, v in zip(keys, out)}


def count_with_timings(g: EdgeArray, num_workers: int | None = None,
                       pools: int = 1) -> tuple[int, PhaseTimings]:
    """Preprocess then count, with per-phase durations (count.py:207-229).

    Timing starts at edge-array handoff: preprocess_ms includes the host->device copy
    of the pairs.  pools > 1 counts over PartitionPlan.even(pools, m) like the reference.
    Phase times are CUDA-event durations on the library stream.
    """
    _resolve_workers(num_workers)
    if pools < 1:
        raise ValueError("num_pools must be >= 1")
    if pools == 1:
        edges = g.edges
        out = ctypes.c_uint64()
        t = _lib.TcTimes()
        _lib.check(_lib.lib().tc_count_with_timings(_lib.ptr(edges), edges.shape[0],
                                                    g.num_vertices, 0, _lib.ALGO_AUTO,
                                                    ctypes.byref(out), ctypes.byref(t)))
        pre = t.h2d_ms + t.preprocess_ms
        return int(out.value), PhaseTimings(preprocess_ms=pre, count_ms=t.count_ms,
                                            total_ms=t.total_ms)
    from .preprocess import preprocess_with_timings
    og, tp = preprocess_with_timings(g)
    plan = PartitionPlan.even(pools, og.m_dir)
    if og.m_dir == 0:
        triangles, count_ms = 0, 0.0
    else:
        triangles, tc = _count_bounds(og, plan.bounds, _lib.ALGO_AUTO)
        count_ms = tc.count_ms
    pre = tp.h2d_ms + tp.preprocess_ms
    return triangles, PhaseTimings(preprocess_ms=pre, count_ms=count_ms, total_ms=pre + count_ms)


def count_with_timings_device(edges, algo: int = _lib.ALGO_AUTO) -> tuple[int, _lib.TcTimes]:
    """count_with_timings over an edge array already resident in HBM (generators.DeviceEdges):
    no host->device copy; returns the library's raw event timings."""
    out = ctypes.c_uint64()
    t = _lib.TcTimes()
    _lib.check(_lib.lib().tc_count_with_timings(ctypes.c_void_p(edges.ptr), edges.npairs,
                                                edges.num_vertices, 1, algo, ctypes.byref(out),
                                                ctypes.byref(t)))
    return int(out.value), t


def preprocess_device(edges, rank_space: bool = False):
    """preprocess() of a device-resident edge array (generators.DeviceEdges).

    rank_space=True builds the count-ready CSR with vertices relabelled by (degree, id)
    rank (isomorphic to the reference OrientedGraph: same orientation and triangles)."""
    from .graph import DeviceGraph
    h = ctypes.c_void_p()
    t = _lib.TcTimes()
    flags = _lib.PREPROCESS_RANK_SPACE if rank_space else 0
    if isinstance(edges, EdgeArray):  # host pairs (copied in by the library)
        ptr, npairs, on_dev = edges.edges.ctypes.data, edges.edges.shape[0], 0
    else:
        ptr, npairs, on_dev = edges.ptr, edges.npairs, 1
    _lib.check(_lib.lib().tc_preprocess_ex(ctypes.c_void_p(ptr), npairs, edges.num_vertices, on_dev,
                                           flags, ctypes.byref(h), ctypes.byref(t)))
    return OrientedGraph._from_device(DeviceGraph(h.value)), t
