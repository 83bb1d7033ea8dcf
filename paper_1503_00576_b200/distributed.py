"""Multi-GPU counting: one process per GPU over torch.distributed (NCCL on B200s).

The reference's multi-device analogue is count_partitioned with P pools over contiguous
edge ranges (reference count.py:181-204); the paper replicates the preprocessed arrays
to every GPU and sums the per-GPU counts on the host.  Here:

  1. rank 0 preprocesses into the count-ready rank-space CSR (tc_preprocess_ex);
  2. edge_dst and node_offsets are broadcast to every rank over NVLink (NCCL);
     every rank rebuilds edge_src, its u32 offsets and hubstart locally
     (tc_graph_finalize);
  3. every rank computes the same estimated-work bounds (sum of d+(u) + d+(v) + c,
     SURVEY.md §8(e)) and counts its own contiguous range;
  4. one all-reduce of a single 64-bit count.

The orchestration is written against a small ``Ops`` interface so the same code runs
under gloo on CPU in the tests (with the CPU oracle behind ``Ops``) and under NCCL on
B200s (``B200Ops``, backed by libtcb200).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["Ops", "B200Ops", "count_distributed", "ShardReport"]


class Ops:
    """Device operations the distributed driver needs (implemented by B200Ops)."""

    def preprocess(self, edges):  # -> graph handle
        raise NotImplementedError

    def graph_shape(self, graph) -> tuple[int, int]:  # (m, n)
        raise NotImplementedError

    def empty_graph(self, m: int, n: int):
        raise NotImplementedError

    def replica_tensors(self, graph):  # tensors over (edge_dst, node_offsets) for broadcast
        raise NotImplementedError

    def finalize(self, graph) -> None:
        raise NotImplementedError

    def work_bounds(self, graph, parts: int) -> np.ndarray:
        raise NotImplementedError

    def count_range(self, graph, lo: int, hi: int) -> int:
        raise NotImplementedError

    def sync(self) -> None:
        pass

    def count_tensor(self, value: int):
        import torch
        return torch.tensor([value], dtype=torch.int64)


@dataclass
class ShardReport:
    triangles: int
    local: int
    bounds: tuple
    m: int
    n: int


def count_distributed(ops: Ops, edges=None, group=None, graph=None) -> ShardReport:
    """Count triangles of ``edges`` (held by rank 0) across all ranks of ``group``.

    Every rank must call it; only rank 0 needs ``edges`` (or an existing ``graph``).
    Returns the global count on every rank.
    """
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if world == 1:
        g = graph if graph is not None else ops.preprocess(edges)
        m, n = ops.graph_shape(g)
        total = ops.count_range(g, 0, m) if m else 0
        return ShardReport(total, total, (0, m), m, n)
    # 1. preprocess on rank 0 and share the shape
    if rank == 0:
        g = graph if graph is not None else ops.preprocess(edges)
        m, n = ops.graph_shape(g)
        shape = torch.tensor([m, n], dtype=torch.int64)
    else:
        shape = torch.zeros(2, dtype=torch.int64)
    shape = _to_backend(shape, ops)
    dist.broadcast(shape, src=_global_src(group), group=group)
    m, n = (int(x) for x in shape.cpu().tolist())
    if rank != 0:
        g = ops.empty_graph(m, n)
    # 2. replicate edge_dst + node_offsets, rebuild the rest locally
    ops.sync()
    for t in ops.replica_tensors(g):
        if t.numel():
            dist.broadcast(t, src=_global_src(group), group=group)
    _backend_sync(ops)
    if rank != 0:
        ops.finalize(g)
    # 3. identical work-balanced bounds on every rank; count the local shard
    bounds = ops.work_bounds(g, world)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    local = ops.count_range(g, lo, hi) if hi > lo else 0
    # 4. one 64-bit all-reduce (counts < 2^63, so int64 sum == uint64 sum bit for bit)
    t = _to_backend(ops.count_tensor(local), ops)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    total = int(t.cpu().item())
    return ShardReport(total, local, tuple(int(b) for b in bounds), m, n)


def _global_src(group) -> int:
    import torch.distributed as dist
    return dist.get_global_rank(group, 0) if group is not None else 0


def _to_backend(t, ops):
    dev = getattr(ops, "torch_device", None)
    return t.to(dev) if dev is not None else t


def _backend_sync(ops) -> None:
    dev = getattr(ops, "torch_device", None)
    if dev is not None and dev.type == "cuda":
        import torch
        torch.cuda.synchronize(dev)


class _CudaArray:
    """Minimal __cuda_array_interface__ so torch can alias library-owned HBM."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


class B200Ops(Ops):
    """Ops over libtcb200 on this process's GPU (cuda:LOCAL_RANK)."""

    def __init__(self, device_index: int):
        import torch
        self.torch_device = torch.device("cuda", device_index)
        torch.cuda.set_device(self.torch_device)
        _lib.lib()

    def preprocess(self, edges):
        """Rank-space CSR (count-ready); host edges are uploaded first."""
        from .graph import DeviceGraph
        h = ctypes.c_void_p()
        t = _lib.TcTimes()
        on_dev = hasattr(edges, "ptr")
        ptr = ctypes.c_void_p(edges.ptr) if on_dev else _lib.ptr(edges.edges)
        npairs = edges.npairs if on_dev else edges.edges.shape[0]
        _lib.check(_lib.lib().tc_preprocess_ex(ptr, npairs, edges.num_vertices, 1 if on_dev else 0,
                                               _lib.PREPROCESS_RANK_SPACE, ctypes.byref(h),
                                               ctypes.byref(t)))
        return DeviceGraph(h.value)

    def graph_shape(self, graph):
        return graph.m, graph.n

    def empty_graph(self, m, n):
        from .graph import DeviceGraph
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().tc_graph_create(m, n, _lib.PREPROCESS_RANK_SPACE, ctypes.byref(h)))
        return DeviceGraph(h.value)

    def replica_tensors(self, graph):
        import torch
        _, dst, off = graph.device_pointers()
        out = []
        for ptr, nbytes in ((dst, graph.m * 4), (off, (graph.n + 1) * 8)):
            if nbytes:
                out.append(torch.as_tensor(_CudaArray(ptr, nbytes), device=self.torch_device))
            else:
                out.append(torch.empty(0, dtype=torch.uint8, device=self.torch_device))
        return out

    def finalize(self, graph):
        _lib.check(_lib.lib().tc_graph_finalize(graph.handle))
        m, n, mo = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint32()
        _lib.check(_lib.lib().tc_graph_info(graph.handle, ctypes.byref(m), ctypes.byref(n),
                                            ctypes.byref(mo)))
        graph.max_out = mo.value

    def work_bounds(self, graph, parts):
        b = np.zeros(parts + 1, dtype=np.int64)
        _lib.check(_lib.lib().tc_work_bounds(graph.handle, parts, _lib.ptr(b)))
        return b

    def count_range(self, graph, lo, hi):
        out = ctypes.c_uint64()
        t = _lib.TcTimes()
        _lib.check(_lib.lib().tc_count(graph.handle, int(lo), int(hi), _lib.ALGO_AUTO,
                                       ctypes.byref(out), ctypes.byref(t)))
        return int(out.value)

    def sync(self):
        _lib.check(_lib.lib().tc_synchronize())
