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

``count_distributed_sharded`` is the v2 path:
no serial preprocessing.  Every rank holds a shard of the edge array (its slice of the
pairs, device-resident or copied from host memory by that rank alone):

  1. shard degree histograms -> all-reduce -> global degrees (every rank);
  2. each rank ranks the vertices by (degree, id) itself (same result everywhere),
     orients + relabels its shard and sorts it locally; out-degrees -> all-reduce;
  3. node_offsets from the global out-degrees; source-rank ranges balanced by edges;
  4. all-to-all: every key goes to the rank owning its source range;
  5. each rank sorts what it received into its slice of edge_dst; the slices are
     all-gathered (one all_gather_into_tensor over slices padded to the longest);
     every rank finalises the same CSR;
  6. work-balanced shards + one 64-bit all-reduce, as in v1.

The orchestration is written against a small ``Ops`` interface so the same code runs
under gloo on CPU in the tests (with the CPU oracle behind ``Ops``) and under NCCL on
B200s (``B200Ops``, backed by libtcb200).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["Ops", "B200Ops", "count_distributed", "count_distributed_sharded", "ShardReport",
           "shard_bounds"]


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

    def shard_plan(self, graph, parts: int):
        """(edge_bounds, head_bounds), parts + 1 entries each.  Default: work-balanced edge
        ranges, every head in shard 0's head range (no v-major split)."""
        _, n = self.graph_shape(graph)
        return self.work_bounds(graph, parts), np.array([0] + [n] * parts, dtype=np.int64)

    def count_shard(self, graph, lo: int, hi: int, hlo: int, hhi: int) -> int:
        return self.count_range(graph, lo, hi) if hi > lo else 0

    def count_shard_timed(self, graph, lo: int, hi: int, hlo: int, hhi: int):
        """(count, edge-side ms, head-side ms) of one shard."""
        return self.count_shard(graph, lo, hi, hlo, hhi), 0.0, 0.0

    def make_planner(self, graph, parts: int):
        """A ShardPlanner for repeated counts of this graph, or None (static plan only)."""
        return None

    def sync(self) -> None:
        pass

    def count_tensor(self, value: int):
        import torch
        return torch.tensor([value], dtype=torch.int64)

    # ---- v2 (sharded preprocessing); tensors returned/accepted are "comm" tensors,
    # i.e. ready for the process group's backend
    def stage(self, shard):  # host shard -> device copy (once per call); device shards as-is
        return shard

    def shard_degrees(self, shard, n: int):  # -> int32[n]
        raise NotImplementedError

    def shard_orient(self, shard, n: int, deg):  # -> (keys, nkeys, outdeg int32[n])
        raise NotImplementedError

    def create_graph(self, m: int, n: int):
        raise NotImplementedError

    def layout(self, graph, outdeg, parts: int):  # -> (cuts[parts+1], edge_cuts[parts+1])
        raise NotImplementedError

    def split(self, keys, nkeys: int, n: int, cuts, parts: int):  # -> counts[parts]
        raise NotImplementedError

    def send_tensor(self, keys, nkeys: int):  # int64[nkeys]
        raise NotImplementedError

    def recv_tensor(self, k: int):  # int64[k]
        raise NotImplementedError

    def place(self, graph, recv, k: int, pos: int) -> None:
        raise NotImplementedError

    def dst_slice(self, graph, lo: int, hi: int):  # int32[hi-lo] view/copy of edge_dst[lo:hi]
        raise NotImplementedError

    def dst_write(self, graph, lo: int, t) -> None:  # edge_dst[lo:lo+len(t)] = t
        raise NotImplementedError

    def comm_empty(self, k: int):  # int32[k] tensor the process group can use
        import torch
        return torch.empty(k, dtype=torch.int32)

    def free_keys(self, keys) -> None:
        pass


@dataclass
class ShardReport:
    triangles: int
    local: int
    bounds: tuple
    m: int
    n: int
    head_bounds: tuple = ()


def count_distributed(ops: Ops, edges=None, group=None, graph=None, plans: dict | None = None) -> ShardReport:
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
    # 3. identical shard plan on every rank (edge ranges for the u-major / light work, head
    #    ranges for the v-major work); count the local shard
    return _count_local_shard(ops, g, rank, world, group, m, n, plans)


def refine_plan(edge_bounds, head_bounds, edge_ms, head_ms, head_floor: int = 0):
    """One measurement-guided refinement of a shard plan: within every shard the measured time
    of each side (edge side: u-major + light kernels; head side: the v-major phase) is
    assumed spread uniformly over its index range, and both sides are re-cut at equal
    cumulative time.  Used for repeated counts of one graph (the first count's per-rank
    times, all-gathered, refine the plan for the next); the cost-model plan (tc_shard_plan)
    is the starting point.  ``head_floor``: first head that can carry v-major work (the
    v-major zone start; heads below it count for nothing)."""
    def recut(bounds, ms):
        bounds = [int(b) for b in bounds]
        P = len(bounds) - 1
        ms = [max(float(t), 1e-9) for t in ms]
        cum = [0.0]
        for t in ms:
            cum.append(cum[-1] + t)
        total = cum[-1]
        out = [bounds[0]]
        r = 0
        for k in range(1, P):
            target = total * k / P
            while r < P - 1 and cum[r + 1] < target:
                r += 1
            frac = (target - cum[r]) / ms[r]
            x = bounds[r] + int(round(frac * (bounds[r + 1] - bounds[r])))
            out.append(max(out[-1], min(x, bounds[-1])))
        out.append(bounds[-1])
        return np.array(out, dtype=np.int64)
    hb = [int(b) for b in head_bounds]
    lo = hb[0]
    hb[0] = max(lo, min(int(head_floor), hb[1]))
    out_h = recut(hb, head_ms)
    out_h[0] = lo
    return recut(edge_bounds, edge_ms), out_h


class ShardPlanner:
    """The shard plan of tc_shard_plan, held on the host as its model costs (per-tile edge-side
    costs, per-head head-side costs) so it can be refined by measurement: after a count, each
    shard's measured time per side (minus a fixed per-shard cost) over its model cost gives a
    correction factor applied to that shard's cost range, and both sides are re-cut at equal
    corrected cost.  Identical inputs give identical plans on every rank (the measured times
    are all-gathered first).  For repeated counts of one graph (bench steps, a service)."""

    def __init__(self, ecost, tile: int, hcost, z0: int, m: int, n: int, parts: int,
                 head_fixed_ms: float = 2.9, edge_fixed_ms: float = 0.1):
        self.parts, self.tile, self.z0, self.m, self.n = parts, int(tile), int(z0), int(m), int(n)
        self.ecost = np.asarray(ecost, dtype=np.float64).copy()
        self.hcost = np.asarray(hcost, dtype=np.float64).copy()
        self.hfix, self.efix = head_fixed_ms, edge_fixed_ms
        self.ecut = self._cut(self.ecost)
        self.hcut = self._cut(self.hcost)

    @classmethod
    def from_device(cls, graph, parts: int) -> "ShardPlanner":
        """From a device graph's model costs (tc_shard_costs); graph has .handle, .m, .n."""
        h = graph.handle
        L = _lib.lib()
        nt, tile, nz = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        z0 = ctypes.c_uint32()
        _lib.check(L.tc_shard_cost_sizes(h, parts, ctypes.byref(nt), ctypes.byref(tile), ctypes.byref(nz),
                                         ctypes.byref(z0)))
        et = np.zeros(max(nt.value, 1), np.uint64)
        hc = np.zeros(max(nz.value, 1), np.uint64)
        _lib.check(L.tc_shard_costs(h, parts, _lib.ptr(et), _lib.ptr(hc)))
        return cls(et[:nt.value], tile.value, hc[:nz.value], z0.value, graph.m, graph.n, parts)

    def _cut(self, cost):
        P = self.parts
        c = np.cumsum(cost)
        total = c[-1] if c.size else 0.0
        cut = [0]
        for k in range(1, P):
            i = int(np.searchsorted(c, total * k / P, side="left")) + 1 if total > 0 else cost.size
            cut.append(min(max(i, cut[-1]), cost.size))
        cut.append(cost.size)
        return cut

    def bounds(self):
        eb = np.array([min(i * self.tile, self.m) for i in self.ecut], dtype=np.int64)
        hb = np.array([self.z0 + i for i in self.hcut], dtype=np.int64)
        hb[0], hb[-1] = 0, self.n
        return eb, hb

    def refine(self, edge_ms, head_ms):
        for cost, cut, ms, fix in ((self.ecost, self.ecut, edge_ms, self.efix),
                                   (self.hcost, self.hcut, head_ms, self.hfix)):
            for r in range(self.parts):
                a, b = cut[r], cut[r + 1]
                model = cost[a:b].sum()
                if b > a and model > 0:
                    cost[a:b] *= max(float(ms[r]) - fix, 1e-3) / model
        self.ecut = self._cut(self.ecost)
        self.hcut = self._cut(self.hcost)
        return self.bounds()


def shard_bounds(npairs: int, world: int) -> list[int]:
    """Contiguous pair ranges [b[r], b[r+1]) of an edge array split over ``world`` ranks."""
    return [npairs * r // world for r in range(world + 1)]


def count_distributed_sharded(ops: Ops, shard, num_vertices: int, group=None,
                              plans: dict | None = None) -> ShardReport:
    """Triangles of the edge array whose shards the ranks of ``group`` hold (v2: sharded
    preprocessing, no serial step).  ``shard`` is this rank's slice of the pairs (any
    split works: the result does not depend on it); ``num_vertices`` is the global
    vertex count, identical on every rank.  Returns the global count on every rank."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    n = int(num_vertices)
    shard = ops.stage(shard)  # host shards: this rank's H2D copy, once
    # 1. global degrees
    deg = ops.shard_degrees(shard, n)
    dist.all_reduce(deg, op=dist.ReduceOp.SUM, group=group)
    _backend_sync(ops)
    # 2. local orientation in rank space; global out-degrees and m
    keys, nkeys, outdeg = ops.shard_orient(shard, n, deg)
    del deg
    dist.all_reduce(outdeg, op=dist.ReduceOp.SUM, group=group)
    mt = _to_backend(torch.tensor([nkeys], dtype=torch.int64), ops)
    dist.all_reduce(mt, op=dist.ReduceOp.SUM, group=group)
    _backend_sync(ops)
    m = int(mt.cpu().item())
    # 3. offsets + source ranges
    g = ops.create_graph(m, n)
    cuts, ecuts = ops.layout(g, outdeg, world)
    del outdeg
    # 4. all-to-all of the keys by source range
    send_counts = [int(c) for c in ops.split(keys, nkeys, n, cuts, world)]
    sc = _to_backend(torch.tensor(send_counts, dtype=torch.int64), ops)
    rc = _to_backend(torch.empty(world, dtype=torch.int64), ops)
    dist.all_to_all_single(rc, sc, group=group)
    _backend_sync(ops)
    recv_counts = [int(c) for c in rc.cpu().tolist()]
    k = sum(recv_counts)
    if k != int(ecuts[rank + 1] - ecuts[rank]):
        raise RuntimeError("all-to-all delivered a different edge count than the layout")
    recv = ops.recv_tensor(k)
    send = ops.send_tensor(keys, nkeys)
    dist.all_to_all_single(recv, send, output_split_sizes=recv_counts,
                           input_split_sizes=send_counts, group=group)
    _backend_sync(ops)
    del send
    ops.free_keys(keys)
    # 5. sort the received keys into this rank's slice of edge_dst; all-gather the slices
    ops.place(g, recv, k, int(ecuts[rank]))
    del recv
    # one all-gather of the edge_dst slices (padded to the longest; the layout balances
    # them by edge count, so the padding is at most one adjacency list)
    lens = [int(ecuts[r + 1] - ecuts[r]) for r in range(world)]
    L = max(lens)
    if L:
        ops.sync()
        send = ops.comm_empty(L)
        if lens[rank]:
            send[:lens[rank]].copy_(ops.dst_slice(g, int(ecuts[rank]), int(ecuts[rank + 1])))
        gathered = ops.comm_empty(world * L)
        dist.all_gather_into_tensor(gathered, send, group=group)
        _backend_sync(ops)
        del send
        for r in range(world):
            if r != rank and lens[r]:
                ops.dst_write(g, int(ecuts[r]), gathered[r * L:r * L + lens[r]])
        del gathered
    ops.finalize(g)
    # 6. count the local shard; one all-reduce
    return _count_local_shard(ops, g, rank, world, group, m, n, plans)


def _count_local_shard(ops: Ops, g, rank: int, world: int, group, m: int, n: int,
                       plans: dict | None = None) -> ShardReport:
    """This rank's shard of the plan every rank computes identically, then one 64-bit
    all-reduce (counts < 2^63, so the int64 sum equals the uint64 sum bit for bit).  With
    ``plans`` (a dict the caller keeps across counts of the same graph) the plan is a
    ShardPlanner refined after every count by the all-gathered per-rank phase times."""
    import torch
    import torch.distributed as dist
    key = (m, n, world)
    planner = None
    if plans is not None:
        if key not in plans:
            plans[key] = ops.make_planner(g, world)
        planner = plans[key]
    eb, hb = planner.bounds() if planner is not None else ops.shard_plan(g, world)
    lo, hi = int(eb[rank]), int(eb[rank + 1])
    hlo, hhi = int(hb[rank]), int(hb[rank + 1])
    local, edge_ms, head_ms = ops.count_shard_timed(g, lo, hi, hlo, hhi)
    t = _to_backend(ops.count_tensor(local), ops)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    total = int(t.cpu().item())
    if planner is not None:
        times = torch.zeros(2 * world, dtype=torch.float64)
        times[2 * rank], times[2 * rank + 1] = edge_ms, head_ms
        times = _to_backend(times, ops)
        dist.all_reduce(times, op=dist.ReduceOp.SUM, group=group)
        tt = times.cpu().numpy()
        planner.refine(tt[0::2], tt[1::2])
    return ShardReport(total, local, tuple(int(b) for b in eb), m, n, tuple(int(b) for b in hb))


def _global_src(group) -> int:
    import torch.distributed as dist
    return dist.get_global_rank(group, 0) if group is not None else 0


def _to_backend(t, ops):
    dev = getattr(ops, "comm_device", None)
    return t.to(dev) if dev is not None else t


def _backend_sync(ops) -> None:
    dev = getattr(ops, "comm_device", None)
    if dev is not None and dev.type == "cuda":
        import torch
        torch.cuda.synchronize(dev)


class _CudaArray:
    """Minimal __cuda_array_interface__ so torch can alias library-owned HBM."""

    def __init__(self, ptr: int, count: int, typestr: str = "|u1"):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


class _Keys:
    """Library-allocated device buffer of sorted rank-space keys (tc_device_free'd)."""

    def __init__(self, ptr: int):
        import weakref
        self.ptr = int(ptr)
        self._fin = weakref.finalize(self, _lib.lib().tc_device_free, ctypes.c_void_p(self.ptr))

    def free(self):
        self._fin()


class B200Ops(Ops):
    """Ops over libtcb200 on this process's GPU (cuda:LOCAL_RANK).

    ``comm="cuda"`` (NCCL) hands device tensors to the collectives, aliasing library
    memory where it can; ``comm="cpu"`` stages every collective through host memory so
    several processes can share one GPU under gloo (the single-GPU test of the v2 path).
    """

    def __init__(self, device_index: int, comm: str = "cuda"):
        import torch
        self.torch_device = torch.device("cuda", device_index)
        self.comm_device = self.torch_device if comm == "cuda" else None
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

    def shard_plan(self, graph, parts):
        eb = np.zeros(parts + 1, dtype=np.int64)
        hb = np.zeros(parts + 1, dtype=np.int64)
        _lib.check(_lib.lib().tc_shard_plan(graph.handle, parts, _lib.ptr(eb), _lib.ptr(hb)))
        return eb, hb

    def count_shard(self, graph, lo, hi, hlo, hhi):
        return self.count_shard_timed(graph, lo, hi, hlo, hhi)[0]

    def count_shard_timed(self, graph, lo, hi, hlo, hhi):
        out = ctypes.c_uint64()
        t = _lib.TcTimes()
        _lib.check(_lib.lib().tc_count_shard(graph.handle, int(lo), int(hi), int(hlo), int(hhi),
                                             ctypes.byref(out), ctypes.byref(t)))
        return int(out.value), t.count_ms - t.vmajor_ms, t.vmajor_ms

    def make_planner(self, graph, parts):
        try:
            return ShardPlanner.from_device(graph, parts)
        except ValueError:  # no v-major split for this graph: the static plan
            return None

    # ---- v2 -----------------------------------------------------------------------
    def _out(self, t):
        return t if self.comm_device is not None else t.cpu()

    def _in(self, t):
        import torch
        if t.is_cuda:
            torch.cuda.synchronize(self.torch_device)
            return t
        return t.to(self.torch_device)

    @staticmethod
    def _shard_args(shard):
        if hasattr(shard, "ptr"):
            return ctypes.c_void_p(shard.ptr), int(shard.npairs), 1
        arr = shard.edges if hasattr(shard, "edges") else shard
        return _lib.ptr(arr), int(arr.shape[0]), 0

    def stage(self, shard):
        if hasattr(shard, "ptr"):
            return shard
        from .generators import DeviceEdges
        arr = shard.edges if hasattr(shard, "edges") else shard
        arr = np.ascontiguousarray(arr, dtype=np.uint32)
        p = ctypes.c_void_p()
        _lib.check(_lib.lib().tc_device_alloc(max(arr.nbytes, 16), ctypes.byref(p)))
        d = DeviceEdges(p.value, arr.shape[0], 0)
        if arr.size:
            _lib.check(_lib.lib().tc_memcpy(p, _lib.ptr(arr), arr.nbytes, 0))
        return d

    def shard_degrees(self, shard, n):
        import torch
        deg = torch.empty(max(n, 1), dtype=torch.int32, device=self.torch_device)[:n]
        p, k, on_dev = self._shard_args(shard)
        torch.cuda.synchronize(self.torch_device)
        _lib.check(_lib.lib().tc_dist_degrees(p, k, on_dev, n, ctypes.c_void_p(deg.data_ptr())))
        return self._out(deg)

    def shard_orient(self, shard, n, deg):
        import torch
        deg = self._in(deg)
        outdeg = torch.empty(max(n, 1), dtype=torch.int32, device=self.torch_device)[:n]
        p, k, on_dev = self._shard_args(shard)
        kp, nk = ctypes.c_void_p(), ctypes.c_uint64()
        _lib.check(_lib.lib().tc_dist_orient(p, k, on_dev, n, ctypes.c_void_p(deg.data_ptr()),
                                             ctypes.byref(kp), ctypes.byref(nk),
                                             ctypes.c_void_p(outdeg.data_ptr())))
        return _Keys(kp.value or 0), int(nk.value), self._out(outdeg)

    def create_graph(self, m, n):
        return self.empty_graph(m, n)

    def layout(self, graph, outdeg, parts):
        outdeg = self._in(outdeg)
        cuts = np.zeros(parts + 1, dtype=np.int64)
        ecuts = np.zeros(parts + 1, dtype=np.int64)
        _lib.check(_lib.lib().tc_dist_layout(graph.handle, ctypes.c_void_p(outdeg.data_ptr()), parts,
                                             _lib.ptr(cuts), _lib.ptr(ecuts)))
        return cuts, ecuts

    def split(self, keys, nkeys, n, cuts, parts):
        counts = np.zeros(parts, dtype=np.int64)
        c = np.ascontiguousarray(cuts, dtype=np.int64)
        _lib.check(_lib.lib().tc_dist_split(ctypes.c_void_p(keys.ptr), nkeys, n, _lib.ptr(c), parts,
                                            _lib.ptr(counts)))
        return counts

    def send_tensor(self, keys, nkeys):
        import torch
        if nkeys == 0:
            return self._out(torch.empty(0, dtype=torch.int64, device=self.torch_device))
        t = torch.as_tensor(_CudaArray(keys.ptr, nkeys, "<i8"), device=self.torch_device)
        return self._out(t)

    def recv_tensor(self, k):
        import torch
        return torch.empty(k, dtype=torch.int64, device=self.comm_device or "cpu")

    def place(self, graph, recv, k, pos):
        recv = self._in(recv)
        _lib.check(_lib.lib().tc_dist_place(graph.handle, ctypes.c_void_p(recv.data_ptr() if k else 0),
                                            k, pos))

    def dst_slice(self, graph, lo, hi):
        import torch
        _, dst, _ = graph.device_pointers()
        t = torch.as_tensor(_CudaArray(dst + 4 * lo, hi - lo, "<i4"), device=self.torch_device)
        return self._out(t)

    def dst_write(self, graph, lo, t):
        import torch
        _, dst, _ = graph.device_pointers()
        d = torch.as_tensor(_CudaArray(dst + 4 * lo, t.numel(), "<i4"), device=self.torch_device)
        d.copy_(t)
        torch.cuda.synchronize(self.torch_device)  # the library's stream reads it next

    def comm_empty(self, k):
        import torch
        return torch.empty(k, dtype=torch.int32, device=self.comm_device or "cpu")

    def free_keys(self, keys):
        keys.free()
