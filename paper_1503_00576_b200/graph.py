"""Boundary containers: the reference's EdgeArray / DegreeOrder / OrientedGraph contract.

Mirrors reference graph.py:101-193 (same names, fields, dtypes, read-only arrays and
equality), with one addition: an OrientedGraph produced by the B200 pipeline lives in
HBM and only materialises its numpy arrays when something on the host reads them, so
``count_triangles(preprocess(g))`` never copies the CSR back.
"""
from __future__ import annotations

import ctypes
import math
import weakref

import numpy as np

from . import _lib

MAX_VERTEX_ID = 2**32 - 1


def _readonly(a: np.ndarray) -> np.ndarray:
    a.flags.writeable = False
    return a


def _pair_array(edges) -> np.ndarray:
    """Coerce pairs to a read-only C-contiguous (k, 2) uint32 array (graph.py:67-81)."""
    if isinstance(edges, EdgeArray):
        return edges.edges
    arr = np.asarray(edges)
    if arr.size == 0:
        return _readonly(np.zeros((0, 2), dtype=np.uint32))
    if arr.ndim != 2 or arr.shape[1] != 2:
        raise ValueError(f"expected a sequence of (u, v) pairs, got shape {arr.shape}")
    if arr.dtype.kind not in "iu":
        raise ValueError(f"vertex ids must be integers, got dtype {arr.dtype}")
    if arr.dtype != np.uint32:
        lo, hi = int(arr.min()), int(arr.max())
        if lo < 0 or hi > MAX_VERTEX_ID:
            bad = lo if lo < 0 else hi
            raise ValueError(f"vertex ids must fit in an unsigned 32-bit integer, got {bad}")
    out = np.ascontiguousarray(arr, dtype=np.uint32)
    if out is arr and out.flags.writeable:
        out = out.view()
    return _readonly(out)


class EdgeArray:
    """Undirected graph as directed (u, v) pairs, one per direction (graph.py:101-129).

    ``num_vertices`` is 1 + the largest id (0 when empty).
    """

    __slots__ = ("edges", "num_vertices", "__weakref__")

    def __init__(self, edges, num_vertices: int | None = None):
        self.edges = _pair_array(edges)
        if num_vertices is None:
            num_vertices = int(self.edges.max()) + 1 if self.edges.size else 0
        self.num_vertices = int(num_vertices)

    @property
    def num_undirected_edges(self) -> int:
        return self.edges.shape[0] // 2

    def pairs(self) -> list[tuple[int, int]]:
        return [tuple(p) for p in self.edges.tolist()]

    def __eq__(self, other) -> bool:
        if not isinstance(other, EdgeArray):
            return NotImplemented
        return np.array_equal(self.edges, other.edges)

    def __repr__(self) -> str:
        return f"EdgeArray(num_vertices={self.num_vertices}, directed_entries={self.edges.shape[0]})"


class DegreeOrder:
    """Undirected degree per vertex and the strict order (deg(v), v) (graph.py:132-143)."""

    __slots__ = ("degrees",)

    def __init__(self, degrees):
        self.degrees = _readonly(np.ascontiguousarray(degrees, dtype=np.int64))

    def precedes(self, u: int, v: int) -> bool:
        return (int(self.degrees[u]), u) < (int(self.degrees[v]), v)


class GraphValidationError(ValueError):
    """Base class for edge-array validation failures (reference graph.py:42-43)."""


class SelfLoopError(GraphValidationError):
    def __init__(self, vertex: int):
        self.vertex = vertex
        super().__init__(f"self-loop at vertex {vertex}")


class AsymmetricEdgeError(GraphValidationError):
    def __init__(self, u: int, v: int):
        self.u, self.v = u, v
        super().__init__(f"edge ({u}, {v}) has no reverse ({v}, {u})")


class DuplicateEdgeError(GraphValidationError):
    def __init__(self, u: int, v: int):
        self.u, self.v = u, v
        super().__init__(f"duplicate edge ({u}, {v})")


def validate_edge_array(edges) -> EdgeArray:
    """Check pairs against the edge-array contract on the device (graph.py:196-242).

    Same checks, order and reported pair as the reference: the first self-loop in input
    order, then the earliest second occurrence of a duplicate directed pair, then the
    first pair whose reverse is missing.  Accepts raw pairs, an EdgeArray or a
    device-resident ``DeviceEdges`` (validated in place, nothing copied).
    """
    if hasattr(edges, "ptr"):
        ptr, npairs, n, on_dev, host = ctypes.c_void_p(edges.ptr), edges.npairs, edges.num_vertices, 1, None
    else:
        g = edges if isinstance(edges, EdgeArray) else EdgeArray(edges)
        host = g.edges
        ptr, npairs, n, on_dev = _lib.ptr(host), host.shape[0], g.num_vertices, 0
    if npairs == 0:
        return edges if hasattr(edges, "ptr") else EdgeArray(host)
    code, index = ctypes.c_int(), ctypes.c_uint64()
    _lib.check(_lib.lib().tc_validate_edge_array(ptr, npairs, n, on_dev, ctypes.byref(code),
                                                 ctypes.byref(index)))
    if code.value:
        i = int(index.value)
        if host is not None:
            u, v = (int(x) for x in host[i])
        else:
            pair = np.empty(2, dtype=np.uint32)
            _lib.check(_lib.lib().tc_memcpy(_lib.ptr(pair), ctypes.c_void_p(edges.ptr + 8 * i), 8, 1))
            u, v = int(pair[0]), int(pair[1])
        if code.value == 1:
            raise SelfLoopError(u)
        if code.value == 2:
            raise DuplicateEdgeError(u, v)
        if code.value == 3:
            raise AsymmetricEdgeError(u, v)
        raise ValueError(f"pair {i} ({u}, {v}) has a vertex id >= num_vertices={n}")
    return edges if hasattr(edges, "ptr") else EdgeArray(host, num_vertices=n)


def degrees_of(g: EdgeArray) -> DegreeOrder:
    """First-column histogram = undirected degree for symmetric input (graph.py:279-281)."""
    return DegreeOrder(np.bincount(g.edges[:, 0], minlength=g.num_vertices))


def max_out_degree_bound(m_dir: int) -> int:
    """ceil(sqrt(2 m)): the cap on any oriented adjacency list (graph.py:284-290)."""
    if m_dir <= 0:
        return 0
    r = math.isqrt(2 * m_dir)
    return r if r * r == 2 * m_dir else r + 1


class DeviceGraph:
    """Owning handle of a tc_graph (device-resident oriented CSR)."""

    __slots__ = ("handle", "m", "n", "max_out", "_fin", "__weakref__")

    def __init__(self, handle: int):
        self.handle = ctypes.c_void_p(handle)
        L = _lib.lib()
        m, n, mo = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint32()
        _lib.check(L.tc_graph_info(self.handle, ctypes.byref(m), ctypes.byref(n), ctypes.byref(mo)))
        self.m, self.n, self.max_out = m.value, n.value, mo.value
        self._fin = weakref.finalize(self, L.tc_graph_free, self.handle)

    @classmethod
    def upload(cls, src: np.ndarray, dst: np.ndarray, off: np.ndarray) -> "DeviceGraph":
        L = _lib.lib()
        h = ctypes.c_void_p()
        _lib.check(L.tc_graph_upload(_lib.ptr(src), _lib.ptr(dst), _lib.ptr(off), src.size,
                                     off.size - 1, ctypes.byref(h)))
        return cls(h.value)

    def download(self):
        src = np.empty(self.m, dtype=np.uint32)
        dst = np.empty(self.m, dtype=np.uint32)
        off = np.empty(self.n + 1, dtype=np.int64)
        _lib.check(_lib.lib().tc_graph_download(self.handle, _lib.ptr(src), _lib.ptr(dst),
                                                _lib.ptr(off)))
        return src, dst, off

    def device_pointers(self):
        s, d, o = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _lib.check(_lib.lib().tc_graph_device_ptrs(self.handle, ctypes.byref(s), ctypes.byref(d),
                                                   ctypes.byref(o)))
        return s.value, d.value, o.value

    def free(self) -> None:
        self._fin()


class OrientedGraph:
    """Degree-ordered CSR in unzipped form (graph.py:146-193).

    ``edge_dst[node_offsets[v]:node_offsets[v+1]]`` is v's sorted out-list and
    ``edge_src[i]`` the source of entry i.  Constructed from host arrays (uploaded on
    first count) or from a device graph (downloaded on first host access).
    """

    __slots__ = ("_src", "_dst", "_off", "_dev", "_m", "_n")

    def __init__(self, edge_src, edge_dst, node_offsets):
        self._src = _readonly(np.ascontiguousarray(edge_src, dtype=np.uint32))
        self._dst = _readonly(np.ascontiguousarray(edge_dst, dtype=np.uint32))
        self._off = _readonly(np.ascontiguousarray(node_offsets, dtype=np.int64))
        self._dev = None
        self._m = int(self._dst.shape[0])
        self._n = int(self._off.shape[0]) - 1

    @classmethod
    def _from_device(cls, dev: DeviceGraph) -> "OrientedGraph":
        og = cls.__new__(cls)
        og._src = og._dst = og._off = None
        og._dev = dev
        og._m, og._n = dev.m, dev.n
        return og

    def _materialise(self) -> None:
        if self._dst is None:
            s, d, o = self._dev.download()
            self._src, self._dst, self._off = _readonly(s), _readonly(d), _readonly(o)

    def device(self) -> DeviceGraph:
        """The device copy (uploaded on first use)."""
        if self._dev is None:
            if self._src.shape[0] != self._m:
                raise ValueError("edge_src and edge_dst lengths differ")
            self._dev = DeviceGraph.upload(self._src, self._dst, self._off)
        return self._dev

    @property
    def edge_src(self) -> np.ndarray:
        self._materialise()
        return self._src

    @property
    def edge_dst(self) -> np.ndarray:
        self._materialise()
        return self._dst

    @property
    def node_offsets(self) -> np.ndarray:
        self._materialise()
        return self._off

    @property
    def num_vertices(self) -> int:
        return self._n

    @property
    def m_dir(self) -> int:
        return self._m

    @property
    def out_degrees(self) -> np.ndarray:
        return np.diff(self.node_offsets)

    def adjacency(self, v: int) -> np.ndarray:
        off = self.node_offsets
        return self.edge_dst[off[v]:off[v + 1]]

    def undirected_degrees(self) -> np.ndarray:
        return self.out_degrees + np.bincount(self.edge_dst, minlength=self.num_vertices)

    def __eq__(self, other) -> bool:
        if not isinstance(other, OrientedGraph):
            return NotImplemented
        return (np.array_equal(self.edge_src, other.edge_src)
                and np.array_equal(self.edge_dst, other.edge_dst)
                and np.array_equal(self.node_offsets, other.node_offsets))

    __hash__ = None

    def __repr__(self) -> str:
        return f"OrientedGraph(num_vertices={self.num_vertices}, m_dir={self.m_dir})"


def validate_oriented_graph(og: OrientedGraph) -> OrientedGraph:
    """Check every OrientedGraph invariant (graph.py:293-332); raises ValueError."""
    off, src, dst = og.node_offsets, og.edge_src, og.edge_dst
    m = og.m_dir
    if off.shape[0] < 1 or off[0] != 0:
        raise ValueError("node_offsets must start at 0")
    if off[-1] != m:
        raise ValueError(f"node_offsets must end at m_dir={m}, got {int(off[-1])}")
    outdeg = np.diff(off)
    if (outdeg < 0).any():
        raise ValueError("node_offsets must be nondecreasing")
    if src.shape[0] != m:
        raise ValueError("edge_src and edge_dst lengths differ")
    if not np.array_equal(src, np.repeat(np.arange(og.num_vertices, dtype=np.uint32), outdeg)):
        raise ValueError("edge_src does not match the grouping implied by node_offsets")
    if m > 1:
        new_list = np.zeros(m, dtype=bool)
        new_list[off[:-1][off[:-1] < m]] = True
        rising = (dst[1:] > dst[:-1]) | new_list[1:]
        if not rising.all():
            raise ValueError(
                f"adjacency list not strictly ascending at edge index {int(np.argmin(rising)) + 1}")
    deg = og.undirected_degrees()
    du, dv = deg[src], deg[dst]
    fwd = (du < dv) | ((du == dv) & (src < dst))
    if not fwd.all():
        i = int(np.argmin(fwd))
        raise ValueError(f"edge ({int(src[i])}, {int(dst[i])}) is not degree-ordered forward")
    top = int(outdeg.max()) if og.num_vertices else 0
    if top > max_out_degree_bound(m):
        raise ValueError(f"max out-degree {top} exceeds bound {max_out_degree_bound(m)}")
    return og
