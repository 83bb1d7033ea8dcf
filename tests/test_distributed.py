"""Multi-process (gloo, world_size 2) test of the distributed driver's host logic:
rank 0 preprocesses, the oriented CSR is broadcast, every rank rebuilds edge_src,
counts its work-balanced shard, and one 64-bit all-reduce combines the counts.
The device operations are replaced by the CPU oracle (paper_1503_00576_b200.distributed.Ops)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1503_00576_b200.distributed import Ops, count_distributed


class OracleOps(Ops):
    """CPU stand-in for B200Ops (test infrastructure only)."""

    def preprocess(self, edges):
        src, dst, off = oracle.preprocess(edges)
        return {"src": src, "dst": dst, "off": off}

    def graph_shape(self, g):
        return int(g["dst"].size), int(g["off"].size) - 1

    def empty_graph(self, m, n):
        return {"src": np.zeros(m, np.uint32), "dst": np.zeros(m, np.uint32),
                "off": np.zeros(n + 1, np.int64)}

    def replica_tensors(self, g):
        return [torch.from_numpy(g["dst"].view(np.uint8)), torch.from_numpy(g["off"].view(np.uint8))]

    def finalize(self, g):
        deg = np.diff(g["off"])
        g["src"] = np.repeat(np.arange(deg.size, dtype=np.uint32), deg)

    def work_bounds(self, g, parts):
        deg = np.diff(g["off"])
        w = deg[g["src"]] + deg[g["dst"]] + 8
        c = np.concatenate([[0], np.cumsum(w)])
        targets = c[-1] * np.arange(parts + 1) / parts
        b = np.searchsorted(c, targets).astype(np.int64)
        b[0], b[-1] = 0, g["dst"].size
        return np.maximum.accumulate(b)

    def count_range(self, g, lo, hi):
        L = oracle.lib()
        return int(L.or_count_strided(oracle._c32(g["src"]), oracle._c32(g["dst"]),
                                      oracle._c64(g["off"]), lo, hi, 0, 1))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, pairs, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rep = count_distributed(OracleOps(), pairs if rank == 0 else None)
        q.put((rank, rep.triangles, rep.local, rep.bounds, rep.m))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_count_distributed_gloo(golden, world):
    rec = golden["graphs"]["rmat_12_16_99"]
    pairs = oracle.symmetrize(oracle.rmat_pairs(12, 16, seed=99))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, pairs, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    totals = {r[1] for r in res}
    assert totals == {rec["triangles"]}
    assert sum(r[2] for r in res) == rec["triangles"]
    bounds = res[0][3]
    assert bounds[0] == 0 and bounds[-1] == rec["m"] and list(bounds) == sorted(bounds)
    assert all(r[3] == bounds for r in res)
