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
from paper_1503_00576_b200.distributed import (Ops, count_distributed, count_distributed_sharded,
                                               shard_bounds)


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

    # ---- v2: numpy restatement of each device step (see include/tricount_b200.h) ----
    @staticmethod
    def _vb(n):
        return max(int(n - 1).bit_length(), 1)

    def shard_degrees(self, shard, n):
        return torch.from_numpy(np.bincount(shard[:, 0], minlength=n).astype(np.int32))

    def shard_orient(self, shard, n, deg):
        deg = deg.numpy().astype(np.int64)
        order = np.lexsort((np.arange(n), deg))
        rank = np.empty(n, np.int64)
        rank[order] = np.arange(n)
        ru, rv = rank[shard[:, 0]], rank[shard[:, 1]]
        keep = ru < rv
        keys = np.sort((ru[keep] << self._vb(n)) | rv[keep]).astype(np.int64)
        outdeg = np.bincount(ru[keep], minlength=n).astype(np.int32)
        return keys, int(keys.size), torch.from_numpy(outdeg)

    def create_graph(self, m, n):
        return self.empty_graph(m, n)

    def layout(self, g, outdeg, parts):
        n = g["off"].size - 1
        np.cumsum(outdeg.numpy().astype(np.int64), out=g["off"][1:])
        m = int(g["off"][-1])
        want = (m * np.arange(parts + 1)) // parts
        cuts = np.searchsorted(g["off"][:n], want, side="left").astype(np.int64)
        cuts[parts] = n
        return cuts, g["off"][cuts].copy()

    def split(self, keys, nkeys, n, cuts, parts):
        pos = np.searchsorted(keys, np.asarray(cuts, np.int64) << self._vb(n))
        pos[-1] = nkeys
        return np.diff(pos)

    def send_tensor(self, keys, nkeys):
        return torch.from_numpy(keys)

    def recv_tensor(self, k):
        return torch.empty(k, dtype=torch.int64)

    def place(self, g, recv, k, pos):
        n = g["off"].size - 1
        keys = np.sort(recv.numpy())
        g["dst"][pos:pos + k] = (keys & ((1 << self._vb(n)) - 1)).astype(np.uint32)

    def dst_slice(self, g, lo, hi):
        return torch.from_numpy(g["dst"][lo:hi].view(np.int32))

    def dst_write(self, g, lo, t):
        g["dst"][lo:lo + t.numel()] = t.numpy().view(np.uint32)


def _rank_space_csr(pairs):
    """Single-process restatement of the rank-space CSR the sharded path must rebuild."""
    n = int(pairs.max()) + 1
    deg = np.bincount(pairs[:, 0], minlength=n)
    order = np.lexsort((np.arange(n), deg))
    rank = np.empty(n, np.int64)
    rank[order] = np.arange(n)
    ru, rv = rank[pairs[:, 0]], rank[pairs[:, 1]]
    keep = ru < rv
    o = np.lexsort((rv[keep], ru[keep]))
    dst = rv[keep][o].astype(np.uint32)
    off = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(ru[keep], minlength=n), out=off[1:])
    return dst, off


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


def _worker_sharded(rank, world, port, pairs, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b = shard_bounds(pairs.shape[0], world)
        ops = OracleOps()
        n = int(pairs.max()) + 1
        holder = {}
        orig = ops.finalize

        def fin(g):
            orig(g)
            holder["g"] = g
        ops.finalize = fin
        rep = count_distributed_sharded(ops, pairs[b[rank]:b[rank + 1]], n)
        g = holder["g"]
        q.put((rank, rep.triangles, rep.local, rep.bounds, rep.m, None, g["dst"].copy(), g["off"].copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shuffle", [(2, False), (3, True), (4, False)])
def test_count_distributed_sharded_gloo(golden, world, shuffle):
    """v2: sharded degrees -> ranks -> local orient/sort -> all-to-all by source range ->
    placed slices -> all-gather; every rank ends with the same rank-space CSR as a
    single-process build and the golden triangle count."""
    rec = golden["graphs"]["rmat_12_16_99"]
    pairs = oracle.symmetrize(oracle.rmat_pairs(12, 16, seed=99))
    if shuffle:
        pairs = pairs[np.random.default_rng(7).permutation(pairs.shape[0])]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_sharded, args=(r, world, port, pairs, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=180) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert {r[1] for r in res} == {rec["triangles"]}
    assert sum(r[2] for r in res) == rec["triangles"]
    dst, off = _rank_space_csr(pairs)
    for r in res:
        assert r[4] == rec["m"]
        assert np.array_equal(r[6], dst) and np.array_equal(r[7], off)


def test_refine_plan_equalises_measured_times():
    """refine_plan re-cuts both sides at equal cumulative measured time (uniform within a
    shard); a plan whose shards already take equal time is a fixed point; heads below the
    floor carry no work."""
    from paper_1503_00576_b200.distributed import refine_plan
    eb, hb = [0, 100, 200, 300, 400], [0, 1000, 1010, 1020, 1030]
    e2, h2 = refine_plan(eb, hb, [1, 1, 1, 1], [2, 2, 2, 2], head_floor=990)
    assert list(e2) == eb
    assert h2[0] == 0 and h2[-1] == 1030 and list(h2[2:]) == [1010, 1020, 1030]
    e3, _ = refine_plan(eb, hb, [3, 1, 1, 3], [1, 1, 1, 1], head_floor=990)
    assert e3[0] == 0 and e3[-1] == 400 and list(e3) == sorted(e3)
    # equal time per shard under the uniform-density assumption
    dens = [3 / 100, 1 / 100, 1 / 100, 3 / 100]

    def t(a, b):
        tot, x = 0.0, a
        while x < b:
            k = min(x // 100, 3)
            nxt = min(b, (k + 1) * 100)
            tot += (nxt - x) * dens[k]
            x = nxt
        return tot
    parts = [t(e3[i], e3[i + 1]) for i in range(4)]
    assert max(parts) - min(parts) < 0.05


def test_shard_planner_refinement_converges():
    """ShardPlanner (pure host logic): with a hidden true cost per tile/head that differs
    from the model by a smooth factor, two refinements bring every shard within 2 % of the
    mean."""
    from paper_1503_00576_b200.distributed import ShardPlanner
    rng = np.random.default_rng(3)
    ecost = rng.random(4096) + 0.1
    hcost = rng.random(2048) ** 3
    etrue = ecost * np.linspace(0.5, 3.0, ecost.size)
    htrue = hcost * np.linspace(2.0, 0.4, hcost.size)
    P = 8
    pl = ShardPlanner(ecost, 16, hcost, 1000, 16 * 4096, 1000 + 2048, P, head_fixed_ms=0.0, edge_fixed_ms=0.0)

    def measure():
        e = [etrue[pl.ecut[r]:pl.ecut[r + 1]].sum() for r in range(P)]
        h = [htrue[pl.hcut[r]:pl.hcut[r + 1]].sum() for r in range(P)]
        return np.array(e), np.array(h)
    e0, h0 = measure()
    for _ in range(2):
        pl.refine(*measure())
    e2, h2 = measure()
    assert e2.max() / e2.mean() < 1.02 and h2.max() / h2.mean() < 1.02
    assert e0.max() / e0.mean() > 1.1
    eb, hb = pl.bounds()
    assert eb[0] == 0 and eb[-1] == 16 * 4096 and hb[0] == 0 and hb[-1] == 3048
    assert all(np.diff(eb) >= 0) and all(np.diff(hb) >= 0)
