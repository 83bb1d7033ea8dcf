"""The v2 sharded path (count_distributed_sharded) through libtcb200 on ONE GPU: two or
three processes share cuda:0 under gloo, staging every collective through host memory
(B200Ops(comm="cpu")).  Device steps are the ones NCCL ranks run; only the transport
differs.  Checks the golden count and that every rank rebuilt the same rank-space CSR as
the single-GPU rank-space preprocess."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, scale, seed, on_device, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), TC_DEVICE="0")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1503_00576_b200 as tcb
        from paper_1503_00576_b200 import generators
        from paper_1503_00576_b200.distributed import (B200Ops, count_distributed_sharded,
                                                       shard_bounds)
        ops = B200Ops(0, comm="cpu")
        dev = generators.rmat_device(scale, 16, seed=seed)
        b = shard_bounds(dev.npairs, world)
        if on_device:
            shard = generators.DeviceEdgesView(dev, b[rank], b[rank + 1])
        else:
            shard = dev.to_host().edges[b[rank]:b[rank + 1]]
        holder = {}
        orig = ops.finalize

        def fin(g):
            orig(g)
            holder["g"] = g
        ops.finalize = fin
        rep = count_distributed_sharded(ops, shard, dev.num_vertices)
        g = holder["g"]
        og = tcb.OrientedGraph._from_device(g)
        ref, _ = tcb.preprocess_device(dev, rank_space=True)
        same = (np.array_equal(og.edge_dst, ref.edge_dst) and np.array_equal(og.node_offsets, ref.node_offsets)
                and np.array_equal(og.edge_src, ref.edge_src))
        q.put((rank, rep.triangles, rep.local, rep.m, same))
    except Exception as e:  # noqa: BLE001 - surfaced through the queue
        q.put((rank, repr(e), None, None, False))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,on_device", [(2, True), (3, False)])
def test_sharded_preprocess_one_gpu(golden, world, on_device):
    rec = golden["graphs"]["rmat_12_16_99"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 12, 99, on_device, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs), res
    assert {r[1] for r in res} == {rec["triangles"]}, res
    assert sum(r[2] for r in res) == rec["triangles"]
    assert all(r[3] == rec["m"] and r[4] for r in res), res


def test_sharded_preprocess_one_gpu_big():
    """R-MAT s20 over 2 sharing processes == the single-GPU golden count."""
    import json
    from conftest import GOLDEN_DIR
    with open(os.path.join(GOLDEN_DIR, "golden_big.json")) as fh:
        want = json.load(fh)["rmat_20_16_0"]["triangles"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 20, 0, True, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=600) for _ in range(2)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
    assert {r[1] for r in res} == {want}, res
    assert all(r[4] for r in res)


def _nccl_worker(port, q):
    """One rank over NCCL (world 1: NCCL refuses two ranks on one GPU): the v2 collectives
    (all-reduce of degrees / out-degrees / m, the key all-to-all, the edge_dst all-gather,
    the count all-reduce) run on device tensors that alias library-owned HBM."""
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), TC_DEVICE="0")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        import paper_1503_00576_b200 as tcb
        from paper_1503_00576_b200 import generators
        from paper_1503_00576_b200.distributed import (B200Ops, count_distributed,
                                                       count_distributed_sharded)
        ops = B200Ops(0, comm="cuda")
        dev = generators.rmat_device(16, 16, seed=0)
        a = count_distributed_sharded(ops, dev, dev.num_vertices).triangles
        b = count_distributed_sharded(ops, dev.to_host().edges, dev.num_vertices).triangles
        c = count_distributed(ops, dev).triangles
        plans = {}
        d = [count_distributed_sharded(ops, dev, dev.num_vertices, plans=plans).triangles for _ in range(2)]
        ref = tcb.count_with_timings_device(dev)[0]
        assert d == [ref, ref], d
        q.put((a, b, c, ref, dist.get_backend()))
    except Exception as e:  # noqa: BLE001
        q.put((repr(e), None, None, None, None))
        raise
    finally:
        dist.destroy_process_group()


def test_nccl_transport_world1():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    p.start()
    res = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0, res
    a, b, c, ref, backend = res
    assert backend == "nccl"
    assert a == b == c == ref, res
