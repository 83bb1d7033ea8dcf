#!/usr/bin/env python
"""Bench: exact triangle count of Graph500-style R-MAT scale 26, edge factor 16, seed 0
(BASELINE.json metric "edges/sec & count time at 1/2/4/8 B200 (R-MAT s26); HBM GB/s vs
peak").  One step = one pass of the hot path (reference count_with_timings,
count.py:207-229): preprocess the edge array into the oriented CSR, then count.

  value : edges/s with the edge array already resident in HBM (device-timed, CUDA events)
  e2e   : edges/s through count_with_timings() from a pinned HOST edge array (H2D of the
          17.2 GB pair array + 8-byte result D2H inside every step)
Input: the reference generator rmat(26, 16, seed=0), reproduced bit-for-bit on the device
(generators.rmat_device), untimed.  Inputs (17.2 GB) exceed L2 (126 MB) -- no flush needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--scale S]
Multi-GPU: torchrun, one process per GPU; rank 0 preprocesses, the CSR is broadcast
over NCCL, shards are work balanced, one 64-bit all-reduce; timing = max over ranks.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "edges/sec & count time at 1/2/4/8 B200 (R-MAT s26); HBM GB/s vs peak"
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--edge-factor", type=int, default=16)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--dist", choices=["v1", "v2"], default="v2",
                    help="multi-GPU path: v1 rank-0 preprocess + broadcast, v2 sharded preprocess")
    ap.add_argument("--share-gpu", action="store_true",
                    help="testing only: all ranks on cuda:0, gloo, collectives staged through host")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU work per baseline sample step")
    return ap.parse_args()


# ----------------------------------------------------------------------- clocks ---
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.device)],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        except OSError:
            pass
        finally:
            if self.path and os.path.exists(self.path):
                os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def dominant_kernel_from_profiles(peak: float):
    """The count's largest kernel in the committed ncu capture (time and DRAM bytes per launch,
    cold-cache / serialised under ncu) -- the kernel-level roofline beside the phase-level one."""
    import csv
    path = os.path.join(ROOT, "profiles", "r01_dram_count_s26_vmajor.csv")
    try:
        rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    except OSError:
        return None
    h = rows[0]
    ki, mi, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = {}
    for r in rows[1:]:
        per.setdefault((int(r[ii]), r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
    (_, name), d = max(per.items(), key=lambda kv: kv[1].get("gpu__time_duration.sum", 0))
    ms = d["gpu__time_duration.sum"] / 1e6
    b = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    return {"name": name.split("(")[0].replace("void ", ""), "ncu_ms": round(ms, 3),
            "dram_bytes": b, "dram_gbs": round(b / ms / 1e6, 1), "dram_frac": round(b / ms / 1e6 / peak, 4),
            "source": "profiles/r01_dram_count_s26_vmajor.csv (ncu, one count call)"}


def traffic_from_profiles(workload: str):
    """dram read+write bytes per count call from the committed ncu capture, if any."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            rec = json.load(fh).get(workload)
        return None if rec is None else rec.get("dram_bytes_per_count")
    except (OSError, ValueError):
        return None


# ------------------------------------------------------------------ CPU baseline ---
def cpu_sample(pairs_host, og_host, m, W, target_s):
    """The reference CPU path (oracle port, all host threads) on a bounded sample of this
    workload: preprocessing of a 1/S_pre slice of the pair array and counting of a strided
    1/S_cnt sample of the oriented edges (the reference's own strided assignment,
    count.py:69), each extrapolated linearly to the full graph."""
    import oracle

    import numpy as np

    cores = os.cpu_count() or 1
    npairs = pairs_host.shape[0]
    n = int(og_host[2].shape[0]) - 1
    s_pre = max(1, npairs // (1 << 24))
    part = np.ascontiguousarray(pairs_host[::s_pre])  # strided: ids span the full range
    t0 = time.perf_counter()
    oracle.preprocess(np.zeros((0, 2), np.uint32), num_vertices=n, threads=cores)
    t_n = time.perf_counter() - t0  # O(n) node-array work, paid once at full size
    t0 = time.perf_counter()
    oracle.preprocess(part, num_vertices=n, threads=cores)
    t_part = time.perf_counter() - t0
    t_pre = max(t_part - t_n, 0.0) * s_pre + t_n
    # ~5 ns per merge step per core; aim for ~target_s of wall time
    s_cnt = max(1, int(W * 5e-9 / (cores * max(target_s - 2.0, 1.0))))
    src, dst, off = og_host
    t0 = time.perf_counter()
    oracle.count_sampled(src, dst, off, s_cnt, threads=cores)
    t_cnt = (time.perf_counter() - t0) * s_cnt
    value = m / (t_pre + t_cnt)
    return {"value": value, "unit": "edges/s", "cores": cores, "kind": "port",
            "sample": (f"oracle C port: preprocess of every {s_pre}-th pair (pair-proportional time x{s_pre}, "
                       f"O(n) node-array time once) and count of every "
                       f"{s_cnt}-th oriented edge, both extrapolated linearly; "
                       f"est preprocess {t_pre:.1f}s + count {t_cnt:.1f}s"),
            "preprocess_s_est": t_pre, "count_s_est": t_cnt}


# ------------------------------------------------------------------------ main ---
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.share_gpu:
        local = 0
    os.environ.setdefault("TC_DEVICE", str(local))
    workload = f"rmat_s{args.scale}_ef{args.edge_factor}_seed{args.seed}"

    if args.impl == "reference":
        return reference_arm(args, world, rank, workload)

    import torch

    import paper_1503_00576_b200 as tcb
    from paper_1503_00576_b200 import _lib, generators
    from paper_1503_00576_b200.distributed import (B200Ops, count_distributed,
                                                   count_distributed_sharded, shard_bounds)

    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if args.share_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L = _lib.lib()

    def timer(a):
        _lib.check(L.tc_timer_record(a))

    def elapsed(a, b):
        import ctypes
        ms = ctypes.c_double()
        _lib.check(L.tc_timer_elapsed(a, b, ctypes.byref(ms)))
        return ms.value

    def launches():
        import ctypes
        c = ctypes.c_uint64()
        L.tc_launch_count(ctypes.byref(c))
        return c.value

    def barrier():
        _lib.check(L.tc_synchronize())
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if args.share_gpu else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    t0 = time.time()
    dev_edges = generators.rmat_device(args.scale, args.edge_factor, seed=args.seed)
    gen_s = time.time() - t0
    npairs = dev_edges.npairs
    m = npairs // 2
    og, _ = tcb.preprocess_device(dev_edges)
    W = tcb.merge_work(og)
    assert og.m_dir == m
    host_graph = None
    ops = B200Ops(local, comm="cpu" if args.share_gpu else "cuda") if world > 1 else None
    sb = shard_bounds(npairs, world)
    shard = generators.DeviceEdgesView(dev_edges, sb[rank], sb[rank + 1])

    def step_device():
        if world == 1:
            tri, t = tcb.count_with_timings_device(dev_edges)
            return tri, t.preprocess_ms, t.count_ms
        if args.dist == "v1":
            rep = count_distributed(ops, dev_edges if rank == 0 else None)
        else:
            rep = count_distributed_sharded(ops, shard, dev_edges.num_vertices)
        return rep.triangles, None, None

    for _ in range(args.warmup):
        tri_ref, _, _ = step_device()
    # ----------------------------------------------------------- timed: value ---
    pre, cnt, tris = [], [], set()
    with ClockSampler(local) as clk:
        barrier()
        l0 = launches()
        timer(0)
        for _ in range(args.steps):
            tri, p, c = step_device()
            tris.add(tri)
            if p is not None:
                pre.append(p)
                cnt.append(c)
        timer(1)
        barrier()
        l1 = launches()
        ms_total = max_over_ranks(elapsed(0, 1))
    clocks = clk.summary()
    if tris != {tri_ref}:
        raise RuntimeError(f"count changed between runs: {tris} vs {tri_ref}")
    ms_per_step = ms_total / args.steps
    value = m * args.steps / (ms_total / 1e3)

    # count-kernel roofline from a standalone count of the resident CSR (events on the
    # library stream around the count kernels of one call)
    count_runs = []
    for _ in range(max(3, min(args.steps, 5))):
        _, tc = tcb.count_device(og)
        count_runs.append(tc)
    count_ms = statistics.median(t.count_ms for t in count_runs)
    heavy_ms = statistics.median(t.heavy_ms for t in count_runs)
    window_ms = statistics.median(t.light_ms for t in count_runs)
    vmajor_ms = statistics.median(t.vmajor_ms for t in count_runs)
    alg_bytes = 4 * W + 40 * m
    peak, peak_src = measured_peak()
    achieved = alg_bytes / (count_ms / 1e3) / 1e9
    traffic = traffic_from_profiles(workload)
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "traffic_gbs": round(traffic / (count_ms / 1e3) / 1e9, 1) if traffic else None,
                "traffic_frac": round(traffic / (count_ms / 1e3) / 1e9 / peak, 4) if traffic else None,
                "kernel": "count phase (k_classify + k_vin_* hub-head index + k_count_vmajor + "
                          "k_count_hub + k_count_light_tpe)",
                "algorithmic_bytes_per_launch": alg_bytes, "launch_ms": round(count_ms, 3),
                "peak_source": peak_src,
                "dominant_kernel": dominant_kernel_from_profiles(peak) if workload == "rmat_s26_ef16_seed0" else None}

    # ------------------------------------------------------------ timed: e2e ---
    e2e = None
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else min(args.steps, 5)
    if world == 1 and e2e_steps > 0:
        host_graph = dev_edges.to_host(pinned=True)
        tcb.count_with_timings(host_graph)  # warm
        barrier()
        timer(2)
        phase = []
        for _ in range(e2e_steps):
            tri, pt = tcb.count_with_timings(host_graph)
            if tri != tri_ref:
                raise RuntimeError("e2e count differs")
            phase.append(pt)
        timer(3)
        barrier()
        e2e_ms = elapsed(2, 3)
        e2e = {"value": m * e2e_steps / (e2e_ms / 1e3), "unit": "edges/s",
               "h2d_bytes_per_step": npairs * 8, "d2h_bytes_per_step": 8,
               "ms_per_step": e2e_ms / e2e_steps,
               "preprocess_ms_incl_h2d": statistics.mean(p.preprocess_ms for p in phase),
               "count_ms": statistics.mean(p.count_ms for p in phase)}
    elif world > 1 and e2e_steps > 0:
        # every rank copies only its own shard of the pinned host edge array (sharded H2D)
        host_shard = generators.pinned_empty((shard.npairs, 2), np.uint32)
        if shard.npairs:
            _lib.check(L.tc_memcpy(_lib.ptr(host_shard), ctypes.c_void_p(shard.ptr), shard.nbytes, 1))
        count_distributed_sharded(ops, host_shard, dev_edges.num_vertices)  # warm
        barrier()
        timer(2)
        for _ in range(e2e_steps):
            rep = count_distributed_sharded(ops, host_shard, dev_edges.num_vertices)
            if rep.triangles != tri_ref:
                raise RuntimeError("e2e count differs")
        timer(3)
        barrier()
        e2e_ms = max_over_ranks(elapsed(2, 3))
        e2e = {"value": m * e2e_steps / (e2e_ms / 1e3), "unit": "edges/s",
               "h2d_bytes_per_step": npairs * 8, "d2h_bytes_per_step": 8 * world,
               "ms_per_step": e2e_ms / e2e_steps,
               "path": "sharded H2D (each rank its 1/N of the pinned pairs) + v2 distributed preprocessing"}

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        if host_graph is None:
            host_graph = dev_edges.to_host(pinned=True)
        og_host = (og.edge_src, og.edge_dst, og.node_offsets)
        cpu = cpu_sample(host_graph.edges, og_host, m, W, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u32/u64 (integer)", "data": "synthetic (reference rmat generator, device-reproduced)",
            "config": {"workload": workload, "scale": args.scale, "edge_factor": args.edge_factor,
                       "seed": args.seed, "num_vertices": dev_edges.num_vertices,
                       "undirected_edges": m, "pairs": npairs, "triangles": tri_ref,
                       "merge_work_W": W, "inputs_vs_L2": "inputs 8*pairs bytes >> 126 MB L2; no flush",
                       "parallelism": f"{world} GPU(s)" + ("" if world == 1 else
                                      (": rank-0 preprocess, NCCL CSR broadcast, work-balanced shards, 1 all-reduce"
                                       if args.dist == "v1" else
                                       ": sharded degrees/orient/sort, NCCL all-to-all by source range, "
                                       "slice all-gather, work-balanced shards, 1 all-reduce"))},
            "phases_ms": {"preprocess": statistics.mean(pre) if pre else None,
                          "count": statistics.mean(cnt) if cnt else None,
                          "count_umajor_heavy": heavy_ms, "count_light": window_ms,
                          "count_vmajor": vmajor_ms,
                          "generate_input_s": gen_s},
            "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks,
            "gpu_launches": l1 - l0,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def reference_arm(args, world, rank, workload):
    """The reference's CPU implementation (oracle C port, all host threads) on a bounded
    sample of the same workload; rank 0 only."""
    if rank != 0:
        return
    import paper_1503_00576_b200 as tcb
    from paper_1503_00576_b200 import generators

    dev_edges = generators.rmat_device(args.scale, args.edge_factor, seed=args.seed)
    og, _ = tcb.preprocess_device(dev_edges)
    W = tcb.merge_work(og)
    m = og.m_dir
    host = dev_edges.to_host(pinned=True)
    og_host = (og.edge_src, og.edge_dst, og.node_offsets)
    dev_edges.free()
    for _ in range(args.warmup):
        cpu_sample(host.edges, og_host, m, W, args.cpu_seconds / 3)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vals.append(cpu_sample(host.edges, og_host, m, W, args.cpu_seconds / 3))
    wall = time.perf_counter() - t0
    value = statistics.mean(v["value"] for v in vals)
    cpu = dict(vals[-1])
    cpu["value"] = value
    line = {"metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": m / value * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u32/u64 (integer)", "data": "synthetic (reference rmat generator)",
            "config": {"workload": workload, "scale": args.scale, "edge_factor": args.edge_factor,
                       "seed": args.seed, "undirected_edges": m, "merge_work_W": W},
            "impl": "reference", "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "wall_s": wall}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
