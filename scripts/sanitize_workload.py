"""Workload for compute-sanitizer runs (memcheck / racecheck / initcheck / synccheck):
every count path on small graphs -- ER G(10^4, p), R-MAT(12, 16, 99), BA(10^3, 3), K_600,
R-MAT s14 with the v-major schedule forced (index, vlow warp tasks, v-major CTA kernel),
a hand-built DAG on the original-id kernels -- each checked against the oracle.

    compute-sanitizer --tool memcheck python scripts/sanitize_workload.py
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import oracle  # noqa: E402
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import _lib, generators  # noqa: E402
from paper_1503_00576_b200.graph import EdgeArray, OrientedGraph  # noqa: E402


def check(name, pairs):
    want = oracle.count(*oracle.preprocess(pairs))
    g = EdgeArray(pairs)
    got = [tcb.count_with_timings(g)[0]]
    og = tcb.preprocess(g)
    got.append(tcb.count_triangles(og))
    got.append(tcb.count_device(og, algo=_lib.ALGO_MERGE_THREAD)[0])
    got.append(tcb.count_partitioned(og, tcb.PartitionPlan.even(3, og.m_dir), 1))
    assert got == [want] * 4, (name, got, want)
    print(name, want, flush=True)


def main():
    check("er_1e4", oracle.gnp_pairs(10_000, 100_000 / (10_000 * 9_999 / 2), 0))
    check("rmat_12_16_99", oracle.rmat_edges(12, 16, seed=99))
    check("ba_1e3_3", oracle.ba_pairs(1000, 3, seed=5))
    iu = np.triu_indices(600, k=1)
    k600 = np.stack([iu[0], iu[1]], 1).astype(np.uint32)
    check("k600", oracle.symmetrize(k600))
    with _lib.options(vmajor=1, vzone_log2=19):
        check("rmat_14_forced_vmajor", oracle.rmat_edges(14, 16, seed=0))
    # the index built at count time (k_vin_pass, overlapped)
    with _lib.options(vmajor=1, vzone_log2=19, vix=0):
        check("rmat_14_forced_vmajor_vix0", oracle.rmat_edges(14, 16, seed=0))
    src = np.array([0, 0, 0, 0, 0, 1, 1], np.uint32)
    dst = np.array([1, 2, 3, 4, 5, 2, 6], np.uint32)
    off = np.array([0, 5, 7, 7, 7, 7, 7, 7], np.int64)
    assert tcb.count_triangles(OrientedGraph(src, dst, off)) == 1
    d = generators.rmat_device(12, 16, seed=99)
    assert tcb.count_with_timings_device(d)[0] == oracle.count(*oracle.preprocess(oracle.rmat_edges(12, 16, seed=99)))
    print("sanitize workload ok", flush=True)


if __name__ == "__main__":
    main()
