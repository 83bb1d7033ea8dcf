"""Development aid: where the two-call path count_triangles(preprocess(g)) spends its time
at R-MAT scale S (host pinned input): preprocess (H2D + reference-id CSR), then the first
full count of that graph (rank-space relabel + count), then a second count (cached copy)."""
import ctypes
import sys
import time

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import _lib, generators  # noqa: E402
from paper_1503_00576_b200.preprocess import preprocess_with_timings  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 26
d = generators.rmat_device(S, 16, seed=0)
g = d.to_host(pinned=True)
if "--bench-like" in sys.argv:  # the bench's order: device-resident fused steps, fused pinned e2e
    for _ in range(8):
        tcb.count_with_timings_device(d)
    for _ in range(6):
        t0 = time.perf_counter()
        tcb.count_with_timings(g)
        print(f"fused pinned wall {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
else:
    d.free()
reps = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 3


def mem_used_gb():
    f, t = ctypes.c_size_t(), ctypes.c_size_t()
    ctypes.CDLL("libcudart.so").cudaMemGetInfo(ctypes.byref(f), ctypes.byref(t))
    return round((t.value - f.value) / 2**30, 1)


for rep in range(reps):
    _lib.check(_lib.lib().tc_synchronize())
    t0 = time.perf_counter()
    og, tp = preprocess_with_timings(g)
    t1 = time.perf_counter()
    tri, tc = tcb.count_device(og)
    t2 = time.perf_counter()
    tri2, tc2 = tcb.count_device(og)
    t3 = time.perf_counter()
    print(f"rep {rep}: preprocess wall {1e3 * (t1 - t0):.1f} ms (h2d {tp.h2d_ms:.1f}, kernels {tp.preprocess_ms:.1f}); "
          f"first count wall {1e3 * (t2 - t1):.1f} ms (events {tc.count_ms:.1f}); "
          f"second count wall {1e3 * (t3 - t2):.1f} ms (events {tc2.count_ms:.1f}); tri {tri} {tri2}", flush=True)
    del og
    print(f"  device memory used {mem_used_gb()} GB", flush=True)
