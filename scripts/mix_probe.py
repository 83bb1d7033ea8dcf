"""Development aid (GPU box): alternate the fused count_with_timings(host pairs) and the
two-call count_triangles(preprocess(g)) at R-MAT scale S and time each call, printing the
device's free memory -- the cross-pool interaction of the scratch and default pools."""
import sys
import time

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import _lib, generators  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 26
order = sys.argv[2] if len(sys.argv) > 2 else "ffttt"
d = generators.rmat_device(S, 16, seed=0)
g = d.to_host(pinned=True)
keep = d if "k" in sys.argv[3:] else None
if keep is None:
    d.free()


def free_gb():
    import ctypes
    cr = ctypes.CDLL("libcudart.so") if False else None  # noqa: F841
    import subprocess
    out = subprocess.run(["nvidia-smi", "--query-gpu=memory.used", "--format=csv,noheader,nounits"],
                         capture_output=True, text=True).stdout.strip()
    return out


for c in order:
    _lib.check(_lib.lib().tc_synchronize())
    t0 = time.perf_counter()
    if c == "f":
        tri = tcb.count_with_timings(g)[0]
    else:
        tri = tcb.count_triangles(tcb.preprocess(g))
    _lib.check(_lib.lib().tc_synchronize())
    print(c, f"{1e3 * (time.perf_counter() - t0):.1f} ms", tri, "used MiB", free_gb(), flush=True)
