"""Development aid: phases of count_with_timings from a pinned host edge array."""
import ctypes
import sys
import time

sys.path.insert(0, ".")
import paper_1503_00576_b200 as tcb  # noqa: E402
from paper_1503_00576_b200 import _lib, generators  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
g = generators.rmat_device(scale, 16, seed=0)
t0 = time.time()
h = g.to_host(pinned=True)
print("to_host s", round(time.time() - t0, 2), flush=True)
if len(sys.argv) > 2:
    g.free()
for i in range(4):
    out = ctypes.c_uint64()
    t = _lib.TcTimes()
    t0 = time.time()
    _lib.check(_lib.lib().tc_count_with_timings(_lib.ptr(h.edges), h.edges.shape[0], h.num_vertices,
                                                0, 0, ctypes.byref(out), ctypes.byref(t)))
    print(i, {k: round(v, 1) for k, v in t.as_dict().items() if k.endswith("ms") and v},
          "wall", round((time.time() - t0) * 1e3, 1), flush=True)
