"""Development aid (GPU box): host->device copy rate from pinned memory, one vs several
copy streams (chunked), to see whether the e2e path's single copy stream leaves PCIe idle."""
import torch

GB = 4
n = GB << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
chunk = 256 << 20
streams = [torch.cuda.Stream() for _ in range(4)]


def run(nstreams, ch):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    evs = []
    for k, off in enumerate(range(0, n, ch)):
        s = streams[k % nstreams]
        s.wait_event(e0) if k < nstreams else None
        with torch.cuda.stream(s):
            d[off:off + ch].copy_(h[off:off + ch], non_blocking=True)
    for s in streams[:nstreams]:
        ev = torch.cuda.Event()
        ev.record(s)
        torch.cuda.current_stream().wait_event(ev)
    e1.record()
    torch.cuda.synchronize()
    return n / (e0.elapsed_time(e1) / 1e3) / 1e9


for rep in range(2):
    for ns, ch in ((1, n), (1, chunk), (2, chunk), (4, chunk), (2, 64 << 20), (4, 64 << 20)):
        print(f"streams={ns} chunk={ch >> 20}MB  {run(ns, ch):.1f} GB/s", flush=True)
