"""Does a kernel that waits on the event of upload part c start before the
whole upload has drained? (torch streams; not part of the product)"""
import time
import torch
n = 1 << 29  # 4 GB of float64
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
parts = 16
up = torch.cuda.Stream()
ks = torch.cuda.Stream()
for inflight_all in (True, False):
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(parts)]
    kev = [torch.cuda.Event(enable_timing=True) for _ in range(parts)]
    start = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record(up)
    sz = n // parts
    for c in range(parts):
        with torch.cuda.stream(up):
            d[c * sz:(c + 1) * sz].copy_(h[c * sz:(c + 1) * sz], non_blocking=True)
            evs[c].record(up)
        if not inflight_all and c >= 1:
            evs[c - 1].synchronize()
        with torch.cuda.stream(ks):
            ks.wait_event(evs[c])
            d[c * sz:(c + 1) * sz].mul_(1.0)
            kev[c].record(ks)
    torch.cuda.synchronize()
    print("all parts queued" if inflight_all else "two in flight")
    print(" part resident (ms):", [round(start.elapsed_time(e), 1) for e in evs])
    print(" kernel done   (ms):", [round(start.elapsed_time(e), 1) for e in kev])
