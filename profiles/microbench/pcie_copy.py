"""Pinned host <-> device copy time at the decode step's transfer sizes."""
import json, torch
res = {}
for nbytes in (4096, 131072, 262144, 393216, 64 << 20):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        for _ in range(10): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(100): fn()
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 100 * 1e3
        res["%s_%d" % (name, nbytes)] = {"us": round(us, 2), "gbs": round(nbytes / us / 1e3, 1)}
print(json.dumps(res))
