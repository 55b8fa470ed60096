"""Pinned D2H / H2D copy bandwidth of the box (test tooling): the ceiling of
the e2e leg (Z download, 3.2 GB per solve at n = 20000)."""
import json
import torch
n = 20000
x = torch.empty((n, n), dtype=torch.float64, device="cuda")
x.fill_(1.0)
h = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
out = {}
for name, f in (("d2h", lambda: h.copy_(x, non_blocking=True)), ("h2d", lambda: x.copy_(h, non_blocking=True))):
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        f()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 3
    out[name] = {"ms": round(ms, 2), "GB_s": round(x.numel() * 8 / ms / 1e6, 1)}
# chunked D2H (blocks of 256 columns on a side stream, as the library does)
s = torch.cuda.Stream()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s):
    a.record(s)
    for c in range(0, n, 256):
        h[c:c + 256].copy_(x[c:c + 256], non_blocking=True)
    b.record(s)
s.synchronize()
ms = a.elapsed_time(b)
out["d2h_blocks256"] = {"ms": round(ms, 2), "GB_s": round(x.numel() * 8 / ms / 1e6, 1)}
print(json.dumps(out))
