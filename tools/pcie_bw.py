"""Pinned host <-> device copy bandwidth on this box (context for the e2e number)."""
import torch
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, f in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        f()
    e1.record(); torch.cuda.synchronize()
    print(name, round(5 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1), "GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory(); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
with torch.cuda.stream(s1):
    for _ in range(5): d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    for _ in range(5): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); e1.record(); torch.cuda.synchronize()
print("both directions", round(10 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9, 1), "GB/s total")
