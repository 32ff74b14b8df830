"""Pinned host<->device bandwidth on this box (context for the e2e line)."""
import torch

n = 512 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h2 = torch.empty(n // 2, dtype=torch.uint8).pin_memory()
d2 = torch.empty(n // 2, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    d.copy_(h, non_blocking=True)
e1.record()
torch.cuda.synchronize()
print(f"H2D {3 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s")
e0.record()
for _ in range(3):
    h.copy_(d, non_blocking=True)
e1.record()
torch.cuda.synchronize()
print(f"D2H {3 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s")
torch.cuda.synchronize()
e0.record()
with torch.cuda.stream(s1):
    s1.wait_event(e0)
    d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    s2.wait_event(e0)
    h2.copy_(d2, non_blocking=True)
torch.cuda.current_stream().wait_stream(s1)
torch.cuda.current_stream().wait_stream(s2)
e1.record()
torch.cuda.synchronize()
print(f"duplex H2D 512 MB + D2H 256 MB: {e0.elapsed_time(e1):.2f} ms")
