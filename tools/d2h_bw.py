"""Raw pinned device->host copy bandwidth (1D and 2D strided like the e2e hand-offs)."""
import time

import torch

n = 4 << 30
d = torch.empty(n // 16, dtype=torch.complex128, device="cuda")
h = torch.empty(n // 16, dtype=torch.complex128).pin_memory()
for it in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"1D D2H {n / dt / 1e9:.1f} GB/s")
s = torch.cuda.Stream()
t = time.perf_counter()
with torch.cuda.stream(s):
    for c in range(4):
        h[c * (n // 64):(c + 1) * (n // 64)].copy_(d[c * (n // 64):(c + 1) * (n // 64)], non_blocking=True)
torch.cuda.synchronize()
print(f"4 chunks D2H {n / 4 / (time.perf_counter() - t) / 1e9:.1f} GB/s")
t = time.perf_counter()
h.copy_(d, non_blocking=True)
d2 = torch.empty_like(d)
h2 = torch.empty_like(h).pin_memory()
torch.cuda.synchronize()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
t = time.perf_counter()
with torch.cuda.stream(s1):
    h.copy_(d, non_blocking=True)
with torch.cuda.stream(s2):
    h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
print(f"2 streams D2H {2 * n / (time.perf_counter() - t) / 1e9:.1f} GB/s")
