import torch, time
n = 1 << 28
d = torch.empty(n, dtype=torch.complex128, device="cuda")
h = torch.empty(n, dtype=torch.complex128, pin_memory=True)
for _ in range(2): h.copy_(d, non_blocking=True); torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5): h.copy_(d, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 5
print(f"D2H 4 GiB: {dt*1e3:.1f} ms = {16*n/dt/1e9:.1f} GB/s")
# two halves on two streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): h[: n // 2].copy_(d[: n // 2], non_blocking=True)
    with torch.cuda.stream(s2): h[n // 2:].copy_(d[n // 2:], non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 5
print(f"D2H 2 streams: {dt*1e3:.1f} ms = {16*n/dt/1e9:.1f} GB/s")
