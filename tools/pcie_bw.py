import torch, time
n = 1 << 28  # 1 GiB fp32
d = torch.empty(n, device="cuda"); h = torch.empty(n, pin_memory=True)
for name, f in [("D2H", lambda: h.copy_(d, non_blocking=True)), ("H2D", lambda: d.copy_(h, non_blocking=True))]:
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5): f()
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 5
    print(name, f"{4 * n / dt / 1e9:.1f} GB/s")
# concurrent both directions on two streams
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
d2 = torch.empty(n // 8, device="cuda"); h2 = torch.empty(n // 8, pin_memory=True)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): h.copy_(d, non_blocking=True)
    with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 5
print("D2H 1 GiB with concurrent H2D 128 MiB:", f"{4 * n / dt / 1e9:.1f} GB/s D2H")
# split D2H into 2 concurrent streams
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): h[: n // 2].copy_(d[: n // 2], non_blocking=True)
    with torch.cuda.stream(s2): h[n // 2 :].copy_(d[n // 2 :], non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 5
print("D2H on 2 streams:", f"{4 * n / dt / 1e9:.1f} GB/s")
