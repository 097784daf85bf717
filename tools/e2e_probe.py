"""H2D / D2H pinned rates on this box, and config 3's host pipeline (spn_hash_f32_host) at several chunk sizes."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
n = 1 << 28
d = torch.empty(n, device="cuda"); h = torch.empty(n, pin_memory=True)
for name, f in [("D2H", lambda: h.copy_(d, non_blocking=True)), ("H2D", lambda: d.copy_(h, non_blocking=True))]:
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5): f()
    torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / 5
    print(name, f"1 GiB: {4 * n / dt / 1e9:.1f} GB/s", flush=True)
for mb in (16, 48, 128):
    m = mb << 18
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for i in range(0, n, m): d[i:i + m].copy_(h[i:i + m], non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"H2D in {mb} MB pieces: {4 * n / dt / 1e9:.1f} GB/s", flush=True)
del d, h
import paper_1610_06209_b200 as spn
rows = 1 << 17
h = spn.MultiTableHasher(spn.SpinnerVariant.hd3_hd2_hd1, 16384, 16384, 8, seed=3)
x = torch.randn(rows, 16384, pin_memory=True).numpy()
h.plan.hash(x[:1024])
for mb in (48, 96, 192):
    os.environ["SPN_HOST_CHUNK_MB"] = str(mb)
    t0 = time.perf_counter(); h.plan.hash(x); dt = time.perf_counter() - t0
    print(f"c3 host pipeline {rows} rows (chunk env {mb} MB, read once per process): {rows / dt:.0f} vec/s, {x.nbytes / dt / 1e9:.1f} GB/s", flush=True)
