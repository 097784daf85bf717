import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1610_06209_b200 as spn
rows = 1 << 17
h = spn.MultiTableHasher(spn.SpinnerVariant.hd3_hd2_hd1, 16384, 16384, 8, seed=3)
x = torch.randn(rows, 16384, pin_memory=True).numpy()
h.plan.hash(x[:4096])
best = 0
for _ in range(3):
    t0 = time.perf_counter(); h.plan.hash(x); dt = time.perf_counter() - t0
    best = max(best, rows / dt)
print(f"streams={os.environ.get('SPN_HOST_STREAMS')} chunk={os.environ.get('SPN_HOST_CHUNK_MB')}: {best:.0f} vec/s, {best * 65536 / 1e9:.1f} GB/s", flush=True)
