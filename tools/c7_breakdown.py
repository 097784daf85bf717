"""Host/device breakdown of one c7 collision-curve step (20000 pairs x 100 trials, n = 256, m = 64)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1610_06209_b200 as spn

rng = np.random.default_rng(88)
P, n, m, trials = 20000, 256, 64, 100
ang = np.pi * (np.arange(P) + 0.5) / P
x = rng.standard_normal((P, n)); u = rng.standard_normal((P, n))
x /= np.linalg.norm(x, axis=1, keepdims=True)
u -= np.sum(u * x, axis=1, keepdims=True) * x; u /= np.linalg.norm(u, axis=1, keepdims=True)
y = np.cos(ang)[:, None] * x + np.sin(ang)[:, None] * u
cx = torch.from_numpy(x.astype(np.float32)).cuda(); cy = torch.from_numpy(y.astype(np.float32)).cuda()
cd = 2.0 * np.sin(ang / 2.0)
fac = spn.make_hasher_factory(spn.SpinnerVariant.hd3_hd2_hd1, n, m)
for it in range(3):
    spn.collision_curve((cx, cy, cd), fac, trials, 90 + it)
torch.cuda.synchronize()
t0 = time.perf_counter()
for it in range(10):
    spn.collision_curve((cx, cy, cd), fac, trials, 100 + it)
torch.cuda.synchronize()
print(f"collision_curve: {(time.perf_counter() - t0) / 10 * 1e3:.2f} ms/step")
t0 = time.perf_counter()
for it in range(10):
    h = spn.MultiTableHasher(spn.SpinnerVariant.hd3_hd2_hd1, n, m, trials, seed=200 + it)
torch.cuda.synchronize()
print(f"  plan (100 tables): {(time.perf_counter() - t0) / 10 * 1e3:.2f} ms")
xy = torch.stack((cx, cy), dim=1).reshape(2 * P, n).contiguous()
t0 = time.perf_counter()
for it in range(10):
    bad = bool((spn.check_rows(xy) != 0).any())
torch.cuda.synchronize()
print(f"  check_rows + sync: {(time.perf_counter() - t0) / 10 * 1e3:.2f} ms")
t0 = time.perf_counter()
for it in range(10):
    ids = h.plan.hash(xy)
torch.cuda.synchronize()
print(f"  hash 40000 x 100 tables: {(time.perf_counter() - t0) / 10 * 1e3:.2f} ms")
