import sys, time; sys.path.insert(0, '.')
import torch, paper_1610_06209_b200 as spn
torch.cuda.init()
for n in (1 << 17, 1 << 14):
    for i in range(3):
        t0 = time.perf_counter(); p = spn._Plan.create(0, n, 2048, 2048, seed=i); t1 = time.perf_counter()
        del p; t2 = time.perf_counter()
        print(n, f"create {1e3*(t1-t0):.2f} ms destroy {1e3*(t2-t1):.2f} ms")
import ctypes, numpy as np
from oracle.oracle import Oracle
o = Oracle()
t0 = time.perf_counter(); o.realize(0, 1 << 17, 2048, 2048, 5); print("oracle realize", 1e3*(time.perf_counter()-t0), "ms")
