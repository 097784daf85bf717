"""Run one config's hot path on a reduced batch (for ncu captures): warm-up + 2 launches."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1610_06209_b200 as spn

cfg, batch = sys.argv[1], int(sys.argv[2])
V = spn.SpinnerVariant
if cfg == "c3":
    h = spn.MultiTableHasher(V.hd3_hd2_hd1, 16384, 16384, 8, seed=3)
    x = torch.empty(batch, 16384, device="cuda")
    for r0 in range(0, batch, 1 << 16):
        x[r0:r0 + (1 << 16)] = torch.randn(min(1 << 16, batch - r0), 16384, device="cuda")
    run = lambda: h.hash_ids(x)
elif cfg == "c4":
    sk = spn.SketchOperator(V.hd3_hd2_hd1, 1 << 17, 2048, 11, mode="random", p_seed=77)
    x = torch.randn(1 << 17, batch, device="cuda")
    run = lambda: sk.apply(x)
elif cfg == "c5":
    sp = spn.StackedSpinner(V.gauss3, 1 << 20, 1 << 20, 1 << 20, 13, scale=1.0)
    x = torch.randn(batch, 1 << 20, device="cuda")
    y = torch.empty_like(x)
    run = lambda: sp.apply(x, relu=True, out=y)
elif cfg == "c2":
    sp = spn.StackedSpinner(V.hd3_hd2_hd1, 1024, 1024, 4096, 5)
    fm = spn.FeatureMap(sp, spn.KernelKind.gaussian(5.0))
    x = torch.rand(batch, 784, device="cuda")
    out = torch.empty(batch, 8192, device="cuda")
    run = lambda: spn.embed(fm, x, out=out)
elif cfg == "c1":
    sp = spn.StackedSpinner(V.hd3_hd2_hd1, 1024, 1024, 1024, 42, scale=1.0)
    x = torch.randn(batch, 1024, device="cuda")
    y = torch.empty_like(x)
    run = lambda: sp.plan.hash(x, y_out=y)
for _ in range(3 if cfg != "c3" or batch < 65536 else 1):
    run()
torch.cuda.synchronize()
print("ok", cfg, batch)
