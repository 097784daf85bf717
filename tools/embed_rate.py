"""HBM rate of the fused Gaussian-feature kernel (B stacked blocks: n inputs -> [cos || sin], 2 B n outputs)
by vector length, against the measured copy peak.  usage: python tools/embed_rate.py [peak_gbs [blocks]]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1610_06209_b200 as spn

peak = float(sys.argv[1]) if len(sys.argv) > 1 else 6548.2
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
V = spn.SpinnerVariant
for ln in (10, 11, 12, 13, 14):
    n = 1 << ln
    batch = (1 << 30) // (8 * B * n)  # 1 GiB out
    sp = spn.StackedSpinner(V.hd3_hd2_hd1, n, n, B * n, 5)
    fm = spn.FeatureMap(sp, spn.KernelKind.gaussian(5.0))
    x = torch.rand(batch, n, device="cuda")
    out = torch.empty(batch, 2 * B * n, device="cuda")
    for _ in range(3):
        spn.embed(fm, x, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        spn.embed(fm, x, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    gbs = (1 + 2 * B) * batch * n * 4 / (ms * 1e-3) / 1e9
    print(f"n=2^{ln}: {ms:.3f} ms, {gbs:.0f} GB/s = {gbs / peak:.2f} of the HBM copy peak")
    del x, out, sp, fm
