"""HBM rate of the fused apply kernel (y = scale * H D3 H D2 H D1 x, one block, fp32 in / out) by vector
length, against the measured copy peak.  usage: python tools/apply_rate.py [peak_gbs]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1610_06209_b200 as spn

peak = float(sys.argv[1]) if len(sys.argv) > 1 else 6548.2
V = spn.SpinnerVariant
for ln in (10, 11, 12, 13, 14):
    n = 1 << ln
    batch = (1 << 30) // (4 * n)  # 1 GiB in + 1 GiB out: beyond the 126 MB L2
    sp = spn.StackedSpinner(V.hd3_hd2_hd1, n, n, n, 42, scale=1.0)
    x = torch.randn(batch, n, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        sp.apply(x, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        sp.apply(x, out=y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    gbs = 2 * batch * n * 4 / (ms * 1e-3) / 1e9
    adds = batch * 3 * n * ln / (ms * 1e-3) / (148 * 1.965e9)
    print(f"n=2^{ln}: {ms:.3f} ms, {gbs:.0f} GB/s = {gbs / peak:.2f} of the HBM copy peak, {adds:.1f} adds/clk/SM")
    del x, y, sp
