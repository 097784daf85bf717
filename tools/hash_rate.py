"""FP32 butterfly rate (adds / clk / SM) of the fused 8-table hash kernel by vector length: how the
register / thread split (R x T) of each size uses the FP32 pipe.  usage: python tools/hash_rate.py"""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1610_06209_b200 as spn

V = spn.SpinnerVariant
for ln in (10, 11, 12, 13, 14):
    n = 1 << ln
    batch = (1 << 31) // (4 * n)  # 2 GiB of input
    h = spn.MultiTableHasher(V.hd3_hd2_hd1, n, n, 8, seed=3)
    x = torch.randn(batch, n, device="cuda")
    for _ in range(2):
        h.hash_ids(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        h.hash_ids(x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    adds = batch * 8 * 3 * n * ln
    print(f"n=2^{ln} R={1 << ((ln + 1) // 2)} T={1 << (ln // 2)}: {ms:.2f} ms, {adds / (ms * 1e-3) / (148 * 1.965e9):.1f} adds/clk/SM "
          f"(peak 128), {batch * n * 4 / (ms * 1e-3) / 1e9:.0f} GB/s of x")
    del x, h
