"""Three warm sketched Newton steps at the c6 shape (for an ncu launch list)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1610_06209_b200 as spn
from paper_1610_06209_b200 import newton as nt

N, d, m = 1 << 17, 256, 2048
g = torch.Generator(device="cuda"); g.manual_seed(1)
p = spn.LogisticProblem(torch.randn((N, d), device="cuda", generator=g),
                        torch.where(torch.rand(N, device="cuda", generator=g) < 0.5, -1.0, 1.0))
p.workspace(m)
x = torch.full((d,), 0.01, dtype=torch.float64, device="cuda")
sk = spn.SketchOperator(spn.SpinnerVariant.hd3_hd2_hd1, N, m, 5)
for _ in range(3):
    step, gr, f = nt._step_dev(p, x, sk)
    s, _ = nt._backtrack(p, x, step, float(f.item()), float(torch.dot(gr, step).item()))
torch.cuda.synchronize()
print("ok")
