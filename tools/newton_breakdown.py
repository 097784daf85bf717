"""Host/device time breakdown of one c6 Newton iteration (plan creation, step, line search)."""
import sys, os, time
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
sk = None
for it in range(6):
    torch.cuda.synchronize(); tz = time.perf_counter()
    del sk
    torch.cuda.synchronize(); t0 = time.perf_counter()
    sk = spn.SketchOperator(spn.SpinnerVariant.hd3_hd2_hd1, N, m, spn.mix_seed(3, it))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    step, gr, f = nt._step_dev(p, x, sk)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    s, _ = nt._backtrack(p, x, step, float(f.item()), float(torch.dot(gr, step).item()))
    torch.cuda.synchronize(); t3 = time.perf_counter()
    step2, _, _ = nt._step_dev(p, x, sk)  # second step with a warm plan
    torch.cuda.synchronize(); t4 = time.perf_counter()
    print(f"del {1e3*(t0-tz):.2f} ms  plan {1e3*(t1-t0):.2f} ms  step {1e3*(t2-t1):.2f} ms  line {1e3*(t3-t2):.2f} ms  warm step {1e3*(t4-t3):.2f} ms")
