"""CUDA-event timings of the sketched-Newton entry points at the c6 shape (131072 x 256)."""
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
step, gr, f = nt._step_dev(p, x, sk)

def timeit(name, fn, reps=20):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record(); torch.cuda.synchronize()
    print(f"{name:28s} {a.elapsed_time(b) / reps * 1e3:9.1f} us")

timeit("eval (pass + reduce)", lambda: nt._eval_dev(p, x))
timeit("line count=4", lambda: nt._line_losses(p, x, step, 1.0, 4))
timeit("line count=41", lambda: nt._line_losses(p, x, step, 1.0, 41))
timeit("sketch apply (A, first m)", lambda: sk.apply(p.features))
timeit("sketched_step (warm)", lambda: nt._step_dev(p, x, sk))
timeit("exact step", lambda: nt._step_dev(p, x, None), reps=5)
