import sys; sys.path.insert(0, '.')
import numpy as np, paper_1610_06209_b200 as spn
from oracle.oracle import Oracle
g = dict(np.load('tests/golden/newton.npz'))
rel = lambda a, b: float(np.linalg.norm(np.asarray(a) - b) / np.linalg.norm(b))
p = spn.LogisticProblem(g['a'], g['y'])
x0 = g['x0']
print('loss', abs(spn.loss(p, x0) - g['loss']) / abs(g['loss']))
print('grad', rel(spn.gradient(p, x0), g['grad']))
print('hsqrt', rel(spn.hessian_sqrt(p, x0).cpu().numpy(), g['hsqrt']))
print('exact', rel(spn.sketched_step(p, x0), g['step_exact']))
sk = spn.SketchOperator(spn.SpinnerVariant.hd3_hd2_hd1, 300, 64, 99)
print('sketch', rel(spn.sketched_step(p, x0, sk), g['step_sketch']))
p2 = spn.LogisticProblem(g['a_zero_col'], g['y'])
print('ridge', rel(spn.sketched_step(p2, x0), g['step_ridge']))
for name, cfg in (("exact", spn.SketchConfig(max_iters=30)), ("sketch", spn.SketchConfig(spn.SpinnerVariant.hd3_hd2_hd1, 64, 30, 1e-10, True, 7))):
    t = spn.solve(p, cfg)
    print(name, len(t.losses), g[f'solve_{name}_losses'].size, t.f_star - g[f'solve_{name}_fstar'], rel(t.iterates[-1], g[f'solve_{name}_x']), t.seconds[:3])
