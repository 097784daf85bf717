"""Golden fixtures for the sketched-Newton row, made by the
REFERENCE ITSELF: proj/src/newton_sketch.cpp compiled unmodified into oracle/_ref
(against oracle/eigen_shim, whose LLT stands in for Eigen's).  Needs /root/reference
(this container), not the GPU box:

    make -C oracle ref && python tests/golden/make_golden_newton.py

Problems are generate_ar1_problem(n, d, seed) rounded to fp32 (the device path's
input precision) and promoted back to fp64 exactly, so fixtures and device runs
see the same data.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import HD3, Reference  # noqa: E402

N, D, SEED = 300, 12, 5
ROWS, SK_SEED = 64, 99


def main():
    r = Reference()
    g = {}
    a, y = r.ar1_problem(N, D, SEED)
    a32 = a.astype(np.float32)
    a = a32.astype(np.float64)
    g["ar1_raw_row0"] = r.ar1_problem(N, D, SEED)[0][0]
    g["a"], g["y"] = a32, y.astype(np.float32)
    x0 = np.linspace(-0.1, 0.1, D)
    g["x0"] = x0
    f, gr, h = r.logistic(a, y, x0)
    g["loss"], g["grad"], g["hsqrt"] = np.array(f), gr, h
    g["step_exact"] = r.sketched_step(a, y, x0)
    g["step_sketch"] = r.sketched_step(a, y, x0, HD3, ROWS, SK_SEED)
    # ridge path: a zero column makes the normal matrix singular; the 1e-10*trace ridge rescues it
    az = a.copy()
    az[:, 0] = 0.0
    g["a_zero_col"] = az.astype(np.float32)
    g["step_ridge"] = r.sketched_step(az, y, x0)
    for name, variant, rows, seed in (("exact", -1, 0, 0), ("sketch", HD3, ROWS, 7)):
        t = r.solve(a, y, variant, rows, 30, 1e-10, True, seed)
        g[f"solve_{name}_losses"] = t["losses"]
        g[f"solve_{name}_gaps"] = t["gaps"]
        g[f"solve_{name}_x"] = t["x"]
        g[f"solve_{name}_fstar"] = np.array(t["f_star"])
        g[f"solve_{name}_converged"] = np.array(t["converged"])
    out = os.path.join(HERE, "newton.npz")
    np.savez_compressed(out, **g)
    print("wrote", out, sorted(g))


if __name__ == "__main__":
    main()
