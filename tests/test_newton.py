"""Sketched Newton for logistic regression (reference
proj/src/newton_sketch.cpp:45-204).

* CPU: the C restatement (oracle/spinner_oracle.c) against the golden fixtures made
  by the reference itself (tests/golden/newton.npz, make_golden_newton.py), and the
  library's host AR(1) generator against the reference's.
* GPU (-m gpu): the device path through the C ABI against the same fixtures.
  Bars: fp64 quantities computed from the same fp32 data (loss, gradient, exact
  steps, f_star): 1e-9 relative; hessian_sqrt (fp32 output): 1e-7; sketched steps
  (fp32 spinner sketch, measured 6.7e-7 on an AR(1) rho = 0.99 problem): 1e-5
  relative; solve traces: the same iteration count, f_star and final iterate.
"""
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
NEWTON = os.path.join(HERE, "golden", "newton.npz")


@pytest.fixture(scope="module")
def gn():
    return dict(np.load(NEWTON))


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


# ------------------------------------------------------------------ CPU: oracle pinning
def test_oracle_logistic_matches_reference(oracle, gn):
    a, y, x0 = gn["a"].astype(np.float64), gn["y"].astype(np.float64), gn["x0"]
    f, g, h = oracle.logistic(a, y, x0)
    assert f == float(gn["loss"])
    assert np.array_equal(g, gn["grad"])
    assert np.array_equal(h, gn["hsqrt"])


def test_oracle_steps_match_reference(oracle, gn):
    a, y, x0 = gn["a"].astype(np.float64), gn["y"].astype(np.float64), gn["x0"]
    rc, s = oracle.sketched_step(a, y, x0)
    assert rc == 0 and np.array_equal(s, gn["step_exact"])
    N, m = 512, 64
    d1, d2, d3 = oracle.realize(0, N, m, m, 99)
    rc, s = oracle.sketched_step(a, y, x0, N, m, np.sqrt(N), 1 / np.sqrt(m), (d1[0], d2[0], d3[0]))
    assert rc == 0 and np.array_equal(s, gn["step_sketch"])
    rc, s = oracle.sketched_step(gn["a_zero_col"].astype(np.float64), y, x0)  # ridge retry path
    assert rc == 0 and np.array_equal(s, gn["step_ridge"])


def test_oracle_singular_and_dimension(oracle, gn):
    y, x0 = gn["y"].astype(np.float64), gn["x0"]
    rc, _ = oracle.sketched_step(np.zeros((300, 12)), y, x0)  # trace 0: the ridge cannot help
    assert rc == 7
    N, m = 512, 8  # m < d
    d1, d2, d3 = oracle.realize(0, N, m, m, 1)
    rc, _ = oracle.sketched_step(gn["a"].astype(np.float64), y, x0, N, m, np.sqrt(N), 1 / np.sqrt(m),
                                 (d1[0], d2[0], d3[0]))
    assert rc == 1


def test_host_ar1_generator_matches_reference(spn, gn):
    import ctypes
    from paper_1610_06209_b200 import newton
    n, d = gn["a"].shape
    f = np.zeros((n, d), np.float32)
    y = np.zeros(n, np.float32)
    spn._check(newton._ar1(n, d, 5, f.ctypes.data_as(ctypes.c_void_p), y.ctypes.data_as(ctypes.c_void_p)))
    assert np.array_equal(f, gn["a"]) and np.array_equal(y, gn["y"])
    assert np.float32(gn["ar1_raw_row0"][0]) == f[0, 0]


# ------------------------------------------------------------------------ GPU parity
@pytest.fixture(scope="module")
def prob(spn, gn):
    return spn.LogisticProblem(gn["a"], gn["y"])


@pytest.mark.gpu
def test_loss_gradient_hessian_sqrt(spn, prob, gn):
    x0 = gn["x0"]
    assert abs(spn.loss(prob, x0) - float(gn["loss"])) <= 1e-9 * abs(float(gn["loss"]))
    assert rel(spn.gradient(prob, x0), gn["grad"]) <= 1e-9
    h = spn.hessian_sqrt(prob, x0).cpu().numpy()
    assert rel(h, gn["hsqrt"]) <= 1e-7


@pytest.mark.gpu
def test_exact_step(spn, prob, gn):
    s = spn.sketched_step(prob, gn["x0"], spn.SketchOperator())
    assert rel(s, gn["step_exact"]) <= 1e-9


@pytest.mark.gpu
def test_sketched_step(spn, prob, gn):
    sk = spn.SketchOperator(spn.SpinnerVariant.hd3_hd2_hd1, prob.observations(), 64, 99)
    s = spn.sketched_step(prob, gn["x0"], sk)
    assert rel(s, gn["step_sketch"]) <= 1e-5


@pytest.mark.gpu
def test_ridge_retry_and_singular(spn, gn):
    p = spn.LogisticProblem(gn["a_zero_col"], gn["y"])
    s = spn.sketched_step(p, gn["x0"])
    assert s[0] == 0.0 and rel(s, gn["step_ridge"]) <= 1e-6
    z = spn.LogisticProblem(np.zeros_like(gn["a"]), gn["y"])
    with pytest.raises(spn.SingularSystemError):
        spn.sketched_step(z, gn["x0"])


@pytest.mark.gpu
def test_sketch_rows_below_d(spn, prob, gn):
    sk = spn.SketchOperator(spn.SpinnerVariant.hd3_hd2_hd1, prob.observations(), 8, 1)
    with pytest.raises(spn.DimensionError):
        spn.sketched_step(prob, gn["x0"], sk)


@pytest.mark.gpu
def test_line_search_candidates(spn, oracle, prob, gn):
    from paper_1610_06209_b200 import newton
    x = newton._dvec(prob, gn["x0"])
    st = newton._dvec(prob, gn["step_exact"])
    got = newton._line_losses(prob, x, st, 1.0, 41)
    a, y = gn["a"].astype(np.float64), gn["y"].astype(np.float64)
    for k in (0, 1, 5, 40):
        want = oracle.logistic(a, y, gn["x0"] + 2.0 ** -k * gn["step_exact"])[0]
        assert abs(got[k] - want) <= 1e-12 * abs(want)


@pytest.mark.gpu
def test_solve_exact_and_sketched(spn, prob, gn):
    for name, cfg in (("exact", spn.SketchConfig(max_iters=30)),
                      ("sketch", spn.SketchConfig(spn.SpinnerVariant.hd3_hd2_hd1, 64, 30, 1e-10, True, 7))):
        t = spn.solve(prob, cfg)
        fstar = float(gn[f"solve_{name}_fstar"])
        assert abs(t.f_star - fstar) <= 1e-10 * abs(fstar)
        assert t.converged == bool(gn[f"solve_{name}_converged"])
        assert t.gaps[-1] <= 1e-10
        assert rel(t.iterates[-1], gn[f"solve_{name}_x"]) <= 1e-6
        assert len(t.losses) == gn[f"solve_{name}_losses"].size
        # the fp32 sketch perturbs each sketched step by ~1e-6 relative -> losses agree to ~1e-8
        tol = 1e-9 if name == "exact" else 1e-7
        assert np.allclose(t.losses, gn[f"solve_{name}_losses"], rtol=tol, atol=0)


@pytest.mark.gpu
def test_larger_problem_vs_oracle(spn, oracle):
    """n = 5000 (pads to 8192, multi-pass sketch), d = 64 (two 32-wide Cholesky panels + d % 64 == 0)."""
    a, y = oracle.ar1_problem(5000, 64, 11)
    a32 = a.astype(np.float32)
    a = a32.astype(np.float64)
    p = spn.LogisticProblem(a32, y)
    x = np.full(64, 0.01)
    f, g, _ = oracle.logistic(a, y, x)
    assert abs(spn.loss(p, x) - f) <= 1e-9 * abs(f)
    assert rel(spn.gradient(p, x), g) <= 1e-9
    rc, s = oracle.sketched_step(a, y, x)
    assert rc == 0 and rel(spn.sketched_step(p, x), s) <= 1e-8
    N, m = 8192, 512
    d1, d2, d3 = oracle.realize(0, N, m, m, 3)
    rc, s = oracle.sketched_step(a, y, x, N, m, np.sqrt(N), 1 / np.sqrt(m), (d1[0], d2[0], d3[0]))
    sk = spn.SketchOperator(spn.SpinnerVariant.hd3_hd2_hd1, 5000, 512, 3)
    assert rc == 0 and rel(spn.sketched_step(p, x, sk), s) <= 1e-5
