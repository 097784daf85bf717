"""Gram-matrix consumers (reference proj/src/kernels.cpp:38-114,
tests restated from proj/tests/test_kernels.cpp:55-133 and acceptance criterion 4).

Device results against the reference's own gram_exact / gram_approx / gram_error
(oracle/_ref) on the same fp32 points: gram_exact to 1e-12 (fp64 from identical inputs);
gram_approx gaussian to 2e-6 absolute (fp32 features, |entry| <= 1); angular entries are
1/2 + <s_i, s_j>/(2d') with sign features, equal except sign flips of near-zero
projections (fp32 vs fp64), bounded by a 0.2 % entry budget of 1/d' steps.
"""
import math

import numpy as np
import pytest

from oracle.oracle import HD3, HDG

pytestmark = pytest.mark.gpu


def blob(oracle, n, count, seed):
    return oracle.rng_fill(seed, "gaussian", count * n).reshape(count, n).astype(np.float32)


def test_gram_exact_anchors(spn):
    a, b = [1.0, 0.0], [0.0, 1.0]
    k = spn.gram_exact(np.array([a, a, b]), spn.KernelKind.angular())
    assert abs(k[0, 1] - 1.0) < 1e-15 and abs(k[0, 2] - 0.5) < 1e-15
    sigma = 0.7
    c = [sigma * math.sqrt(2.0), 0.0]
    kg = spn.gram_exact(np.array([[0.0, 0.0], c]), spn.KernelKind.gaussian(sigma))
    assert kg[0, 0] == 1.0 and abs(kg[0, 1] - math.exp(-1.0)) < 1e-7  # c rounded to fp32
    with pytest.raises(spn.DomainError):
        spn.gram_exact(np.zeros((1, 2)), spn.KernelKind.angular())


def test_gram_error_anchors(spn):
    k = np.eye(2)
    assert spn.gram_error(k, k) == 0.0
    assert abs(spn.gram_error(k, np.zeros((2, 2))) - 1.0) < 1e-15
    kt = k.copy()
    kt[0, 1] = kt[1, 0] = 0.1
    assert abs(spn.gram_error(k, kt) - 0.1) < 1e-13
    with pytest.raises(spn.DomainError):
        spn.gram_error(np.zeros((2, 2)), k)


@pytest.mark.parametrize("kind", ["gaussian", "angular"])
def test_gram_exact_matches_reference(spn, oracle, ref, kind):
    pts = blob(oracle, 64, 300, 77)
    kk = spn.KernelKind.gaussian(4.0) if kind == "gaussian" else spn.KernelKind.angular()
    got = spn.gram_exact(pts, kk)
    want = ref.gram_exact(pts, 0 if kind == "gaussian" else 1, 4.0)
    assert np.abs(got - want).max() <= 1e-12


@pytest.mark.parametrize("variant", [HD3, HDG])
@pytest.mark.parametrize("dprime", [32, 128])
def test_gram_approx_matches_reference(spn, oracle, ref, variant, dprime):
    n, count = 64, 300
    pts = blob(oracle, n, count, 78)
    seed = spn.mix_seed(6000 + variant, dprime * 100)
    sp = spn.StackedSpinner(spn.SpinnerVariant(variant), n, min(n, dprime), dprime, seed)
    # gaussian
    got = spn.gram_approx(spn.FeatureMap(sp, spn.KernelKind.gaussian(4.0)), pts)
    want = ref.gram_approx(variant, n, dprime, seed, 0, 4.0, pts)
    assert np.abs(got - want).max() <= 2e-6
    assert np.all(np.diag(got) == 1.0) and np.array_equal(got, got.T)
    # angular: multiples of 1/d' apart, rare
    got = spn.gram_approx(spn.FeatureMap(sp, spn.KernelKind.angular()), pts)
    want = ref.gram_approx(variant, n, dprime, seed, 1, 0.0, pts)
    diff = np.abs(got - want) * dprime
    assert np.allclose(diff, np.round(diff), atol=1e-9)
    assert np.count_nonzero(diff > 0.5) <= 0.002 * count * count
    # the acceptance metric itself
    ex = ref.gram_exact(pts, 0, 4.0)
    e_got = spn.gram_error(ex, spn.gram_approx(spn.FeatureMap(sp, spn.KernelKind.gaussian(4.0)), pts))
    e_ref = ref.gram_error(ex, ref.gram_approx(variant, n, dprime, seed, 0, 4.0, pts))
    assert abs(e_got - e_ref) <= 1e-5 * e_ref


def test_antipodal_angular_and_scalar_oracle(spn, oracle):
    n, dprime = 8, 8  # test_kernels.cpp:71-123 (HD3 family)
    x = oracle.gaussian_rows(9, 1, n)[0]
    sp = spn.StackedSpinner(spn.SpinnerVariant.hd3_hd2_hd1, n, n, dprime, 8)
    k = spn.gram_approx(spn.FeatureMap(sp, spn.KernelKind.angular()), np.stack([x, -x]))
    assert k[0, 0] == 1.0 and k[1, 1] == 1.0 and abs(k[0, 1]) < 1e-15 and k[0, 1] == k[1, 0]
    pts = oracle.gaussian_rows(10, 3, n)
    got = spn.gram_approx(spn.FeatureMap(sp, spn.KernelKind.angular()), pts)
    proj = sp.apply(pts)
    s = np.where(np.asarray(proj) < 0, -1.0, 1.0)
    for i in range(3):
        for j in range(3):
            want = 1.0 - np.count_nonzero(s[i] != s[j]) / dprime
            assert abs(got[i, j] - want) < 1e-12
