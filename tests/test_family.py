"""The rest of the spinner family: Gaussian circulant /
Toeplitz / skew-circulant G D2 H D1 (in-house FFT) and the dense Gaussian baseline,
against the reference itself (oracle/_ref runs proj/src/{spinner,transforms}.cpp:
StackedSpinner with these variants, CirculantOperator via the reference's FFT).

Bars: fp32 outputs <= 1e-5 relative L2 per vector (1e-5 also for the dense baseline's
fp32 accumulation); ids exact except near-ties (the reference's top-two |y| within
1e-5 relative: counted, must be rare); features as for the Hadamard variants.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CIRC, TOEP, SKEW, DENSE = 2, 3, 4, 5
RTOL = 1e-5


def row_rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b, axis=-1) / np.maximum(np.linalg.norm(b, axis=-1), 1e-30)


@pytest.fixture(scope="module")
def torch():
    import torch as t
    return t


CASES = [(CIRC, 8, 8, 8), (CIRC, 64, 32, 96), (CIRC, 1024, 1024, 1024), (CIRC, 8192, 512, 512),
         (TOEP, 16, 16, 16), (TOEP, 256, 100, 300), (TOEP, 4096, 1024, 1024),
         (SKEW, 8, 8, 8), (SKEW, 512, 512, 1024), (SKEW, 4096, 4096, 4096),
         (DENSE, 100, 50, 120), (DENSE, 256, 64, 64), (DENSE, 1024, 1024, 2048)]


@pytest.mark.parametrize("variant,n,m,k", CASES)
def test_apply_matches_reference(spn, oracle, ref, torch, variant, n, m, k):
    sp = spn.StackedSpinner(spn.SpinnerVariant(variant), n, m, k, 17 + n)
    x = oracle.gaussian_rows(n + variant, 24, n)
    y = sp.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    want = ref.apply(variant, n, m, k, 17 + n, 0.0, x)
    assert row_rel(y, want).max() <= RTOL


@pytest.mark.parametrize("variant,n,m,k", [c for c in CASES if c[1] <= 4096])
def test_hash_matches_reference(spn, oracle, ref, torch, variant, n, m, k):
    seeds = [spn.mix_seed(3 + n, t) for t in range(3)]
    h = spn.MultiTableHasher(spn.SpinnerVariant(variant), n, m, 3, table_seeds=seeds)
    x = oracle.gaussian_rows(200 + n, 40, n, unit=True)
    ids = h.hash_ids(torch.from_numpy(x).cuda()).cpu().numpy()
    want = ref.hash(variant, n, m, seeds, x)
    # near-ties: recompute the reference projections and measure the top-two gap
    bad = 0
    for t in range(3):
        y = ref.apply(variant, n, min(m, n), m, seeds[t], 0.0, x)
        a = np.sort(np.abs(y), axis=1)
        gap = (a[:, -1] - a[:, -2]) / np.maximum(a[:, -1], 1e-30) if m > 1 else np.ones(len(x))
        mism = ids[:, t] != want[:, t]
        assert np.all(gap[mism] < 1e-5), (t, gap[mism])
        bad += int(mism.sum())
    assert bad <= 2


@pytest.mark.parametrize("variant,n", [(CIRC, 64), (TOEP, 128), (SKEW, 1024), (DENSE, 96)])
def test_embed_matches_reference(spn, oracle, ref, torch, variant, n):
    dprime = 2 * n
    x = oracle.gaussian_rows(300 + n, 16, n)
    sp = spn.StackedSpinner(spn.SpinnerVariant(variant), n, min(n, dprime), dprime, 5)
    for kind, sigma in ((0, 3.0), (1, 0.0)):
        kk = spn.KernelKind.gaussian(sigma) if kind == 0 else spn.KernelKind.angular()
        got = spn.embed(spn.FeatureMap(sp, kk), torch.from_numpy(x).cuda()).cpu().numpy()
        want = ref.embed(variant, n, dprime, 5, kind, sigma, x)
        if kind == 0:
            assert row_rel(got, want).max() <= RTOL
        else:
            assert np.count_nonzero(got != want) <= 2  # sign flips only for |projection| ~ 0


def test_family_size_limits(spn):
    with pytest.raises(spn.SpinnerError):
        spn.StackedSpinner(spn.SpinnerVariant.gcirc_d2_hd1, 16384, 16, 16, 1)
    with pytest.raises(spn.SpinnerError):
        spn.StackedSpinner(spn.SpinnerVariant.gtoeplitz_d2_hd1, 8192, 16, 16, 1)


def test_default_scale_and_names(spn):
    assert spn.SpinnerSpec(spn.SpinnerVariant.gcirc_d2_hd1, 16, 16, 1).effective_scale() == 1.0
    assert spn.SpinnerSpec(spn.SpinnerVariant.hd3_hd2_hd1, 16, 16, 1).effective_scale() == 4.0
    for name in ("HD3HD2HD1", "HDgHD2HD1", "GcircD2HD1", "GToeplitzD2HD1", "GSkewCircD2HD1", "GaussianDense"):
        assert spn.variant_to_string(spn.variant_from_string(name)) == name
    with pytest.raises(spn.DimensionError):
        spn.StackedSpinner(spn.SpinnerVariant.gcirc_d2_hd1, 12, 12, 12, 1)  # Hadamard stage needs pow2 n
