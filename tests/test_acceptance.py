"""The reference's acceptance criteria that touch the hot path, restated against the device
path with oracles independent of both fast paths (tests/acceptance.cpp, tests/oracles.hpp):

  * criterion 1 — every variant equals the dense composition of explicit matrices built from the
    realised diagonals, H[i][j] = (-1)^popcount(i & j) / sqrt(n) (oracles.hpp:19-33,67-98),
    n in {4..32}, with truncation (m < n) and stacking (k > m) (acceptance.cpp:35-49);
  * embed anchors: self-similarity 1 and the cos-difference identity (test_kernels.cpp:28-53);
  * hash invariances under positive scaling and negation at every fused n (test_lsh.cpp:37-55).

fp32 device arithmetic against fp64 oracles: relative L2 <= 1e-5 per vector (BASELINE.json).
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RTOL = 1e-5


@pytest.fixture(scope="module")
def torch():
    import torch as t
    return t


def sylvester(n):
    i = np.arange(n)
    pc = np.vectorize(lambda v: bin(v).count("1"))(i[:, None] & i[None, :])
    return np.where(pc % 2 == 0, 1.0, -1.0) / math.sqrt(n)


def dense_stack(sp, n, m, k, scale):
    H = sylvester(n)
    d1, d2, d3 = (a.astype(np.float32).astype(np.float64) for a in sp.plan.diagonals())
    rows = []
    for b in range(d1.shape[1]):
        M = H @ np.diag(d3[0, b]) @ H @ np.diag(d2[0, b]) @ H @ np.diag(d1[0, b])
        rows.append(scale * M[:m])
    return np.concatenate(rows, axis=0)[:k]


def rel(got, want):
    return np.linalg.norm(got - want, axis=1) / np.linalg.norm(want, axis=1)


@pytest.mark.parametrize("n", [4, 8, 16, 32])
@pytest.mark.parametrize("variant", ["hd3_hd2_hd1", "hdg_hd2_hd1"])
def test_dense_oracle_equivalence(spn, torch, n, variant):
    v = getattr(spn.SpinnerVariant, variant)
    rng = np.random.default_rng(n)
    for trial, (m, k) in enumerate([(n, n), (n // 2 + 1, n // 2 + 1), (n // 2, 3 * n // 2 + 1)]):
        sp = spn.StackedSpinner(v, n, m, k, 21 + 100 * trial)
        W = dense_stack(sp, n, m, k, math.sqrt(n))
        x = rng.standard_normal((16, n)).astype(np.float32)
        y = sp.apply(torch.from_numpy(x).cuda()).cpu().numpy()
        assert rel(y, x.astype(np.float64) @ W.T).max() <= RTOL, (n, m, k)


@pytest.mark.parametrize("n", [64, 1024, 4096])
def test_embed_anchors(spn, torch, n):
    k, sigma = 2 * n, 3.0
    sp = spn.StackedSpinner(spn.SpinnerVariant.hd3_hd2_hd1, n, n, k, 9)
    fm = spn.FeatureMap(sp, spn.KernelKind.gaussian(sigma))
    rng = np.random.default_rng(1)
    x = rng.random((8, n)).astype(np.float32)
    y = rng.random((8, n)).astype(np.float32)
    fx = spn.embed(fm, torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64)
    fy = spn.embed(fm, torch.from_numpy(y).cuda()).cpu().numpy().astype(np.float64)
    # self-similarity: (1/k) sum cos^2 + sin^2 = 1
    assert np.max(np.abs(np.sum(fx * fx, axis=1) - 1.0)) < 1e-5
    # cos-difference identity: <f(x), f(y)> = (1/k) sum_i cos(t_i(x) - t_i(y)), t = z / sigma
    zx = sp.apply(torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64) / sigma
    zy = sp.apply(torch.from_numpy(y).cuda()).cpu().numpy().astype(np.float64) / sigma
    want = np.mean(np.cos(zx - zy), axis=1)
    assert np.max(np.abs(np.sum(fx * fy, axis=1) - want)) < 1e-5


@pytest.mark.parametrize("n", [2, 16, 256, 1024, 2048, 8192, 16384])
def test_hash_scale_and_negation(spn, torch, n):
    sp = spn.StackedSpinner(spn.SpinnerVariant.hd3_hd2_hd1, n, n, n, 4)
    x = torch.from_numpy(np.random.default_rng(n).standard_normal((64, n)).astype(np.float32)).cuda()
    ids = sp.plan.hash(x).cpu().numpy()[:, 0]
    assert np.array_equal(sp.plan.hash(x * 4.0).cpu().numpy()[:, 0], ids)  # powers of 2: exact scaling
    neg = sp.plan.hash(-x).cpu().numpy()[:, 0]
    assert np.array_equal(neg % n, ids % n) and np.all((neg >= n) != (ids >= n))
    assert np.array_equal(sp.plan.hash(x).cpu().numpy()[:, 0], ids)  # determinism


@pytest.mark.parametrize("logn", [0, 1, 2, 5, 10, 13, 14, 15, 17, 20])
def test_fwht_normalized_matches_oracle(spn, oracle, torch, logn):
    """fwht_normalized (transforms.cpp:52-71) on the device, batch and single-vector host calls."""
    n = 1 << logn
    x = oracle.gaussian_rows(logn + 1, 3, n)
    want = np.stack([oracle.fwht(r.astype(np.float64)) for r in x.astype(np.float32)])
    got = spn.fwht_normalized(torch.from_numpy(x).cuda()).cpu().numpy()
    assert rel(got, want).max() <= RTOL
    assert rel(spn.fwht_normalized(x[:1].astype(np.float64)), want[:1]).max() <= RTOL
    if n >= 2:  # involution, in place on the device
        t = torch.from_numpy(x).cuda()
        spn.fwht_normalized(t, out=t)
        spn.fwht_normalized(t, out=t)
        assert rel(t.cpu().numpy(), x.astype(np.float64)).max() <= RTOL


def test_fwht_kats_and_diag(spn, torch):
    h2 = spn.fwht_normalized(np.array([1.0, 0.0]))
    assert np.allclose(h2, [1 / math.sqrt(2), 1 / math.sqrt(2)], atol=1e-6)  # test_transforms.cpp:11-15
    assert np.allclose(spn.fwht_normalized(np.array([1.0, 2.0, 3.0, 4.0])), [5.0, -1.0, -2.0, 0.0], atol=1e-6)
    assert np.array_equal(spn.diag_matvec([2.0, -1.0, 0.5], [1.0, 3.0, -4.0]), [2.0, -3.0, -2.0])
    d = torch.tensor([2.0, -1.0, 0.5], device="cuda")
    x = torch.tensor([[1.0, 3.0, -4.0], [0.0, 1.0, 2.0]], device="cuda")
    assert torch.equal(spn.diag_matvec(d, x), torch.tensor([[2.0, -3.0, -2.0], [0.0, -1.0, 1.0]], device="cuda"))


# -------------------------------------------- circulant-family operators (transforms.cpp:64-226)
def dense_circulant(kind, row, col=None):
    """oracles.hpp:35-58: the explicit matrices."""
    n = row.size
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    if kind == 0:
        return row[(j - i) % n]
    if kind == 1:
        return np.where(i >= j, col[np.abs(i - j)], row[np.abs(j - i)])
    return np.where(j >= i, row[(j - i) % n], -row[(n + j - i) % n])


@pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 64, 100, 1000, 1024, 4096, 8192])
@pytest.mark.parametrize("kind", [0, 1, 2])
def test_circulant_operator_matches_dense(spn, torch, n, kind):
    if kind == 1 and n > 4096 or kind != 1 and n & (n - 1) and n > 4096:
        pytest.skip("FFT length > 2^13")
    rng = np.random.default_rng(n * 3 + kind)
    row = rng.standard_normal(n)
    col = rng.standard_normal(n) if kind == 1 else None
    if kind == 1:
        col[0] = row[0]
    spec = spn.CirculantSpec(kind, row, col)
    op = spn.CirculantOperator(spec)
    x = rng.standard_normal((4, n)).astype(np.float32)
    want = x.astype(np.float64) @ dense_circulant(kind, row, col).T
    got = op.apply(torch.from_numpy(x).cuda()).cpu().numpy()
    assert rel(got, want).max() <= RTOL, (n, kind)
    one = op.apply(x[0].astype(np.float64))  # single host vector, fp64 in / out
    assert rel(one[None], want[:1]).max() <= RTOL
    fn = [spn.circulant_matvec, spn.toeplitz_matvec, spn.skew_circulant_matvec][kind]
    assert rel(fn(spec, x[1].astype(np.float64))[None], want[1:2]).max() <= RTOL
    with pytest.raises(spn.DomainError):
        [spn.toeplitz_matvec, spn.skew_circulant_matvec, spn.circulant_matvec][kind](spec, x[0])
