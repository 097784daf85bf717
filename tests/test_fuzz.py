"""Seeded random-shape fuzzing of the device entry points against the reference itself
(oracle/_ref: the reference's StackedSpinner / CrossPolytopeHasher / embed on the same
fp32 inputs).  Every case draws a variant, n (2..2^16), m, k (stacking), batch, n_in
(ragged zero padding), a row stride and an output stride, then checks apply / hash /
embed.  Bars as in test_gpu_parity.py: 1e-5 relative L2 per vector, ids exact except
near-ties (reference top-two |y| within 1e-5 relative), angular signs exact except
projections within 1e-6 of zero.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RTOL = 1e-5


def row_rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b, axis=-1) / np.maximum(np.linalg.norm(b, axis=-1), 1e-30)


@pytest.fixture(scope="module")
def torch():
    import torch as t
    return t


def draw_case(rng):
    variant = int(rng.choice([0, 1, 2, 3, 4, 5]))
    hi = {0: 16, 1: 16, 2: 13, 3: 12, 4: 13, 5: 10}[variant]
    logn = int(rng.integers(1, hi + 1))
    n = 1 << logn
    if variant == 5 and rng.random() < 0.5:  # the dense baseline takes any n
        n = int(rng.integers(2, 700))
    m = int(rng.integers(1, n + 1))
    k = int(rng.integers(1, 3 * m + 1)) if n <= 4096 else m
    batch = int(rng.integers(1, 7))
    n_in = int(rng.integers(1, n + 1)) if rng.random() < 0.4 else n
    ld = n_in + int(rng.integers(0, 9)) if rng.random() < 0.3 else n_in
    return variant, n, m, k, batch, n_in, ld


@pytest.mark.parametrize("case", range(40))
def test_fuzz_apply_hash_embed(spn, oracle, ref, torch, case):
    rng = np.random.default_rng(1000 + case)
    variant, n, m, k, batch, n_in, ld = draw_case(rng)
    seed = int(rng.integers(0, 2**62))
    V = spn.SpinnerVariant(variant)
    xs = oracle.gaussian_rows(case, batch, ld)
    xs[:, n_in:] = 7.0  # beyond n_in: must be ignored
    xd = torch.from_numpy(xs).cuda()

    # apply (reference StackedSpinner::apply on the zero-padded first n_in entries)
    sp = spn.StackedSpinner(V, n, m, k, seed)
    ldy = k + int(rng.integers(0, 5))
    y = torch.full((batch, ldy), float("nan"), device="cuda")
    sp.plan.apply(xd[:, :n_in], out=y[:, :k])
    y = y[:, :k].cpu().numpy()
    want = ref.apply(variant, n, m, k, seed, 0.0, xs[:, :n_in], n_in=n_in)
    assert row_rel(y, want).max() <= RTOL, (variant, n, m, k, n_in)

    # hash (2 tables, make_hasher_factory(v, n, m)); skip rows that are zero after truncation
    if n_in >= 1 and np.all(np.any(xs[:, :n_in] != 0, axis=1)) and n <= 16384:
        seeds = [spn.mix_seed(seed, t) for t in range(2)]
        h = spn.MultiTableHasher(V, n, m, 2, table_seeds=seeds)
        ids = h.hash_ids(xd[:, :n_in].contiguous()).cpu().numpy()
        want_ids = ref.hash(variant, n, m, seeds, xs[:, :n_in], n_in=n_in)
        for t in range(2):
            yt = ref.apply(variant, n, min(m, n), m, seeds[t], 0.0, xs[:, :n_in], n_in=n_in)
            a = np.sort(np.abs(yt), axis=1)
            gap = (a[:, -1] - a[:, -2]) / np.maximum(a[:, -1], 1e-30) if m > 1 else np.ones(batch)
            bad = ids[:, t] != want_ids[:, t]
            assert np.all(gap[bad] < 1e-5), (variant, n, m, t)

    # embed (gaussian and angular) with d' = k, when the kernels support the size
    if n <= 16384 and k <= 4 * n:
        for kind, sigma in ((0, 0.5 + 3 * rng.random()), (1, 0.0)):
            kk = spn.KernelKind.gaussian(sigma) if kind == 0 else spn.KernelKind.angular()
            sp2 = spn.StackedSpinner(V, n, min(n, k), k, seed + 1)
            got = spn.embed(spn.FeatureMap(sp2, kk), xd[:, :n_in].contiguous()).cpu().numpy()
            want = ref.embed(variant, n, k, seed + 1, kind, sigma, xs[:, :n_in], n_in=n_in)
            if kind == 0:
                assert row_rel(got, want).max() <= RTOL, (variant, n, k)
            else:
                proj = ref.apply(variant, n, min(n, k), k, seed + 1, 0.0, xs[:, :n_in], n_in=n_in)
                scale = np.maximum(np.abs(proj).max(axis=1, keepdims=True), 1e-30)
                flip = got != want
                assert np.all(np.abs(proj[flip]) <= 1e-6 * np.broadcast_to(scale, proj.shape)[flip]), (variant, n)


@pytest.mark.parametrize("case", range(16))
def test_fuzz_multipass_apply(spn, ref, oracle, torch, case):
    """n = 2^15 .. 2^20 (the row/column pass path): random m, stacking, ragged n_in, strides, ReLU."""
    rng = np.random.default_rng(5000 + case)
    logn = int(rng.integers(15, 21))
    n = 1 << logn
    variant = int(rng.choice([0, 1]))
    m = int(rng.integers(1, n + 1)) if rng.random() < 0.5 else n
    k = m if rng.random() < 0.6 else min(2 * m + int(rng.integers(0, 7)), 3 * n)
    batch = int(rng.integers(1, 4))
    n_in = n if rng.random() < 0.5 else int(rng.integers(1, n + 1))
    ld = n_in + (int(rng.integers(1, 9)) if rng.random() < 0.4 else 0)
    relu = bool(rng.random() < 0.3)
    seed = int(rng.integers(0, 2**62))
    xs = oracle.gaussian_rows(7000 + case, batch, ld)
    xd = torch.from_numpy(xs).cuda()
    sp = spn.StackedSpinner(spn.SpinnerVariant(variant), n, m, k, seed)
    y = sp.apply(xd[:, :n_in], relu=relu).cpu().numpy()
    want = ref.apply(variant, n, m, k, seed, 0.0, xs[:, :n_in], n_in=n_in, relu=relu, threads=8)
    assert row_rel(y, want).max() <= RTOL, (variant, n, m, k, n_in, relu)


@pytest.mark.parametrize("case", range(12))
def test_fuzz_sketch(spn, ref, oracle, torch, case):
    """SketchOperator with random (non-pow2) input dims, ragged column counts, first-m and random P."""
    rng = np.random.default_rng(9000 + case)
    N_in = int(rng.integers(2, 1 << int(rng.integers(3, 18))))
    padded = 1 << max(0, (N_in - 1).bit_length())
    d = int(rng.integers(1, 300))
    m = int(rng.integers(1, padded + 1))
    mode = "first" if rng.random() < 0.5 else "random"
    seed = int(rng.integers(0, 2**62))
    a = oracle.gaussian_rows(9100 + case, N_in, d)
    sk = spn.SketchOperator(spn.SpinnerVariant.hd3_hd2_hd1, N_in, m, seed, mode=mode, p_seed=seed + 1)
    got = sk.apply(torch.from_numpy(a).cuda()).cpu().numpy()
    rows = None if mode == "first" else sk.row_list
    want = ref.sketch(0, a, m, seed, row_list=rows, threads=8)
    assert row_rel(got.T, want.T).max() <= RTOL, (N_in, d, m, mode)
