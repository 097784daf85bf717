"""GPU parity: the sm_100a kernels (through the C ABI) against the reference's
outputs (golden fixtures made by the reference itself) and the pinned C oracle.

Bars (BASELINE.json north_star):
  * fp32 projections / features: relative L2 error per vector <= 1e-5 (RTOL below);
  * bucket ids and subsample indices: bit-exact except documented near-ties
    (oracle top-two |y| within 1e-5 relative, NEAR_TIE below).
"""
import math

import numpy as np
import pytest

import cases
from oracle.oracle import GAUSS3, HD3, HDG

pytestmark = pytest.mark.gpu

RTOL = 1e-5
NEAR_TIE = 1e-5


@pytest.fixture(scope="module")
def torch():
    import torch as t
    return t


def dev(torch, x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def row_rel(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    num = np.linalg.norm(got - want, axis=-1)
    den = np.maximum(np.linalg.norm(want, axis=-1), 1e-30)
    return num / den


def assert_ids(got, want, gaps):
    got, want, gaps = np.asarray(got), np.asarray(want), np.asarray(gaps)
    bad = (got != want) & ~(gaps < NEAR_TIE)
    assert not bad.any(), f"{bad.sum()} id mismatches outside near-ties (of {got.size})"


# ------------------------------------------------------------------ configs
def test_config1_hash_and_projection(spn, oracle, golden, torch):
    c = cases.C1
    sp = spn.StackedSpinner(spn.SpinnerVariant.hd3_hd2_hd1, c["n"], c["n"], c["n"], c["table_seed"], scale=1.0)
    x = dev(torch, golden["c1_x"])
    y = torch.empty((c["batch"], c["n"]), device="cuda")
    ids = sp.plan.hash(x, y_out=y)
    torch.cuda.synchronize()
    assert row_rel(y.cpu().numpy(), golden["c1_y"]).max() <= RTOL
    d = oracle.realize(HD3, c["n"], c["n"], c["n"], c["table_seed"])
    _, gaps = oracle.hash(*d, c["n"], c["n"], c["n"], 1, 1.0, golden["c1_x"])
    assert_ids(ids.cpu().numpy()[:, 0], golden["c1_ids"], gaps[:, 0])
    # the default-scale hasher (make_hasher_factory) gives the same ids
    h = spn.make_hasher_factory(spn.SpinnerVariant.hd3_hd2_hd1, c["n"], c["n"])(c["table_seed"])
    assert_ids(h.projector.plan.hash(x).cpu().numpy()[:, 0], golden["c1_ids"], gaps[:, 0])


def test_config1_permuted_and_general_kernels_agree_with_reference(spn, oracle, golden, torch):
    """16-B aligned rows take the permuted-coordinate n = 1024 hash + y kernel (OP_APPLY_P: 16-B x loads and
    y stores, host-permuted sign masks); rows at a 4-B offset take the general kernel.  Both match the
    reference: ids bit-exact except near-ties, y within RTOL, and the two agree to RTOL."""
    c = cases.C1
    sp = spn.StackedSpinner(spn.SpinnerVariant.hd3_hd2_hd1, c["n"], c["n"], c["n"], c["table_seed"], scale=1.0)
    xs = golden["c1_x"]
    d = oracle.realize(HD3, c["n"], c["n"], c["n"], c["table_seed"])
    _, gaps = oracle.hash(*d, c["n"], c["n"], c["n"], 1, 1.0, xs)
    b = xs.shape[0]
    xa = dev(torch, xs)                                                   # aligned: permuted kernel
    buf = torch.zeros(b * c["n"] + 1, device="cuda")
    buf[1:] = xa.reshape(-1)
    xu = buf[1:].view(b, c["n"])                                          # 4-B offset: general kernel
    ya = torch.empty((b, c["n"]), device="cuda")
    ybuf = torch.empty(b * c["n"] + 1, device="cuda")
    yu = ybuf[1:].view(b, c["n"])
    ida = sp.plan.hash(xa, y_out=ya).cpu().numpy()[:, 0]
    idu = sp.plan.hash(xu, y_out=yu).cpu().numpy()[:, 0]
    torch.cuda.synchronize()
    for ids, y in ((ida, ya), (idu, yu)):
        assert_ids(ids, golden["c1_ids"], gaps[:, 0])
        assert row_rel(y.cpu().numpy(), golden["c1_y"]).max() <= RTOL
    assert row_rel(ya.cpu().numpy(), yu.cpu().numpy()).max() <= RTOL


def test_config2_random_features(spn, golden, torch):
    c = cases.C2
    sp = spn.StackedSpinner(spn.SpinnerVariant.hd3_hd2_hd1, c["n"], min(c["n"], c["k"]), c["k"], c["seed"])
    fm = spn.FeatureMap(sp, spn.KernelKind.gaussian(c["sigma"]))
    x = dev(torch, golden["c2_x"])
    f = spn.embed(fm, x).cpu().numpy()
    assert f.shape == golden["c2_feat"].shape
    assert row_rel(f, golden["c2_feat"]).max() <= RTOL
    # angular kernel: signs agree except where the projection is ~0
    fa = spn.embed(spn.FeatureMap(sp, spn.KernelKind.angular()), x).cpu().numpy()
    assert (fa != golden["c2_ang"]).mean() < 1e-3


def test_config2_unaligned_output_uses_general_kernel(spn, golden, torch):
    """ld_out not a multiple of 4 -> the non-permuted (4-B store) kernel; same results."""
    c = cases.C2
    sp = spn.StackedSpinner(spn.SpinnerVariant.hd3_hd2_hd1, c["n"], min(c["n"], c["k"]), c["k"], c["seed"])
    fm = spn.FeatureMap(sp, spn.KernelKind.gaussian(c["sigma"]))
    x = dev(torch, golden["c2_x"])
    buf = torch.zeros((x.shape[0], 2 * c["k"] + 1), device="cuda")
    f = spn.embed(fm, x, out=buf[:, 1:]).cpu().numpy()
    assert row_rel(f, golden["c2_feat"]).max() <= RTOL
    assert float(buf[:, 0].abs().max()) == 0.0  # nothing written outside the view


def test_config3_multitable_hash(spn, oracle, golden, torch):
    c = cases.C3
    h = spn.MultiTableHasher(spn.SpinnerVariant.hd3_hd2_hd1, c["n"], c["n"], c["tables"], seed=c["seed"])
    x = oracle.gaussian_rows(c["seed_x"], c["batch"], c["n"], unit=True)
    ids = h.hash_ids(dev(torch, x)).cpu().numpy()
    gaps = np.zeros_like(ids, dtype=np.float64)
    for t in range(c["tables"]):
        d = oracle.realize(HD3, c["n"], c["n"], c["n"], h.table_seeds[t])
        _, g = oracle.hash(*d, c["n"], c["n"], c["n"], 1, 1.0, x)
        gaps[:, t] = g[:, 0]
    assert_ids(ids, golden["c3_ids"], gaps)


@pytest.mark.parametrize("mode", ["first", "random"])
def test_config4_sketch(spn, oracle, golden, torch, mode):
    c = cases.C4
    sk = spn.SketchOperator(spn.SpinnerVariant.hd3_hd2_hd1, c["N"], c["m"], c["seed"], mode=mode,
                            p_seed=c["p_seed"])
    a = oracle.gaussian_rows(c["seed_x"], c["N"], c["d"])
    out = sk.apply(dev(torch, a)).cpu().numpy()
    want = golden["c4_first"] if mode == "first" else golden["c4_random"]
    if mode == "random":
        assert np.array_equal(sk.row_list, golden["c4_rows"])
    assert row_rel(out.T, want.T).max() <= RTOL


def test_config5_fixture(spn, oracle, golden, torch):
    c = cases.C5
    d = [a.astype(np.float32).astype(np.float64) for a in oracle.realize(GAUSS3, c["n"], c["n"], c["n"], c["seed"])]
    sp = spn.StackedSpinner.from_diagonals(*d, c["n"], c["n"], c["n"], scale=1.0)
    x = oracle.gaussian_rows(c["seed_x"], c["batch"], c["n"])
    y = sp.apply(dev(torch, x), relu=True).cpu().numpy()
    assert row_rel(y[:, :: c["stride"]], golden["c5_y_strided"]).max() <= RTOL
    assert np.max(np.abs(np.linalg.norm(y, axis=1) / golden["c5_y_norm"] - 1)) <= RTOL


def test_config5_full_size(spn, oracle, torch):
    n = 1 << 20
    sp = spn.StackedSpinner(spn.SpinnerVariant.gauss3, n, n, n, 13, scale=1.0)
    d1, d2, d3 = (a.astype(np.float32).astype(np.float64) for a in sp.diagonals())
    x = oracle.gaussian_rows(5005, 2, n)
    y = sp.apply(dev(torch, x), relu=True).cpu().numpy()
    want = oracle.apply(d1[None], d2[None], d3[None], n, n, n, 1.0, x, relu=True)
    assert row_rel(y, want).max() <= RTOL


# ------------------------------------------------------------------ sweeps
LOGNS = list(range(1, 15))


@pytest.mark.parametrize("logn", LOGNS)
@pytest.mark.parametrize("variant", [HD3, HDG, GAUSS3])
def test_apply_sweep(spn, oracle, torch, logn, variant):
    n = 1 << logn
    for m, k in [(n, n), (max(1, n // 2 + 1), 2 * max(1, n // 2 + 1) + 3)]:
        sp = spn.StackedSpinner(variant, n, m, k, 1000 + logn)
        d = tuple(a.astype(np.float32).astype(np.float64) for a in sp.plan.diagonals())
        d = tuple(a[0] for a in d)
        x = oracle.gaussian_rows(logn, 9, n)
        y = sp.apply(dev(torch, x)).cpu().numpy()
        want = oracle.apply(*d, n, m, k, math.sqrt(n), x)
        assert y.shape == (9, k)
        assert row_rel(y, want).max() <= RTOL, (n, m, k)


@pytest.mark.parametrize("logn", LOGNS)
def test_hash_sweep(spn, oracle, torch, logn):
    n = 1 << logn
    for m in sorted({n, max(1, n // 3)}):
        seeds = [spn.mix_seed(7, t) for t in range(3)]
        h = spn.MultiTableHasher(spn.SpinnerVariant.hd3_hd2_hd1, n, m, 3, table_seeds=seeds)
        x = oracle.gaussian_rows(50 + logn, 33, n, unit=True)
        ids = h.hash_ids(dev(torch, x)).cpu().numpy()
        for t in range(3):
            d = oracle.realize(HD3, n, m, m, seeds[t])
            want, gaps = oracle.hash(*d, n, m, m, 1, math.sqrt(n), x)
            assert_ids(ids[:, t], want[:, 0], gaps[:, 0])


@pytest.mark.parametrize("logn", [2, 5, 8, 10, 11, 12, 13, 14])
def test_embed_sweep(spn, oracle, torch, logn):
    n = 1 << logn
    k = 2 * n + n // 2
    sp = spn.StackedSpinner(spn.SpinnerVariant.hd3_hd2_hd1, n, n, k, 3 + logn)
    d = sp.plan.diagonals()
    d = tuple(a[0] for a in d)
    n_in = max(1, (3 * n) // 4)
    x = oracle.uniform_rows(logn, 7, n_in)
    f = spn.embed(spn.FeatureMap(sp, spn.KernelKind.gaussian(2.5)), dev(torch, x)).cpu().numpy()
    want = oracle.embed(*d, n, n, k, math.sqrt(n), 0, 2.5, x, n_in=n_in)
    assert row_rel(f, want).max() <= RTOL


@pytest.mark.parametrize("logn", [15, 16, 17, 18, 20])
@pytest.mark.parametrize("variant", [HD3, GAUSS3])
def test_big_apply_sweep(spn, oracle, torch, logn, variant):
    n = 1 << logn
    for m, k in [(n, n), (n // 2 + 1, n + 2)]:
        sp = spn.StackedSpinner(variant, n, m, k, 77 + logn)
        d = tuple(a[0].astype(np.float32).astype(np.float64) for a in sp.plan.diagonals())
        n_in = n - 5
        x = oracle.gaussian_rows(logn, 2, n_in)
        y = sp.apply(dev(torch, x), relu=(m == n)).cpu().numpy()
        want = oracle.apply(*d, n, m, k, math.sqrt(n), x, n_in=n_in, relu=(m == n))
        assert row_rel(y, want).max() <= RTOL, (n, m, k)


@pytest.mark.parametrize("N_in,d,m", [(8, 1, 8), (1000, 33, 100), (1024, 64, 1024), (1 << 11, 5, 300),
                                      (1 << 13, 40, 512), (70000, 3, 2048)])
@pytest.mark.parametrize("mode", ["first", "random"])
def test_sketch_sweep(spn, oracle, torch, N_in, d, m, mode):
    sk = spn.SketchOperator(spn.SpinnerVariant.hd3_hd2_hd1, N_in, m, 19, mode=mode, p_seed=3)
    a = oracle.gaussian_rows(N_in + d, N_in, d)
    out = sk.apply(dev(torch, a)).cpu().numpy()
    D = tuple(x[0] for x in sk.plan.diagonals())
    want = oracle.sketch(*D, sk.padded, math.sqrt(sk.padded), sk.norm, a, m, rows=sk.row_list)
    assert out.shape == (m, d)
    assert row_rel(out.T, want.T).max() <= RTOL


# ------------------------------------------------------------------ properties & edges
def test_full_size_isometry_and_hash_invariances(spn, oracle, torch):
    n = 16384
    sp = spn.StackedSpinner(spn.SpinnerVariant.hd3_hd2_hd1, n, n, n, 5, scale=1.0)
    x = oracle.gaussian_rows(9, 64, n)
    xt = dev(torch, x)
    y = sp.apply(xt).cpu().numpy()
    assert np.max(np.abs(np.linalg.norm(y, axis=1) / np.linalg.norm(x, axis=1) - 1)) < 1e-5
    ids = sp.plan.hash(xt).cpu().numpy()[:, 0]
    assert np.array_equal(sp.plan.hash(xt * 3.0).cpu().numpy()[:, 0], ids)  # positive scale invariance
    neg = sp.plan.hash(-xt).cpu().numpy()[:, 0]
    assert np.array_equal(neg % n, ids % n) and np.all((neg >= n) != (ids >= n))  # antisymmetry


def test_zero_vector_and_ties(spn, torch):
    sp = spn.StackedSpinner(spn.SpinnerVariant.hd3_hd2_hd1, 64, 64, 64, 1)
    ids = sp.plan.hash(torch.zeros((3, 64), device="cuda")).cpu().numpy()
    assert np.all(ids == 0)  # signed_argmax of all zeros: index 0, sign +1 (lsh.cpp:20)
    with pytest.raises(spn.DomainError):
        spn.CrossPolytopeHasher(sp).hash(np.zeros(64, np.float32))  # hash() rejects zero (lsh.cpp:25-28)
    # identity-like case: x = e_0 through an all-(+1) explicit spinner gives a flat |y| -> smallest index
    n = 16
    ones = np.ones(n)
    spi = spn.StackedSpinner.from_diagonals(ones, ones, ones, n, n, n)
    x = np.zeros((1, n), np.float32)
    x[0, 0] = 1.0
    # H H H e0 = H e0 = all entries 1/sqrt(n): every |y_i| ties -> index 0, sign +
    assert int(spi.plan.hash(dev(torch, x)).cpu().numpy()[0, 0]) == 0


def test_batch_zero_strided_and_host_paths(spn, oracle, torch):
    n = 1024
    sp = spn.StackedSpinner(spn.SpinnerVariant.hd3_hd2_hd1, n, n, 3 * n, 4)
    empty = torch.empty((0, n), device="cuda")
    assert sp.apply(empty).shape == (0, 3 * n)
    big = dev(torch, oracle.gaussian_rows(1, 10, 2 * n))
    strided = big[:, 100:100 + n]  # ld_x = 2n
    y1 = sp.apply(strided).cpu().numpy()
    y2 = sp.apply(strided.contiguous()).cpu().numpy()
    assert np.array_equal(y1, y2)
    # host entry points (e2e path) are bit-identical to the device path
    xh = oracle.uniform_rows(3, 300, 784)
    fm = spn.FeatureMap(sp, spn.KernelKind.gaussian(5.0))
    f_dev = spn.embed(fm, dev(torch, xh)).cpu().numpy()
    f_host = spn.embed(fm, xh)
    assert np.array_equal(f_dev, f_host)
    assert np.array_equal(sp.apply(xh), sp.apply(dev(torch, xh)).cpu().numpy())
    assert np.array_equal(sp.plan.hash(xh), sp.plan.hash(dev(torch, xh)).cpu().numpy())


def test_single_vector_api_matches_reference(spn, oracle, golden):
    c = cases.C1
    h = spn.make_hasher_factory(spn.SpinnerVariant.hd3_hd2_hd1, c["n"], c["n"])(c["table_seed"])
    d = oracle.realize(HD3, c["n"], c["n"], c["n"], c["table_seed"])
    _, gaps = oracle.hash(*d, c["n"], c["n"], c["n"], 1, 1.0, golden["c1_x"][:8])
    for i in range(8):
        idx, sg = h.hash(golden["c1_x"][i])
        want = int(golden["c1_ids"][i])
        if gaps[i, 0] >= NEAR_TIE:
            assert (idx + (c["n"] if sg < 0 else 0)) == want


def test_check_rows(spn, torch):
    x = torch.ones((4, 100), device="cuda")
    x[1].zero_()
    x[2, 5] = float("nan")
    assert spn.check_rows(x).cpu().tolist() == [0, 2, 1, 0]


def test_structured_spinner_build_uses_spec_seed(spn, oracle, torch):
    spec = spn.SpinnerSpec.make(spn.SpinnerVariant.hd3_hd2_hd1, 16, 16, 21)
    sp = spn.StructuredSpinner.build(spec)
    d = oracle.realize_block(HD3, 16, 21)
    h = np.array([[1.0]])
    while h.shape[0] < 16:
        h = np.block([[h, h], [h, -h]])
    h /= 4.0
    dense = 4.0 * h @ np.diag(d[2]) @ h @ np.diag(d[1]) @ h @ np.diag(d[0])
    x = oracle.gaussian_rows(300, 10, 16)
    y = sp.apply(dev(torch, x)).cpu().numpy()
    assert np.max(np.abs(y - x.astype(np.float64) @ dense.T)) < 1e-5


@pytest.mark.parametrize("logn", [19, 20])
def test_big_inplace_groups(spn, oracle, torch, logn):
    """In-place 4-pass schedule over several L2 groups on alternating streams (config-5 shape)."""
    n = 1 << logn
    sp = spn.StackedSpinner(spn.SpinnerVariant.gauss3, n, n, n, 31 + logn, scale=1.0)
    d = tuple(a[0].astype(np.float32).astype(np.float64) for a in sp.plan.diagonals())
    x = oracle.gaussian_rows(logn + 100, 19, n)  # more vectors than one 32 MB group
    y = sp.apply(dev(torch, x), relu=True).cpu().numpy()
    want = oracle.apply(*d, n, n, n, 1.0, x, relu=True)
    assert row_rel(y, want).max() <= RTOL


# ------------------------------------------- device realisation of Rademacher sketch plans
@pytest.mark.parametrize("N", [1 << 15, 1 << 17, 1 << 20])
def test_sketch_device_realisation_bit_exact(spn, oracle, torch, N):
    """Single-block HD3 plans with N > 2^14 (SketchOperator) draw D1..D3 on the device with the
    reference's mt19937_64 (mt_rademacher_sketch_kernel).  The sketch must equal, bit for bit,
    the same sketch through an explicit plan carrying the C oracle's host realisation, and the
    lazily host-drawn diagonals of the plan must equal the oracle's."""
    m, d, seed = 256, 32, 23
    sk = spn.SketchOperator(spn.SpinnerVariant.hd3_hd2_hd1, N, m, seed)
    a = dev(torch, oracle.gaussian_rows(77, N, d))
    out = sk.apply(a).cpu().numpy()
    D = oracle.realize(HD3, N, m, m, seed)
    ex = spn.StackedSpinner.from_diagonals(D[0][0], D[1][0], D[2][0], N, m, m)
    want = ex.plan.sketch(a, m, sk.norm).cpu().numpy()
    assert np.array_equal(out, want)
    got_d = sk.plan.diagonals()
    for g, w in zip(got_d, D):
        assert np.array_equal(g.reshape(-1), w.reshape(-1))


def test_lazy_plan_apply_and_side_stream(spn, oracle, torch):
    """A lazily realised plan used through apply (host draws on demand) and a device-realised
    sketch made on a side stream then reused on the default stream."""
    N, seed = 1 << 16, 31
    sp = spn.StackedSpinner(spn.SpinnerVariant.hd3_hd2_hd1, N, N, N, seed)
    x = dev(torch, oracle.gaussian_rows(5, 3, N))
    D = oracle.realize(HD3, N, N, N, seed)
    ex = spn.StackedSpinner.from_diagonals(D[0][0], D[1][0], D[2][0], N, N, N)
    assert np.array_equal(sp.apply(x).cpu().numpy(), ex.apply(x).cpu().numpy())
    sk = spn.SketchOperator(spn.SpinnerVariant.hd3_hd2_hd1, N, 512, seed)
    a = dev(torch, oracle.gaussian_rows(6, N, 64))
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        o1 = sk.apply(a, stream=side)
    o2 = sk.apply(a)
    torch.cuda.synchronize()
    want = ex.plan.sketch(a, 512, sk.norm)
    assert torch.equal(o1, want) and torch.equal(o2, want)
    del sk  # pool memory goes back after the uses recorded on both streams
    torch.cuda.synchronize()


def test_plan_destroyed_while_in_flight(spn, oracle, torch):
    """Dropping a sketch plan right after an asynchronous call returns its pooled memory only after
    that call (stream-ordered free after the recorded use): a plan created next, reusing the pool,
    must not disturb the first result."""
    N, m = 1 << 17, 512
    a = dev(torch, oracle.gaussian_rows(12, N, 64))
    ref1 = spn.SketchOperator(spn.SpinnerVariant.hd3_hd2_hd1, N, m, 101).apply(a).clone()
    ref2 = spn.SketchOperator(spn.SpinnerVariant.hd3_hd2_hd1, N, m, 202).apply(a).clone()
    torch.cuda.synchronize()
    for _ in range(3):
        torch.cuda._sleep(50_000_000)  # keep the device busy so the calls below are still queued
        sk1 = spn.SketchOperator(spn.SpinnerVariant.hd3_hd2_hd1, N, m, 101)
        out1 = sk1.apply(a)
        del sk1
        sk2 = spn.SketchOperator(spn.SpinnerVariant.hd3_hd2_hd1, N, m, 202)
        out2 = sk2.apply(a)
        del sk2
        torch.cuda.synchronize()
        assert torch.equal(out1, ref1) and torch.equal(out2, ref2)


# ---------------------------------------------- hash / embed beyond the fused sizes (n > 2^14)
@pytest.mark.parametrize("logn", [15, 16, 18])
def test_big_hash_multitable(spn, oracle, torch, logn):
    """CrossPolytopeHasher::hash at n > 2^14 (multi-pass projection + row argmax), three tables,
    full and truncated tables, against the oracle (lsh.cpp:9-30)."""
    n = 1 << logn
    for m in (n, n // 2 + 3):
        seeds = [spn.mix_seed(9 + logn, t) for t in range(3)]
        h = spn.MultiTableHasher(spn.SpinnerVariant.hd3_hd2_hd1, n, m, 3, table_seeds=seeds)
        x = oracle.gaussian_rows(logn + m, 5, n, unit=True)
        ids = h.hash_ids(dev(torch, x)).cpu().numpy()
        assert ids.shape == (5, 3)
        for t in range(3):
            d = oracle.realize(HD3, n, m, m, seeds[t])
            want, gaps = oracle.hash(*d, n, m, m, 1, math.sqrt(n), x)
            assert_ids(ids[:, t], want[:, 0], gaps[:, 0])


def test_big_hash_with_projection(spn, oracle, torch):
    n = 1 << 15
    sp = spn.StackedSpinner(spn.SpinnerVariant.hd3_hd2_hd1, n, n, n, 44, scale=1.0)
    x = oracle.gaussian_rows(3, 4, n, unit=True)
    y = torch.empty((4, n), device="cuda")
    ids = sp.plan.hash(dev(torch, x), y_out=y).cpu().numpy()[:, 0]
    d = oracle.realize(HD3, n, n, n, 44)
    assert row_rel(y.cpu().numpy(), oracle.apply(*d, n, n, n, 1.0, x)).max() <= RTOL
    want, gaps = oracle.hash(*d, n, n, n, 1, 1.0, x)
    assert_ids(ids, want[:, 0], gaps[:, 0])


@pytest.mark.parametrize("logn", [15, 17])
@pytest.mark.parametrize("kind", ["gaussian", "angular"])
def test_big_embed(spn, oracle, torch, logn, kind):
    """embed (kernels.cpp:17-36) at n > 2^14, stacked k > m with a truncated last block, ragged n_in."""
    n = 1 << logn
    k = n + n // 2 + 5
    sp = spn.StackedSpinner(spn.SpinnerVariant.hd3_hd2_hd1, n, n, k, 5 + logn)
    kk = spn.KernelKind.gaussian(3.0) if kind == "gaussian" else spn.KernelKind.angular()
    n_in = n - 77
    # rows of norm 20 (angles |z / sigma| of a few units): the fp32 projection's absolute angle error
    # grows with |z|, so uniform [0, 1] rows of this length (|z| ~ sqrt(n / 3) ~ 200) would sit at the
    # fp32 floor of the 1e-5 bar whatever the kernel (the reference is fp64)
    x = 20.0 * oracle.gaussian_rows(logn, 3, n_in, unit=True)
    f = spn.embed(spn.FeatureMap(sp, kk), dev(torch, x)).cpu().numpy()
    d = tuple(a[0] for a in sp.plan.diagonals())
    want = oracle.embed(*d, n, n, k, math.sqrt(n), 0 if kind == "gaussian" else 1, 3.0, x, n_in=n_in)
    if kind == "gaussian":
        assert row_rel(f, want).max() <= RTOL
    else:  # signs: exact except where |z| is at rounding level
        assert np.mean(f == want) > 0.9999


@pytest.mark.parametrize("variant", ["hd3_hd2_hd1", "hdg_hd2_hd1", "gcirc_d2_hd1", "gtoeplitz_d2_hd1",
                                     "gskew_circ_d2_hd1", "gaussian_dense"])
def test_structured_spinner_build_all_variants(spn, oracle, torch, variant):
    """StructuredSpinner::build(spec) draws block 0 from spec.seed itself (spinner.cpp:137-151) for
    every variant: it must equal, bit for bit, the stacked plan whose block 0 spec seed is
    mix_seed(S, 0) (spinner.cpp:255); apply_front_blocks (spinner.cpp:186-198) against the
    diagonals composed in fp64."""
    v = getattr(spn.SpinnerVariant, variant)
    n, m, S = 64, 48, 1234
    spec = spn.SpinnerSpec.make(v, n, m, spn.mix_seed(S, 0))
    sp = spn.StructuredSpinner.build(spec)
    stacked = spn.StackedSpinner(v, n, m, m, S)
    x = oracle.gaussian_rows(77, 6, n)
    a = sp.apply(dev(torch, x)).cpu().numpy()
    b = stacked.apply(dev(torch, x)).cpu().numpy()
    assert a.shape == (6, m) and np.array_equal(a, b)
    if variant == "gaussian_dense":
        with pytest.raises(spn.DomainError):
            sp.apply_front_blocks(x[0])
        return
    d1, d2, _ = (t[0, 0] for t in sp.plan.diagonals())
    d1, d2 = (t.astype(np.float32).astype(np.float64) for t in (d1, d2))
    xd = x.astype(np.float64)
    front = np.stack([oracle.fwht(r * d1) * d2 for r in xd])
    if variant in ("hd3_hd2_hd1", "hdg_hd2_hd1"):
        front = np.stack([oracle.fwht(r) for r in front])
    got = sp.apply_front_blocks(dev(torch, x)).cpu().numpy()
    assert row_rel(got, front).max() <= RTOL
    assert row_rel(sp.apply_front_blocks(xd[0])[None], front[:1]).max() <= RTOL


def test_big_hash_stacked_blocks(spn, oracle, torch):
    """signed argmax over the k rows of a stacked (k > m) plan at n > 2^14, truncated last block."""
    n = 1 << 15
    k = n + n // 2 + 7
    sp = spn.StackedSpinner(spn.SpinnerVariant.hd3_hd2_hd1, n, n, k, 61)
    x = oracle.gaussian_rows(8, 4, n, unit=True)
    ids = sp.plan.hash(dev(torch, x)).cpu().numpy()[:, 0]
    d = tuple(a[0] for a in sp.plan.diagonals())
    want, gaps = oracle.hash(*d, n, n, k, 1, math.sqrt(n), x)
    assert_ids(ids, want[:, 0], gaps[:, 0])


def test_concurrent_host_and_stream_calls(spn, oracle, torch):
    """Plans are immutable and reentrant (spinner.hpp:55): host-buffer calls from several
    threads on one plan (serialised per plan) and device calls on several streams give the same bits
    as one call."""
    import concurrent.futures
    n, k = 1024, 2048
    sp = spn.StackedSpinner(spn.SpinnerVariant.hd3_hd2_hd1, n, n, k, 17)
    fm = spn.FeatureMap(sp, spn.KernelKind.gaussian(4.0))
    xs = [oracle.uniform_rows(100 + i, 300, n) for i in range(6)]
    want = [spn.embed(fm, dev(torch, x)).cpu().numpy() for x in xs]
    with concurrent.futures.ThreadPoolExecutor(6) as ex:
        got = list(ex.map(lambda x: spn.embed(fm, x), xs))  # host arrays -> spn_embed_f32_host
    for g, w in zip(got, want):
        assert np.array_equal(g, w)
    streams = [torch.cuda.Stream() for _ in range(3)]
    xd = [dev(torch, x) for x in xs[:3]]
    torch.cuda.synchronize()
    outs = []
    for s, x in zip(streams, xd):
        with torch.cuda.stream(s):
            outs.append(spn.embed(fm, x, stream=s))
    torch.cuda.synchronize()
    for o, w in zip(outs, want[:3]):
        assert np.array_equal(o.cpu().numpy(), w)
