"""Batched LSH drivers: collision_curve / compare_families (
reference proj/src/lsh.cpp:38-96, tests restated from proj/tests/test_lsh.cpp:57-190).

The device curve is checked against the reference's own collision_curve (oracle/_ref)
on the same pairs and seeds: bucket counts exactly; collision hits exactly except
(pair, trial) events where either vector is a near-tie for that trial's hasher
(oracle top-two |y| within 1e-5 relative: fp32 vs fp64 argmax), which are counted and
bound the allowed difference.
"""
import math

import numpy as np
import pytest

from oracle.oracle import HD3, HDG

NEAR_TIE = 1e-5


def pairs_at_angle(oracle, n, theta, count, seed):
    """count (x, y) unit pairs at angle theta: y = cos(theta) x + sin(theta) u, u _|_ x."""
    g = oracle.rng_fill(seed, "gaussian", 2 * count * n).reshape(2 * count, n)
    x, u = g[0::2], g[1::2]
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    u -= np.sum(u * x, axis=1, keepdims=True) * x
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    y = math.cos(theta) * x + math.sin(theta) * u
    dist = np.full(count, 2.0 * math.sin(theta / 2.0))
    return x.astype(np.float32), y.astype(np.float32), dist


def spread_pairs(oracle, n, per):
    xs, ys, ds = [], [], []
    for theta in (0.3, 0.8, 1.3, 1.9, 2.5):
        x, y, d = pairs_at_angle(oracle, n, theta, per, int(theta * 997))
        xs.append(x), ys.append(y), ds.append(d)
    return np.concatenate(xs), np.concatenate(ys), np.concatenate(ds)


# ------------------------------------------------------------------------- CPU checks
def test_argument_errors(spn, oracle):
    x, y, d = pairs_at_angle(oracle, 16, 0.5, 4, 1)
    f = spn.make_hasher_factory(spn.SpinnerVariant.hd3_hd2_hd1, 16, 8)
    with pytest.raises(spn.DimensionError):
        spn.collision_curve((x, y, d), f, 0, 1)
    with pytest.raises(spn.DimensionError):
        spn.collision_curve((x, y, d), f, 3, 1, buckets=0)
    with pytest.raises(spn.DomainError):
        spn.collision_curve((x, y, -d), f, 3, 1)
    with pytest.raises(spn.DomainError):
        spn.collision_curve((x, y, d * np.inf), f, 3, 1)


def test_reference_collision_curve_is_bound(ref, oracle):
    """The reference's own driver runs through oracle/_ref (used as the GPU checker below)."""
    x, y, d = pairs_at_angle(oracle, 16, math.pi / 4, 50, 21)
    c = ref.collision_curve(HD3, 16, 8, x, y, d, 4, 5)
    assert c["bucket_edges"].size == 26 and c["bucket_edges"][0] == 0.0
    assert abs(c["bucket_edges"][-1] - 2.0) < 1e-12
    assert int(c["counts"].sum()) == 50 * 4


# ------------------------------------------------------------------------- GPU parity
@pytest.mark.gpu
def test_identical_and_antipodal_pairs(spn, oracle):
    n, m = 16, 8  # test_lsh.cpp:57-78 (HD3 family here; the dense family is out of scope)
    x = oracle.gaussian_rows(100, 20, n, unit=True)
    f = spn.make_hasher_factory(spn.SpinnerVariant.hd3_hd2_hd1, n, m)
    same = spn.collision_curve((x, x, np.zeros(20)), f, 5, 11)
    assert same.counts[0] == 100 and same.probabilities[0] == 1.0
    assert same.counts[1] == 0 and math.isnan(same.probabilities[1])
    anti = spn.collision_curve([spn.HashedPair(x[i], -x[i], 2.0) for i in range(20)], f, 5, 11)
    assert anti.probabilities[24] == 0.0 and anti.counts[24] == 100


@pytest.mark.gpu
def test_bucket_edges_and_scale_invariance(spn, oracle):
    n, m = 16, 8  # test_lsh.cpp:80-105
    x, y, d = pairs_at_angle(oracle, n, math.pi / 4, 50, 21)
    f = spn.make_hasher_factory(spn.SpinnerVariant.hd3_hd2_hd1, n, m)
    c = spn.collision_curve((x, y, d), f, 4, 5)
    assert len(c.bucket_edges) == 26 and c.bucket_edges[0] == 0.0 and abs(c.bucket_edges[-1] - 2.0) < 1e-12
    cs = spn.collision_curve((7.5 * x, 7.5 * y, d), f, 4, 5)
    assert cs.counts == c.counts
    for a, b in zip(c.probabilities, cs.probabilities):
        assert (math.isnan(a) and math.isnan(b)) or a == b


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [HD3, HDG])
def test_curve_matches_reference(spn, oracle, ref, variant):
    n, m, trials, seed = 64, 32, 20, 77  # test_lsh.cpp:173-190 shapes
    x, y, d = spread_pairs(oracle, n, 400)
    f = spn.make_hasher_factory(spn.SpinnerVariant(variant), n, m)
    got = spn.collision_curve((x, y, d), f, trials, seed)
    want = ref.collision_curve(variant, n, m, x, y, d, trials, seed)
    assert np.array_equal(np.array(got.counts), want["counts"].astype(np.int64))
    assert np.allclose(got.bucket_edges, want["bucket_edges"], rtol=0, atol=0)
    # near-tie allowance per bucket: events where x or y is within 1e-5 of an argmax tie
    width = 2.0 / 25
    bucket = np.minimum((d / width).astype(np.int64), 24)
    allow = np.zeros(25, dtype=np.int64)
    for t in range(trials):
        dd = oracle.realize(variant, n, m, m, spn.mix_seed(seed, t))
        _, gx = oracle.hash(*dd, n, m, m, 1, math.sqrt(n), x)
        _, gy = oracle.hash(*dd, n, m, m, 1, math.sqrt(n), y)
        near = (gx[:, 0] < NEAR_TIE) | (gy[:, 0] < NEAR_TIE)
        np.add.at(allow, bucket[near], 1)
    for b in range(25):
        cnt = got.counts[b]
        if cnt == 0:
            assert math.isnan(got.probabilities[b]) and math.isnan(want["probabilities"][b])
            continue
        hits_got = round(got.probabilities[b] * cnt)
        hits_want = round(want["probabilities"][b] * cnt)
        assert abs(hits_got - hits_want) <= allow[b], (b, hits_got, hits_want, allow[b])


@pytest.mark.gpu
def test_compare_families_identical_seeds(spn, oracle):
    n, m = 16, 8  # test_lsh.cpp:140-146
    x, y, d = pairs_at_angle(oracle, n, math.pi / 3, 50, 55)
    f = spn.make_hasher_factory(spn.SpinnerVariant.hd3_hd2_hd1, n, m)
    cmp = spn.compare_families((x, y, d), f, f, 5, 9, 9)
    assert cmp.sup_difference == 0.0


@pytest.mark.gpu
def test_families_within_binomial_noise_and_decreasing(spn, oracle):
    n, m, trials = 64, 32, 10  # test_lsh.cpp:148-190 with the two Hadamard families
    x, y, d = spread_pairs(oracle, n, 400)
    fa = spn.make_hasher_factory(spn.SpinnerVariant.hd3_hd2_hd1, n, m)
    fb = spn.make_hasher_factory(spn.SpinnerVariant.hdg_hd2_hd1, n, m)
    cmp = spn.compare_families((x, y, d), fa, fb, trials, 1001, 2002)
    for b, diff in enumerate(cmp.bucket_differences):
        if math.isnan(diff):
            continue
        events = float(cmp.curve_a.counts[b])
        pa, pb = cmp.curve_a.probabilities[b], cmp.curve_b.probabilities[b]
        pbar = min(0.5, max(pa, pb, 1.0 / events))
        assert diff <= 3.5 * math.sqrt(2.0 * pbar * (1.0 - pbar) / events) + 1e-12
    for curve in (cmp.curve_a, cmp.curve_b):
        prev = 1.03
        for p in curve.probabilities:
            if math.isnan(p):
                continue
            assert p <= prev + 0.03
            prev = p


@pytest.mark.gpu
def test_zero_vector_rejected(spn, oracle):
    x, y, d = pairs_at_angle(oracle, 16, 0.5, 4, 2)
    y[1] = 0.0
    with pytest.raises(spn.DomainError):
        spn.collision_curve((x, y, d), spn.make_hasher_factory(spn.SpinnerVariant.hd3_hd2_hd1, 16, 8), 2, 1)
