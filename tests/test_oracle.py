"""Pin the C oracle (oracle/spinner_oracle.c) before trusting it.

1. Against golden vectors produced by the REFERENCE's own code (oracle/_ref,
   tests/golden/make_golden.py): bit-exact for the generator, the realised
   diagonals and the ids; <= 1e-14 relative for fp64 arithmetic.
2. Against the reference's in-code known-answer tests, restated
   (proj/tests/test_transforms.cpp, test_spinner.cpp, test_lsh.cpp, test_kernels.cpp,
   test_newton.cpp).
"""
import math

import numpy as np
import pytest

import cases
from oracle.oracle import GAUSS3, HD3, HDG

RTOL = 1e-13


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def sylvester(n):
    h = np.array([[1.0]])
    while h.shape[0] < n:
        h = np.block([[h, h], [h, -h]])
    return h / math.sqrt(n)


# ---------------------------------------------------------------- generator
@pytest.mark.parametrize("seed", [0, 7, 42, 5489])
def test_rng_streams_match_reference(oracle, golden, seed):
    assert np.array_equal(oracle.rng_stream(seed, 16, "u64"), golden[f"rng_u64_{seed}"])
    assert np.array_equal(oracle.rng_stream(seed, 16, "uniform01"), golden[f"rng_uniform_{seed}"])
    assert np.array_equal(oracle.rng_stream(seed, 17, "gaussian"), golden[f"rng_gauss_{seed}"])
    assert np.array_equal(oracle.rng_stream(seed, 16, "rademacher"), golden[f"rng_rad_{seed}"])


def test_mt19937_64_standard_value(oracle):
    # C++ [rand.predef]: the 10000th output of a default-constructed mt19937_64.
    assert int(oracle.rng_stream(5489, 10000, "u64")[-1]) == 9981545732273789042


def test_mix_seed(oracle, golden):
    got = [oracle.mix_seed(int(a), int(b)) for a, b in golden["mix_seed_in"]]
    assert np.array_equal(np.array(got, dtype=np.uint64), golden["mix_seed_out"])


@pytest.mark.parametrize("v", [HD3, HDG])
@pytest.mark.parametrize("n,m,k,seed", [(16, 16, 40, 44), (64, 64, 64, 3), (1024, 1024, 4096, 5)])
def test_realised_diagonals_bit_exact(oracle, golden, v, n, m, k, seed):
    d = oracle.realize(v, n, m, k, seed)
    for i in range(3):
        assert np.array_equal(d[i], golden[f"realize_v{v}_n{n}_k{k}_s{seed}_d{i + 1}"])


def test_gauss3_uses_reference_streams(oracle):
    # builder-defined all-Gaussian variant: D1, D2 from the front stream, D3 from the tail
    d1, d2, d3 = oracle.realize(GAUSS3, 64, 64, 64, 9)
    s = oracle.mix_seed(9, 0)
    front = oracle.rng_fill(oracle.mix_seed(s, 1), "gaussian", 128)
    tail = oracle.rng_fill(oracle.mix_seed(s, 2), "gaussian", 64)
    assert np.array_equal(d1[0], front[:64]) and np.array_equal(d2[0], front[64:])
    assert np.array_equal(d3[0], tail)


# ---------------------------------------------------------------- transforms
@pytest.mark.parametrize("n", [1, 2, 4, 8, 64, 1024, 16384])
def test_fwht_matches_reference(oracle, golden, n):
    assert np.array_equal(oracle.fwht(golden[f"fwht_in_{n}"]), golden[f"fwht_out_{n}"])


def test_fwht_kats(oracle):
    # test_transforms.cpp:11-21
    y = oracle.fwht([1.0, 0.0])
    assert abs(y[0] - 1 / math.sqrt(2)) < 1e-15 and abs(y[1] - 1 / math.sqrt(2)) < 1e-15
    x = np.array([1.0, 2.0, 3.0, 4.0])
    assert np.max(np.abs(oracle.fwht(x) - sylvester(4) @ x)) < 1e-12
    # :23-37 involution and norm
    for n in (1, 2, 8, 64, 1024):
        x = oracle.rng_fill(100 + n, "gaussian", n)
        assert np.max(np.abs(oracle.fwht(oracle.fwht(x)) - x)) < 1e-12
        assert abs(np.linalg.norm(oracle.fwht(x)) / np.linalg.norm(x) - 1) < 1e-12


def test_signed_argmax_kats(oracle):
    # test_lsh.cpp:26-35
    assert oracle.signed_argmax([0.1, -0.9, 0.3]) == (1, -1)
    assert oracle.signed_argmax([-2.0, 2.0]) == (0, -1)
    assert oracle.signed_argmax([0.0, 0.0]) == (0, 1)
    assert oracle.signed_argmax([-0.0, 0.0]) == (0, 1)


def test_signed_argmax_matches_reference(oracle, ref):
    rng = np.random.default_rng(0)
    for _ in range(50):
        y = np.round(rng.standard_normal(33), 1)  # rounding creates ties
        assert oracle.signed_argmax(y) == ref.signed_argmax(y)


# ---------------------------------------------------------------- spinner
def test_dense_composition_oracle(oracle):
    # test_spinner.cpp:46-59: sqrt(16) * H D3 H D2 H D1 at n=m=16, seed 21 (block seed 21)
    n = 16
    d1, d2, d3 = (np.zeros(n) for _ in range(3))
    oracle.lib.orc_realize_block(HD3, n, 21, d1, d2, d3)
    h = sylvester(n)
    dense = math.sqrt(n) * h @ np.diag(d3) @ h @ np.diag(d2) @ h @ np.diag(d1)
    for t in range(10):
        x = oracle.rng_fill(300 + t, "gaussian", n)
        y = np.zeros(n)
        oracle.lib.orc_block_apply(n, n, math.sqrt(n), d1, d2, d3, x, y)
        assert np.max(np.abs(y - dense @ x)) < 1e-9


def test_isometry_at_scale_one(oracle):
    # test_spinner.cpp:24-35
    d = oracle.realize(HD3, 64, 64, 64, 3)
    x = oracle.gaussian_rows(100, 20, 64, unit=True)
    y = oracle.apply(*d, 64, 64, 64, 1.0, x)
    assert np.max(np.abs(np.linalg.norm(y, axis=1) - 1)) < 1e-6  # fp32-rounded unit inputs


def test_stacking_blocks_are_independent(oracle):
    # test_spinner.cpp:122-153
    n, m = 16, 8
    d = oracle.realize(HD3, n, m, 2 * m, 33)
    x = oracle.gaussian_rows(1, 1, n)
    y = oracle.apply(*d, n, m, 2 * m, 4.0, x)[0]
    y0 = oracle.apply(d[0][:1], d[1][:1], d[2][:1], n, m, m, 4.0, x)[0]
    y1 = oracle.apply(d[0][1:], d[1][1:], d[2][1:], n, m, m, 4.0, x)[0]
    assert np.array_equal(y[:m], y0) and np.array_equal(y[m:], y1)
    assert np.max(np.abs(y0 - y1)) > 1e-6


# ---------------------------------------------------------------- configs vs reference goldens
def test_config1_matches_reference(oracle, golden):
    c = cases.C1
    d = oracle.realize(HD3, c["n"], c["n"], c["n"], c["table_seed"])
    ids, _ = oracle.hash(*d, c["n"], c["n"], c["n"], 1, math.sqrt(c["n"]), golden["c1_x"])
    assert np.array_equal(ids[:, 0], golden["c1_ids"])
    y = oracle.apply(*d, c["n"], c["n"], c["n"], 1.0, golden["c1_x"])
    assert np.array_equal(y, golden["c1_y"])


def test_config2_matches_reference(oracle, golden):
    c = cases.C2
    d = oracle.realize(HD3, c["n"], c["n"], c["k"], c["seed"])
    f = oracle.embed(*d, c["n"], c["n"], c["k"], math.sqrt(c["n"]), 0, c["sigma"], golden["c2_x"])
    assert rel(f, golden["c2_feat"]) < RTOL
    a = oracle.embed(*d, c["n"], c["n"], c["k"], math.sqrt(c["n"]), 1, 0.0, golden["c2_x"])
    assert np.array_equal(a, golden["c2_ang"])


def test_config3_matches_reference(oracle, golden):
    c = cases.C3
    x = oracle.gaussian_rows(c["seed_x"], c["batch"], c["n"], unit=True)
    for t in range(c["tables"]):
        d = oracle.realize(HD3, c["n"], c["n"], c["n"], oracle.mix_seed(c["seed"], t))
        ids, _ = oracle.hash(*d, c["n"], c["n"], c["n"], 1, math.sqrt(c["n"]), x)
        assert np.array_equal(ids[:, 0], golden["c3_ids"][:, t])


def test_config4_matches_reference(oracle, golden):
    c = cases.C4
    a = oracle.gaussian_rows(c["seed_x"], c["N"], c["d"])
    d = oracle.realize(HD3, c["N"], c["m"], c["m"], c["seed"])
    norm = 1 / math.sqrt(c["m"])
    first = oracle.sketch(*d, c["N"], math.sqrt(c["N"]), norm, a, c["m"])
    assert rel(first, golden["c4_first"]) < RTOL
    rows = oracle.sample_rows(c["N"], c["m"], c["p_seed"])
    assert np.array_equal(rows, golden["c4_rows"])
    rnd = oracle.sketch(*d, c["N"], math.sqrt(c["N"]), norm, a, c["m"], rows=rows)
    assert rel(rnd, golden["c4_random"]) < RTOL


def test_config5_matches_reference(oracle, golden):
    c = cases.C5
    d = [a.astype(np.float32).astype(np.float64) for a in oracle.realize(GAUSS3, c["n"], c["n"], c["n"], c["seed"])]
    x = oracle.gaussian_rows(c["seed_x"], c["batch"], c["n"])
    y = oracle.apply(*d, c["n"], c["n"], c["n"], 1.0, x, relu=True)
    assert rel(y[:, :: c["stride"]], golden["c5_y_strided"]) < RTOL
    assert rel(np.linalg.norm(y, axis=1), golden["c5_y_norm"]) < RTOL


def test_sampler_properties(oracle):
    rows = oracle.sample_rows(1000, 100, 5)
    assert len(set(rows.tolist())) == 100 and rows.min() >= 0 and rows.max() < 1000
    assert np.all(np.diff(rows) > 0)
    assert np.array_equal(oracle.sample_rows(8, 8, 1), np.arange(8))
