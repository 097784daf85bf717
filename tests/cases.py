"""Seeded parity cases shaped like BASELINE.json's five configs (small slices).

Inputs come from the reference's own generator (Rng = mt19937_64 + Box-Muller,
proj/include/spinners/common.hpp:61-92) through the C oracle, so they are
reproducible bit for bit on any host.  BASELINE's datasets (MNIST-shaped
pixels, unit-sphere vectors) are stood in for by these seeded synthetic rows.
"""
import math

# config 1 — cross-polytope LSH, one table, n=1024, y at scale 1
C1 = dict(n=1024, batch=64, seed_x=1001, table_seed=42)
# config 2 — Gaussian RFF, 784 -> 1024 zero pad, k=4 blocks -> 4096 rows, sigma 5
C2 = dict(n=1024, n_in=784, batch=16, k=4096, sigma=5.0, seed=5, seed_x=2002)
# config 3 — multi-table LSH, n=16384, 8 tables (table t seed = mix_seed(seed, t))
C3 = dict(n=16384, batch=6, tables=8, seed=3, seed_x=3003)
# config 4 — sketch along N=2^17 of A[N][d], m=2048 rows (first-m and random P)
C4 = dict(N=1 << 17, d=4, m=2048, seed=11, seed_x=4004, p_seed=77)
# config 5 — all-Gaussian diagonals + ReLU, scale 1 (fixture at n=2^15; full n=2^20 in gpu tests)
C5 = dict(n=1 << 15, batch=2, seed=13, seed_x=5005, stride=4)


def sqrt(n):
    return math.sqrt(n)
