"""Generate the golden fixtures from the REFERENCE ITSELF.

Runs the reference's own code (proj/src/{transforms,spinner,lsh,kernels}.cpp
compiled unmodified into oracle/_ref/libspinners_ref.so; SketchOperator restated
in oracle/ref_api.cpp over the real StackedSpinner) on the seeded cases of
tests/cases.py and writes tests/golden/golden.npz.  Needs /root/reference (this
container), not the GPU box:

    make -C oracle && make -C oracle ref && python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle.oracle import GAUSS3, HD3, HDG, Oracle, Reference  # noqa: E402
import cases  # noqa: E402


def main():
    o, r = Oracle(), Reference()
    g = {}
    # --- generator KATs (common.hpp:51-92)
    for seed in (0, 7, 42, 5489):
        g[f"rng_u64_{seed}"] = r.rng_stream(seed, 16, "u64")
        g[f"rng_uniform_{seed}"] = r.rng_stream(seed, 16, "uniform01")
        g[f"rng_gauss_{seed}"] = r.rng_stream(seed, 17, "gaussian")
        g[f"rng_rad_{seed}"] = r.rng_stream(seed, 16, "rademacher")
    g["mix_seed_in"] = np.array([[0, 0], [42, 0], [42, 1], [2**64 - 1, 5], [123456789, 2**40]], dtype=np.uint64)
    g["mix_seed_out"] = np.array([r.mix_seed(int(a), int(b)) for a, b in g["mix_seed_in"]], dtype=np.uint64)
    # --- transforms (transforms.cpp:52-71)
    for n in (1, 2, 4, 8, 64, 1024, 16384):
        x = o.rng_fill(100 + n, "gaussian", n)
        g[f"fwht_in_{n}"] = x
        g[f"fwht_out_{n}"] = r.fwht(x)
    # --- realised diagonals (spinner.cpp:137-151,248-256)
    for v in (HD3, HDG):
        for (n, m, k, seed) in ((16, 16, 40, 44), (64, 64, 64, 3), (1024, 1024, 4096, 5)):
            d = r.realize(v, n, m, k, seed)
            for i, a in enumerate(d):
                g[f"realize_v{v}_n{n}_k{k}_s{seed}_d{i + 1}"] = a
    # --- config 1: hash ids (scale default) + y at scale 1
    c = cases.C1
    x = o.gaussian_rows(c["seed_x"], c["batch"], c["n"], unit=True)
    g["c1_x"] = x
    g["c1_ids"] = r.hash(HD3, c["n"], c["n"], [c["table_seed"]], x)[:, 0]
    g["c1_y"] = r.apply(HD3, c["n"], c["n"], c["n"], c["table_seed"], 1.0, x)
    # --- config 2: Gaussian RFF features
    c = cases.C2
    x = o.uniform_rows(c["seed_x"], c["batch"], c["n_in"])
    g["c2_x"] = x
    g["c2_feat"] = r.embed(HD3, c["n"], c["k"], c["seed"], 0, c["sigma"], x, n_in=c["n_in"])
    g["c2_ang"] = r.embed(HD3, c["n"], c["k"], c["seed"], 1, 0.0, x, n_in=c["n_in"])
    # --- config 3: 8 tables of ids
    c = cases.C3
    x = o.gaussian_rows(c["seed_x"], c["batch"], c["n"], unit=True)
    seeds = [o.mix_seed(c["seed"], t) for t in range(c["tables"])]
    g["c3_ids"] = r.hash(HD3, c["n"], c["n"], seeds, x, threads=8)
    # --- config 4: sketch (reference first-m; builder random P)
    c = cases.C4
    a = o.gaussian_rows(c["seed_x"], c["N"], c["d"])
    rows = o.sample_rows(c["N"], c["m"], c["p_seed"])
    g["c4_rows"] = rows
    g["c4_first"] = r.sketch(HD3, a, c["m"], c["seed"], threads=4)
    g["c4_random"] = r.sketch(HD3, a, c["m"], c["seed"], row_list=rows, threads=4)
    # --- config 5 (fixture size): all-Gaussian diagonals rounded to fp32, ReLU, scale 1
    c = cases.C5
    d = [a[0].astype(np.float32).astype(np.float64) for a in o.realize(GAUSS3, c["n"], c["n"], c["n"], c["seed"])]
    x = o.gaussian_rows(c["seed_x"], c["batch"], c["n"])
    y = r.chain(d[0], d[1], d[2], 1.0, x, relu=True, threads=2)
    g["c5_y_strided"] = y[:, :: c["stride"]]
    g["c5_y_norm"] = np.linalg.norm(y, axis=1)
    out = os.path.join(HERE, "golden.npz")
    np.savez_compressed(out, **g)
    print(f"wrote {out} ({os.path.getsize(out) / 1e6:.2f} MB, {len(g)} arrays)")


if __name__ == "__main__":
    main()
