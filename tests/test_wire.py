"""The reference CLI's result-table wire format (proj/tools/spinners_cli.cpp:26-51,165-176): the
``# {json}`` echo line and ``%.17g`` numbers, pinned against lines produced by nlohmann::json and
snprintf themselves (tests/golden/make_wire_golden.cpp -> tests/golden/wire_golden.txt)."""
import io
import math
import os
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import ROOT

GOLDEN = os.path.join(ROOT, "tests", "golden", "wire_golden.txt")


@pytest.fixture(scope="module")
def wire():
    import importlib.util
    spec = importlib.util.spec_from_file_location("wire", os.path.join(ROOT, "paper_1610_06209_b200", "wire.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


@pytest.fixture(scope="module")
def golden_lines():
    return open(GOLDEN).read().splitlines()


def test_fmt17_matches_snprintf(wire, golden_lines):
    vals = [0.0, -0.0, 1.0, 0.1, 2.0 / 3.0, 1e-300, 6.02214076e23, -1.5, 0.08, float("nan"), float("inf"), 0.5,
            1e21, 123456789.125]
    want = [ln[2:] for ln in golden_lines if ln.startswith("f ")]
    assert [wire.fmt17(v) for v in vals] == want


def test_echo_lines_match_nlohmann(wire, golden_lines):
    echoes = [ln for ln in golden_lines if ln.startswith("# ")]
    cfgs = [
        ("lsh-collision", {"variant": "HD3HD2HD1", "n": 256, "rows": 64, "pairs": 20000, "trials": 100, "seed": 42}),
        ("lsh-compare", {"a": "HD3HD2HD1", "b": "GaussianDense", "n": 64, "rows": 64, "pairs": 500, "trials": 50,
                         "seed": 42}),
        ("newton-sketch", {"sketch": "HD3HD2HD1", "rows": 1024, "n": 8192, "d": 64, "iters": 30,
                           "gap_tolerance": 1e-10, "line_search": True, "seed": 42}),
        ("kernel-approx", {"variant": "HD3HD2HD1", "kernel": "gaussian", "sigma": 2.5, "features": [64, 128, 256],
                           "seeds": 3, "seed": 42, "dataset": {"data": "", "label_column": -1, "pad": False,
                                                               "synth_dim": 64, "synth_count": 200}}),
    ]
    for (cmd, cfg), want in zip(cfgs, echoes):
        buf = io.StringIO()
        wire.emit_config(buf, cmd, cfg)
        assert buf.getvalue() == want + "\n"


def test_curve_table_round_trip(wire):
    curve = SimpleNamespace(bucket_edges=[0.0, 0.08, 0.16, 0.24], probabilities=[1.0, float("nan"), 0.1],
                            counts=[300, 0, 7])
    other = SimpleNamespace(bucket_edges=curve.bucket_edges, probabilities=[0.9, float("nan"), 0.2],
                            counts=curve.counts)
    cmp = SimpleNamespace(curve_a=curve, curve_b=other, bucket_differences=[0.1, float("nan"), 0.1],
                          sup_difference=0.1)
    text = wire.to_string(wire.write_lsh_compare, {"n": 8}, cmp)
    lines = text.splitlines()
    assert lines[1] == "# sup_difference 0.10000000000000001"
    assert lines[2] == "bucket_low,bucket_high,count,prob_a,prob_b,abs_diff"
    assert lines[3] == "0,0.080000000000000002,300,1,0.90000000000000002,0.10000000000000001"
    assert lines[4].split(",")[3] == "nan"
    echo, comments, header, rows = wire.read_table(text)
    assert echo == {"command": "lsh-compare", "config": {"n": 8}, "library": "spinners 1.0"}
    assert comments == ["sup_difference 0.10000000000000001"]
    assert rows[2] == [0.16, 0.24, 7, 0.1, 0.2, 0.1]
    assert math.isnan(rows[1][3])


def test_newton_and_kernel_tables(wire):
    tr = SimpleNamespace(losses=[0.5, 0.25], gaps=[1e-3, 0.0], seconds=[0.001, 0.002])
    text = wire.to_string(wire.write_newton_sketch, {"d": 4}, tr)
    assert text.splitlines()[1:] == ["iter,loss,gap,seconds", "0,0.5,0.001,0.001",
                                     "1,0.25,0,0.002"]
    text = wire.to_string(wire.write_kernel_approx, {"seed": 1}, [(64, 0.125, 0.0)])
    assert text.splitlines()[1:] == ["features,mean_error,sd_error", "64,0.125,0"]
    # every float field survives the round trip exactly (%.17g)
    v = np.random.default_rng(0).standard_normal(100)
    assert all(float(wire.fmt17(x)) == x for x in v)


@pytest.mark.gpu
def test_gpu_collision_table_equals_reference_table(spn, ref, wire):
    """The lsh-collision table written from the GPU curve is byte-identical to the one written from the
    reference's own collision_curve on the same pairs (counts and hit ratios are exact)."""
    n, m, P, trials, seed = 64, 32, 400, 20, 7
    rng = np.random.default_rng(3)
    ang = np.pi * (np.arange(P) + 0.5) / P
    x = rng.standard_normal((P, n))
    u = rng.standard_normal((P, n))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    u -= np.sum(u * x, axis=1, keepdims=True) * x
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    y = np.cos(ang)[:, None] * x + np.sin(ang)[:, None] * u
    d = 2.0 * np.sin(ang / 2.0)
    x32, y32 = x.astype(np.float32), y.astype(np.float32)
    import torch
    fac = spn.make_hasher_factory(spn.SpinnerVariant.hd3_hd2_hd1, n, m)
    ours = spn.collision_curve((torch.from_numpy(x32).cuda(), torch.from_numpy(y32).cuda(), d), fac, trials, seed)
    r = ref.collision_curve(0, n, m, x32, y32, d, trials, seed)
    theirs = SimpleNamespace(bucket_edges=list(r["bucket_edges"]), probabilities=list(r["probabilities"]),
                             counts=[int(c) for c in r["counts"]])
    cfg = {"variant": "HD3HD2HD1", "n": n, "rows": m, "pairs": P, "trials": trials, "seed": seed}
    assert wire.to_string(wire.write_lsh_collision, cfg, ours) == wire.to_string(wire.write_lsh_collision, cfg, theirs)
