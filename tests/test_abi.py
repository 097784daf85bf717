"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and its host logic (seeded generator, sampler, argument
validation) matches the reference.  No kernel launches here."""
import ctypes
import os
import re

import numpy as np
import pytest

import cases
from conftest import ROOT
from oracle.oracle import GAUSS3, HD3, HDG

HEADER = os.path.join(ROOT, "include", "spinners_b200.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"SPN_API\s+[\w\s\*]+?\b(spn_\w+)\s*\(", txt)))


def test_library_exports_every_declared_symbol(spn):
    lib = ctypes.CDLL(spn.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    assert set(spn.ABI_SYMBOLS) <= set(syms)


def test_library_is_sm100a(spn):
    import subprocess
    out = subprocess.run(["cuobjdump", "-lelf", spn.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_status_strings(spn):
    assert "sm_100a" in spn.version()
    assert spn._status_string(1).decode() == "dimension error"


def test_mix_seed_matches_reference(spn, golden):
    for (a, b), want in zip(golden["mix_seed_in"], golden["mix_seed_out"]):
        assert spn.mix_seed(int(a), int(b)) == int(want)


@pytest.mark.parametrize("v", [HD3, HDG, GAUSS3])
@pytest.mark.parametrize("n,seed", [(16, 21), (1024, 7), (1 << 17, 11)])
def test_host_generator_is_the_reference_generator(spn, oracle, v, n, seed):
    got = spn.realize_block(v, n, seed)
    want = oracle.realize_block(v, n, seed)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


def test_stacked_block_seeds_match_reference(spn, golden):
    # StackedSpinner block b uses spec seed mix_seed(seed, b) (spinner.cpp:255)
    for b in range(3):
        d = spn.realize_block(HD3, 16, spn.mix_seed(44, b))
        assert np.array_equal(d[0], golden["realize_v0_n16_k40_s44_d1"][b])
        assert np.array_equal(d[2], golden["realize_v0_n16_k40_s44_d3"][b])


def test_sampler_matches_oracle(spn, oracle):
    for N, m, s in [(10, 3, 1), (1 << 17, 2048, 77), (64, 64, 2)]:
        assert np.array_equal(spn.sample_rows(N, m, s), oracle.sample_rows(N, m, s))


def test_config4_rows_fixture(spn, golden):
    c = cases.C4
    assert np.array_equal(spn.sample_rows(c["N"], c["m"], c["p_seed"]), golden["c4_rows"])


def test_validation_errors_before_any_device_work(spn):
    # spinner.cpp:59-67 -> DimensionError / DomainError, raised before CUDA is touched
    with pytest.raises(spn.DimensionError):
        spn.StackedSpinner(spn.SpinnerVariant.hd3_hd2_hd1, 6, 6, 6, 0)
    with pytest.raises(spn.DimensionError):
        spn.StackedSpinner(spn.SpinnerVariant.hd3_hd2_hd1, 8, 9, 9, 0)
    with pytest.raises(spn.DimensionError):
        spn.StackedSpinner(spn.SpinnerVariant.hd3_hd2_hd1, 8, 0, 8, 0)
    with pytest.raises(spn.DimensionError):
        spn.StackedSpinner(spn.SpinnerVariant.hd3_hd2_hd1, 8, 8, 0, 0)
    with pytest.raises(spn.DomainError):
        spn.variant_from_string("NotAVariant")
    with pytest.raises(spn.DomainError):
        spn.KernelKind.gaussian(0.0)
    with pytest.raises(spn.DimensionError):
        spn.sample_rows(4, 5, 0)
    with pytest.raises(spn.DimensionError):
        spn.SpinnerSpec.make(spn.SpinnerVariant.hd3_hd2_hd1, 12, 4, 0)


def test_raw_abi_null_and_bad_arguments(spn):
    lib = spn._lib
    assert lib.spn_plan_create(None, None) == spn.SPN_EINVAL
    assert lib.spn_plan_destroy(None) == spn.SPN_OK
    assert spn._apply(None, None, 0, 0, 1, None, 0, 0, None) == spn.SPN_EINVAL
    assert spn._realize_block(7, 8, 0, None, None, None) == spn.SPN_EINVAL
    # fwht_normalized / diag_matvec (transforms.cpp:52-71,228-235): shape errors before any device work
    assert spn._fwht(3, None, 1, 3, None, 3, 0, None) == spn.SPN_EDIM
    assert spn._fwht(0, None, 1, 0, None, 0, 0, None) == spn.SPN_EDIM
    assert spn._fwht_host(6, None, 1, 6, None, 6, 0) == spn.SPN_EDIM
    assert spn._fwht(8, None, 1, 4, None, 8, 0, None) == spn.SPN_EINVAL
    assert spn._diag_host(4, None, None, 1, 2, None, 4, 0) == spn.SPN_EDIM
    with pytest.raises(spn.DimensionError):
        spn.fwht_normalized([1.0, 2.0, 3.0])
    with pytest.raises(spn.DomainError):
        spn.fwht_normalized([1.0, float("inf")])
    with pytest.raises(spn.DimensionError):
        spn.diag_matvec([1.0], [1.0, 2.0])
    # CirculantSpec::validate (transforms.cpp:98-110) before any device work
    import ctypes
    h = spn._vp()
    row = np.array([1.0, 2.0]); bad = np.array([3.0, 2.0]); nan = np.array([np.nan, 1.0])
    assert spn._circ_create(ctypes.byref(h), 0, 0, row.ctypes.data, None, 0) == spn.SPN_EDIM
    assert spn._circ_create(ctypes.byref(h), 1, 2, row.ctypes.data, bad.ctypes.data, 0) == spn.SPN_EDOMAIN
    assert spn._circ_create(ctypes.byref(h), 0, 2, nan.ctypes.data, None, 0) == spn.SPN_EDOMAIN
    assert spn._circ_create(ctypes.byref(h), 0, 2, row.ctypes.data, row.ctypes.data, 0) == spn.SPN_EDIM
    assert spn._circ_create(ctypes.byref(h), 7, 2, row.ctypes.data, None, 0) == spn.SPN_EDOMAIN
    with pytest.raises(spn.DomainError):
        spn.CirculantSpec.toeplitz([1.0, 2.0], [2.0, 3.0])
    with pytest.raises(spn.DimensionError):
        spn.CirculantSpec(spn.CirculantKind.circulant, [1.0, 2.0], [1.0, 2.0])


def test_signed_argmax_host_helper(spn):
    assert spn.signed_argmax([0.1, -0.9, 0.3]) == (1, -1)
    assert spn.signed_argmax([-2.0, 2.0]) == (0, -1)
    assert spn.signed_argmax([0.0, 0.0]) == (0, 1)
    assert spn.decode_id(1030, 1024) == (6, -1) and spn.decode_id(6, 1024) == (6, 1)


def test_spec_json_round_trip(spn):
    """SpinnerSpec::to_json / from_json (spinner.cpp:72-89)."""
    import json
    for v in ("HD3HD2HD1", "GToeplitzD2HD1", "GaussianDense"):
        s = spn.SpinnerSpec.make(spn.variant_from_string(v), 64, 32, 7)
        j = json.loads(json.dumps(s.to_json()))
        assert j["variant"] == v and j["scale"] == s.effective_scale()
        t = spn.SpinnerSpec.from_json(j)
        assert (t.variant, t.n, t.m, t.seed, t.effective_scale()) == (s.variant, 64, 32, 7, s.effective_scale())
    with pytest.raises(spn.DomainError):
        spn.SpinnerSpec.from_json({"variant": "Nope", "n": 4, "m": 4, "seed": 0})


def test_host_allocation_failure_is_a_status_not_an_abort(spn):
    """Every C-ABI entry point is an exception barrier: a host allocation that cannot succeed (2^25 tables
    of 2^20-point HDg blocks = 2^45 doubles per diagonal) comes back as SPN_ENOMEM instead of terminating
    the process (std::bad_alloc never crosses the extern "C" boundary)."""
    import ctypes
    d = spn._Desc()
    d.variant, d.n, d.m, d.k, d.tables = int(spn.SpinnerVariant.hdg_hd2_hd1), 1 << 20, 1 << 20, 1 << 20, 1 << 25
    seeds = (spn._u64 * 4)(1, 2, 3, 4)  # never read: the allocation fails first
    d.table_seeds = ctypes.cast(seeds, ctypes.POINTER(spn._u64))
    h = spn._vp()
    assert spn._plan_create(ctypes.byref(h), ctypes.byref(d)) == spn.SPN_ENOMEM
    assert not h.value
    assert "allocation" in spn._last_error().decode()


def test_new_entry_points_reject_bad_arguments(spn):
    import ctypes
    h = spn._vp()
    r = np.zeros(4)
    assert spn._plan_resample(None, None, 0, 1) == spn.SPN_EINVAL
    assert spn._plan_resample(ctypes.byref(h), None, 0, 1) == spn.SPN_EINVAL
    assert spn._plan_with_tail(ctypes.byref(h), None, r.ctypes.data) == spn.SPN_EINVAL
    assert spn._sketch_host(None, None, 1, 1, 1, None, 1, 1.0, None, 1) == spn.SPN_EINVAL
    assert spn._hash_project_host(None, None, 1, 1, 1, None, None, 1) == spn.SPN_EINVAL
    assert spn._hash_peers(None, None, 1, 1, 1, None, 1, 0, 1, None) == spn.SPN_EINVAL
