"""CPU-side checks of the product boundary: the C-ABI library loads, exports every
symbol include/hyphen.h declares, refuses to run without a device, and its
host-side encoder agrees bit-for-bit with the oracle's (DESIGN R-ENCODE)."""
import os
import re

import numpy as np
import pytest

import oracle
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def hy():
    from paper_2302_02407_b200 import build
    build.build()
    import paper_2302_02407_b200 as hy
    return hy


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hyphen.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hy_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(hy):
    import ctypes
    L = ctypes.CDLL(hy.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    # the Python binding declares a signature for every exported entry point
    assert set(syms) <= set(hy.SIGNATURES), set(syms) - set(hy.SIGNATURES)


def test_no_device_fails_loudly(hy):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    with pytest.raises(hy.HyError) as e:
        hy.Context(**synth.PARAMS["toy"])
    assert e.value.code == 11  # HY_E_NO_DEVICE


@pytest.mark.parametrize("pset,scale_kind", [("toy", "pow2"), ("mini", "prime"), ("hyp", "pow2"), ("hyp", "prime")])
def test_encode_matches_oracle(hy, pset, scale_kind):
    prm = synth.PARAMS[pset]
    o = oracle.Oracle(**prm)
    scale = 2 ** prm["log_scale"] if scale_kind == "pow2" else o.q[-1]
    for seed in range(2):
        z = synth.slots_uniform(100 + seed, o.n)
        a = hy.encode_coeffs(prm["log_n"], z, scale)
        b = o.encode_coeffs(z, scale)
        assert np.array_equal(a, b)
    # short vector (zero padded), structured 0/1 mask (exact algebraic values)
    z = np.zeros(o.n)
    z[::4] = 1.0
    assert np.array_equal(hy.encode_coeffs(prm["log_n"], z, scale), o.encode_coeffs(z, scale))
    z = synth.slots_uniform(7, o.n // 3)
    assert np.array_equal(hy.encode_coeffs(prm["log_n"], z, scale), o.encode_coeffs(z, scale))


def test_encode_tie_rule(hy):
    for c, scale, want in [(0.5, 1, 1), (-0.5, 1, -1), (1.5, 1, 2), (-2.5, 1, -3)]:
        m = hy.encode_coeffs(10, np.full(512, c), scale)
        assert int(m[0]) == want and not np.any(m[1:])


@pytest.mark.parametrize("pset", ["toy", "hyp"])
def test_decode_coeffs_matches_oracle(hy, pset):
    """Host decode (hy_decode_coeffs) = the oracle's canonical embedding m(zeta^{5^j}) / scale (its own
    pinned eval_slots, an independent 2N-point FFT) for random integer coefficients, and it inverts encode."""
    prm = synth.PARAMS[pset]
    o = oracle.Oracle(**prm)
    scale = 2.0 ** prm["log_scale"]
    m = np.random.default_rng(5).integers(-2**50, 2**50, o.N).astype(np.float64)
    got = hy.decode_coeffs(prm["log_n"], m, scale)
    want = o.eval_slots(m) / scale
    assert np.max(np.abs(got - want)) < 1e-9 * np.max(np.abs(want))
    z = synth.slots_uniform(9, o.n)
    back = hy.decode_coeffs(prm["log_n"], hy.encode_coeffs(prm["log_n"], z, int(scale)).astype(np.float64), scale)
    assert np.max(np.abs(back - z)) < 2**-25
    assert hy.decode_coeffs(prm["log_n"], m, scale, n_slots=7).shape == (7,)


@pytest.mark.parametrize("spec,code", [
    ((4, 4, 8, 3, 1, 8, 1, 3, 1, "RA"), 6),    # m not a power of two: HY_E_FORMAT
    ((4, 4, 8, 2, 1, 8, 1, 1, 1, "RA"), 4),    # even filter: HY_E_SHAPE
    ((4, 4, 8, 3, 3, 8, 1, 1, 1, "CA"), 4),    # stride 3: HY_E_SHAPE
    ((4, 4, 16, 3, 1, 8, 1, 1, 1, "CA"), 5),   # image wider than the physical width: HY_E_CAPACITY
    ((4, 4, 8, 3, 2, 8, 1, 1, 1, "RA"), 6),    # stride-2 RAConv: HY_E_FORMAT (downsampling is in CAConv)
    ((4, 4, 8, 3, 1, 8, 2, 1, 1, "CA"), 6),    # m d not a multiple of g^2: HY_E_FORMAT
])
def test_conv_plan_errors(hy, spec, code):
    """hy_conv_plan_create checks the spec on the host (no device) and returns the documented status."""
    with pytest.raises(hy.HyError) as e:
        hy.ConvPlan(None, *spec, log_n=12)
    assert e.value.code == code, hy.lib().hy_last_error()


def test_host_entry_errors(hy):
    """host-only entry points: more slots than N/2 is HY_E_CAPACITY, log_n out of range is HY_E_ARG."""
    with pytest.raises(hy.HyError) as e:
        hy.encode_coeffs(10, np.zeros(513), 2**20)
    assert e.value.code == 5
    with pytest.raises(hy.HyError) as e:
        hy.decode_coeffs(10, np.zeros(1024), 2.0**20, n_slots=513)
    assert e.value.code == 5
    with pytest.raises(hy.HyError) as e:
        hy.decode_coeffs(1, np.zeros(2), 1.0)
    assert e.value.code == 1
