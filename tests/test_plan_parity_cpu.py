"""The product's host-side conv plans (C++) against the oracle's (numpy), CPU only:
identical rotation amounts, counts and bit-identical weight / mask slot vectors."""
import numpy as np
import pytest

import synth
from oracle import hyphen as H
from test_hyphen_plan import PRCR, R20


@pytest.fixture(scope="module")
def hy():
    from paper_2302_02407_b200 import build
    build.build()
    import paper_2302_02407_b200 as hy
    return hy


CASES = dict(R20)
CASES["C1_raconv"] = H.ConvSpec(4, 4, 8, 3, 1, 8, 1, 1, 1, "RA", n=2048)
CASES["toy_dsconv"] = H.ConvSpec(4, 8, 8, 3, 2, 8, 1, 1, 2, "CA", n=2048)
CASES["r18_L4_ra"] = H.ConvSpec(512, 512, 7, 3, 1, 64, 8, 8, 8, "RA")
# ResNet-18 downsampling blocks (full weights): dsconv from plan (1,1) and the stage-4 pconv from (4,4)
CASES["r18_L2_ds"] = H.ConvSpec(64, 128, 56, 3, 2, 64, 1, 1, 1, "CA")
CASES["r18_L4_pconv"] = H.ConvSpec(256, 512, 14, 1, 2, 64, 4, 4, 4, "CA")
CASES.update(PRCR)


@pytest.mark.parametrize("name", list(CASES))
def test_plan_matches_oracle(hy, name):
    s = CASES[name]
    K = synth.conv_weight(7, s.co, s.ci, s.f)
    log_n = (2 * s.n).bit_length() - 1
    p = hy.ConvPlan(None, s.ci, s.co, s.w, s.f, s.s, s.wp, s.g, s.m, s.d, s.algo, log_n=log_n, S=s.S)
    big = s.ci * s.co > 64 * 64
    o = (H.plan_caconv if s.algo == "CA" else H.plan_raconv)(s, K, with_weights=not big)
    assert (p.n_in, p.n_out) == (o.n_in, o.n_out)
    assert p.rots == H.rotation_amounts(o, s.n)
    assert p.counts == o.counts
    assert p.has_mask == (o.mask is not None)
    keys = sorted(o.weights) if not big else []
    for idx, key in enumerate(keys):
        assert np.array_equal(p.weight_slots(K, idx), o.weights[key]), (name, key)
    if o.mask is not None:
        assert np.array_equal(p.weight_slots(K, p.n_pt), o.mask)


@pytest.mark.parametrize("name", ["C1_raconv", "toy_dsconv", "L1_ca", "L2_ra", "L3_ds", "r18_L4_pconv"]
                         + [k for k in PRCR][:2])
def test_bias_slots_match_oracle(hy, name):
    """DESIGN R-BIAS: the product's bias plaintext slots (hy_conv_bias_slots) = the oracle's packing of the bias
    image in the output format, for every output ciphertext"""
    s = CASES[name]
    log_n = (2 * s.n).bit_length() - 1
    b = synth.conv_bias(9, s.co)
    p = hy.ConvPlan(None, s.ci, s.co, s.w, s.f, s.s, s.wp, s.g, s.m, s.d, s.algo, log_n=log_n, S=s.S, bias=True)
    o = (H.plan_caconv if s.algo == "CA" else H.plan_raconv)(s, synth.conv_weight(7, s.co, s.ci, s.f),
                                                              with_weights=False)
    want = H.bias_slots(o, b)
    for j in range(p.n_out):
        assert np.array_equal(p.bias_slots(b, j), want[j]), (name, j)
