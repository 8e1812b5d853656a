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


def _keysets(n, wp):
    """three key-set readings (DESIGN R-KEYSET): Slide taps + both-sign powers of two; Slide taps + positive powers
    of two; a sparse set forcing long synthesized chains"""
    pos = [1 << i for i in range((n).bit_length() - 1)]
    return {"pm2i": pos + [-x for x in pos], "p2i": pos, "sparse": [1, 3 * wp, 7]}


@pytest.mark.parametrize("name", ["C1_raconv", "toy_dsconv", "L1_ca", "L2_ca", "L3_ds", "L3_ra", "r18_L4_pconv"])
def test_keyset_synthesis_matches_oracle(hy, name):
    """R-KEYSET: the product's shortest decompositions (C++ BFS) = the oracle's (Python BFS), the plan's loaded key
    list and effective rotation counts ("eff. total") agree, Slide amounts stay loaded"""
    s = CASES[name]
    log_n = (2 * s.n).bit_length() - 1
    K = synth.conv_weight(7, s.co, s.ci, s.f)
    o = (H.plan_caconv if s.algo == "CA" else H.plan_raconv)(s, K, with_weights=False)
    taps = [r % s.n for r in o.taps if r % s.n]
    for kname, extra in _keysets(s.n, s.wp).items():
        amounts = taps + extra
        ks_o = H.KeySet(s.n, amounts)
        ks_p = hy.KeySet(log_n, amounts)
        g = np.random.default_rng(3)
        for r in list(g.integers(0, s.n, 40)) + [-1, -s.wp, s.n // 2, 5 * s.wp + 3]:
            assert ks_p.decompose(int(r)) == ks_o.steps(int(r)), (kname, r)
        p = hy.ConvPlan(None, s.ci, s.co, s.w, s.f, s.s, s.wp, s.g, s.m, s.d, s.algo, log_n=log_n, S=s.S)
        p.set_keyset(ks_p)
        assert p.rots == H.keyset_amounts(o, ks_o), kname
        assert p.eff_counts == H.eff_counts(o, ks_o), kname
        assert p.counts == o.counts
        for r in taps:
            assert r in p.rots


def test_keyset_decompose_basics(hy):
    ks = hy.KeySet(12, [1, 8, 64])
    assert ks.decompose(0) == [] and ks.decompose(8) == [8] and ks.decompose(9) == [1, 8]
    assert sum(ks.decompose(-1)) % 2048 == 2047
    assert ks.decompose(2047) == H.KeySet(2048, [1, 8, 64]).steps(2047)
    with pytest.raises(hy.HyError):          # only even amounts reachable from {2}: 3 is not
        hy.KeySet(12, [2]).decompose(3)
    # a plan whose Slide amount is not loaded is refused (MISSING_KEY = 8)
    p = hy.ConvPlan(None, 4, 4, 8, 3, 1, 8, 1, 1, 1, "RA", log_n=12)
    with pytest.raises(hy.HyError) as e:
        p.set_keyset(hy.KeySet(12, [1]))
    assert e.value.code == 8
