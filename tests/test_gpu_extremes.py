"""GPU parity on max-magnitude residues (VERDICT r01 "weak" 2b, ADVICE hy_arith.cuh:84).

The FP64-pipe kernels (DESIGN R-FP64) keep NTT values unreduced across up to 8 butterfly stages and feed
them into further products; their exactness rests on the growth bound of DESIGN R-FP64 (largest fmulmod
operand 6.62 q < 2^51 / q_max).  Random residues and fresh encryptions rarely approach it, so every step of the
path is run here, bit-exact against the oracle, on limbs that are all q-1, alternating 0 / q-1, all (q-1)/2 and
all 1, at Set_hyp (the 48-bit q_0 and p_k are the primes that come closest to the bound) and at the toy set.
"""
import numpy as np
import pytest

import oracle
import synth
from oracle import hyphen as H

pytestmark = pytest.mark.gpu

SK, EK = synth.SEED_SK, synth.SEED_EVK
PATTERNS = ("max", "alt", "half", "one")


def to_np(t):
    return t.detach().cpu().numpy().view(np.uint64)


def to_dev(a, ctx):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(ctx.device)


def limbs(o, chain, pattern):
    """one limb per chain index, every word set by `pattern` (residues of o.moduli[t])"""
    out = np.empty((len(chain), o.N), np.uint64)
    for i, t in enumerate(chain):
        q = int(o.moduli[t])
        if pattern == "max":
            out[i] = q - 1
        elif pattern == "alt":
            out[i, 0::2], out[i, 1::2] = 0, q - 1
        elif pattern == "half":
            out[i] = (q - 1) // 2
        else:
            out[i] = 1
    return out


def ct_limbs(o, level, pattern):
    return limbs(o, list(range(level + 1)) * 2, pattern).reshape(2, level + 1, o.N)


_PAIRS = {}


def _pair(name):
    if name not in _PAIRS:
        import paper_2302_02407_b200 as hy
        prm = synth.PARAMS[name]
        _PAIRS[name] = (hy.Context(**prm, max_batch=8), oracle.Oracle(**prm))
    return _PAIRS[name]


@pytest.mark.parametrize("name", ["toy", "hyp"])
@pytest.mark.parametrize("pattern", PATTERNS)
def test_ntt_extremes(name, pattern):
    ctx, o = _pair(name)
    chain = list(range(o.nq + o.np_))
    a = limbs(o, chain, pattern)
    A = to_np(ctx.ntt(to_dev(a, ctx), chain))
    assert np.array_equal(A, np.stack([o.ntt(a[t], t) for t in chain]))
    assert np.array_equal(to_np(ctx.ntt(to_dev(a, ctx), chain, inverse=True)),
                          np.stack([o.intt(a[t], t) for t in chain]))


@pytest.mark.parametrize("pattern", PATTERNS)
def test_modup_moddown_extremes(pattern):
    ctx, o = _pair("hyp")
    for level in (23, 9):
        d = limbs(o, list(range(level + 1)), pattern)
        assert np.array_equal(to_np(ctx.modup(level, to_dev(d, ctx))), o.modup_coeff(level, d))
        uu = limbs(o, o.ext_chain(level), pattern)
        assert np.array_equal(to_np(ctx.moddown(level, to_dev(uu, ctx))), o.moddown(level, uu))


_KEYS = {}


def _keys(name, rs):
    ctx, o = _pair(name)
    out = []
    for r in rs:
        if (name, r) not in _KEYS:
            ok = o.keygen_rot(SK, EK, r)
            _KEYS[(name, r)] = (ok, ctx.evk_pack(to_dev(ok, ctx)))
        out.append(_KEYS[(name, r)])
    return out


def test_ks_inner_product_extremes():
    """IP with max-magnitude extended digits (the products of the key-switch inner product)"""
    ctx, o = _pair("hyp")
    level = 23
    (ok, dk), = _keys("hyp", [1])
    for pattern in ("max", "alt"):
        d = limbs(o, list(range(level + 1)), pattern)
        oext = o.modup_coeff(level, d)
        u = ctx.ks_inner_product(level, to_dev(oext, ctx), dk)
        assert np.array_equal(to_np(u), o.ks_inner_product(level, oext, ok))


@pytest.mark.parametrize("level", [23, 9])
@pytest.mark.parametrize("pattern", ["max", "alt", "half"])
def test_hrot_variants_extremes(level, pattern):
    """plain (batched), hoisted and lazy-sum HRot of ciphertexts whose limbs are max-magnitude (not encryptions:
    the key switch is a limbwise-defined map, the oracle computes the same one)"""
    ctx, o = _pair("hyp")
    rs = [1, -5]
    ks = _keys("hyp", rs)
    a = ct_limbs(o, level, pattern)
    b = ct_limbs(o, level, "max" if pattern != "max" else "alt")
    da, db = to_dev(a, ctx), to_dev(b, ctx)
    oa, ob = oracle.Ct(a, level, 1.0), oracle.Ct(b, level, 1.0)
    outs = ctx.hrot_batch([k[1] for k in ks], [da, db], level, rs)
    for out, oc, r, k in zip(outs, (oa, ob), rs, ks):
        assert np.array_equal(to_np(out), o.hrot(oc, k[0], r).data), r
    hh = ctx.hrot_hoisted([k[1] for k in ks], da, level, rs)
    for g, w in zip(hh, o.hrot_hoisted(oa, [k[0] for k in ks], rs)):
        assert np.array_equal(to_np(g), w.data)
    s = ctx.hrot_sum([k[1] for k in ks], [da, db], level, rs)
    assert np.array_equal(to_np(s), o.hrot_sum([oa, ob], [k[0] for k in ks], rs).data)


@pytest.mark.parametrize("pattern", PATTERNS)
def test_pmult_rescale_extremes(pattern):
    ctx, o = _pair("hyp")
    for level in (23, 9, 1):
        a = ct_limbs(o, level, pattern)
        p = limbs(o, list(range(level + 1)), "max")
        A, Pt = oracle.Ct(a, level, 1.0), oracle.Pt(p, level, 1.0)
        da, dp = to_dev(a, ctx), to_dev(p, ctx)
        assert np.array_equal(to_np(ctx.pmult(da, dp, level)), o.pmult(A, Pt).data)
        acc = ctx.pmult_acc([da, da, da], [dp, dp, dp], level)
        want = o.add(o.add(o.pmult(A, Pt), o.pmult(A, Pt)), o.pmult(A, Pt))
        assert np.array_equal(to_np(acc), want.data)
        assert np.array_equal(to_np(ctx.rescale(da, level)), o.rescale(A).data)


@pytest.mark.parametrize("pattern", ["max", "alt"])
def test_conv_layer_extremes(pattern):
    """CAConv (hoisted Slide, MulFilter&Sum block kernel k_pmult_block, rescale, RaS) and RAConv (PMult, lazy
    HRotSum) at N = 2^16 on max-magnitude input ciphertexts: a sampled output bit-exact vs the oracle"""
    import paper_2302_02407_b200 as hy
    from test_hyphen_plan import R20
    ctx, o = _pair("hyp")
    for name, j in (("L3_ca", 2), ("L1_ra", 0)):
        spec = R20[name]
        level = 9 if spec.algo == "CA" else 6
        K = synth.conv_weight(23, spec.co, spec.ci, spec.f)
        p = hy.ConvPlan(ctx, spec.ci, spec.co, spec.w, spec.f, spec.s, spec.wp, spec.g, spec.m, spec.d, spec.algo,
                        S=spec.S)
        plan = H.plan_caconv(spec, K) if spec.algo == "CA" else H.plan_raconv(spec, K)
        octs = [oracle.Ct(ct_limbs(o, level, pattern), level, 2.0**42) for _ in range(plan.n_in)]
        evks = {r: ctx.keygen_rot(SK, EK, r) for r in p.rots}
        out = p.run(evks, [to_dev(c.data, ctx) for c in octs], level, p.encode_weights(K, level), out_begin=j,
                    out_end=j + 1)[0]
        oevks = {r: o.keygen_rot(SK, EK, r) for r in H.rotation_amounts(plan, o.n)}
        want = H.EncConv(o, plan, oevks).run(octs, [j])[0]
        assert np.array_equal(to_np(out), want.data), name
