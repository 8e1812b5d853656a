"""GPU parity of the HyPHEN conv layers (hy_caconv / hy_raconv through the C ABI)
against the oracle's encrypted execution of its own plan: bit-exact on every RNS
limb.  Toy layers (N = 2^12) run in full; ResNet-20 layers at Set_hyp (N = 2^16)
are checked on sampled output ciphertexts at the conv levels (l+1 = 10 / 7)."""
import numpy as np
import pytest

import oracle
import synth
from oracle import hyphen as H
from test_hyphen_plan import R20

pytestmark = pytest.mark.gpu
SK, EK = synth.SEED_SK, synth.SEED_EVK


def to_np(t):
    return t.detach().cpu().numpy().view(np.uint64)


@pytest.fixture(scope="module")
def ctx_toy():
    import paper_2302_02407_b200 as hy
    return hy.Context(**synth.PARAMS["toy"])


@pytest.fixture(scope="module")
def ctx_hyp():
    import paper_2302_02407_b200 as hy
    return hy.Context(**synth.PARAMS["hyp"])


def gpu_layer(ctx, spec, X, K, level, scale, out_begin=0, out_end=None):
    import paper_2302_02407_b200 as hy
    p = hy.ConvPlan(ctx, spec.ci, spec.co, spec.w, spec.f, spec.s, spec.wp, spec.g, spec.m, spec.d, spec.algo,
                    S=spec.S)
    fin = H.Fmt("CA" if spec.algo == "CA" else "RA", spec.n, spec.wp, spec.g, spec.m, spec.d, spec.S)
    cts = [ctx.encrypt(SK, 900, i, ctx.encode(v, scale, level), level) for i, v in enumerate(H.pack(X, fin))]
    evks = {r: ctx.keygen_rot(SK, EK, r) for r in p.rots}
    pts = p.encode_weights(K, level)
    outs = p.run(evks, cts, level, pts, out_begin=out_begin, out_end=out_end)
    return p, outs


def oracle_layer(o, spec, X, K, level, scale, outputs=None):
    plan = H.plan_caconv(spec, K) if spec.algo == "CA" else H.plan_raconv(spec, K)
    cts = [o.encrypt(SK, 900, i, o.encode(v, scale, level)) for i, v in enumerate(H.pack(X, plan.fin))]
    wanted = range(plan.n_out) if outputs is None else outputs
    need = set()
    for r in H.rotation_amounts(plan, o.n):
        need.add(r)
    evks = {r: o.keygen_rot(SK, EK, r) for r in need}
    return plan, H.EncConv(o, plan, evks).run(cts, list(wanted))


TOY = [
    H.ConvSpec(4, 4, 8, 3, 1, 8, 1, 1, 1, "RA", n=2048),
    H.ConvSpec(4, 4, 8, 3, 1, 8, 1, 1, 1, "CA", n=2048),
    H.ConvSpec(8, 8, 8, 3, 1, 8, 1, 1, 2, "CA", n=2048),
    H.ConvSpec(8, 8, 8, 3, 1, 8, 1, 2, 1, "RA", n=2048),
    H.ConvSpec(8, 8, 4, 3, 1, 8, 2, 2, 4, "CA", n=2048),
    H.ConvSpec(4, 8, 8, 3, 2, 8, 1, 1, 2, "CA", n=2048),
    H.ConvSpec(4, 8, 8, 1, 2, 8, 1, 1, 2, "CA", n=2048),
    H.ConvSpec(64, 8, 6, 3, 1, 8, 1, 1, 1, "CA", n=2048, S=2),
    H.ConvSpec(8, 64, 6, 3, 1, 8, 1, 1, 1, "RA", n=2048, S=2),
]


@pytest.mark.parametrize("spec", TOY, ids=["C1_raconv", "ca11", "ca12", "ra21", "ca_g2", "dsconv", "pconv",
                                           "prcr_ca", "prcr_ra"])
def test_toy_layers_bit_exact(ctx_toy, orc_toy, spec):
    level = orc_toy.nq - 1
    X = synth.image(11, spec.ci, spec.w)
    K = synth.conv_weight(12, spec.co, spec.ci, spec.f)
    p, outs = gpu_layer(ctx_toy, spec, X, K, level, 2 ** 40)
    plan, ref = oracle_layer(orc_toy, spec, X, K, level, 2 ** 40)
    assert len(outs) == len(ref) == plan.n_out
    for a, b in zip(outs, ref):
        assert np.array_equal(to_np(a), b.data)
    # and the decryption is the plaintext convolution (2^-10, north star)
    dec = [np.real(orc_toy.decode(orc_toy.decrypt(SK, oracle.Ct(to_np(a), b.level, b.scale)))) for a, b in zip(outs, ref)]
    got = H.unpack(dec, plan.fout, spec.co, spec.wo, spec.wo)
    want = H.conv2d(X, K, spec.s)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 2 ** -10


R18 = {"r18_L1_ca_S8": H.ConvSpec(64, 64, 56, 3, 1, 64, 1, 1, 1, "CA", S=8),
       # PRCR RAConv over 64 input ciphertexts (PRot-gathered weights, lazy HRotSum), stage-4 CAConv at (8, 8)
       "r18_L1_ra_S8": H.ConvSpec(64, 64, 56, 3, 1, 64, 1, 1, 1, "RA", S=8),
       "r18_L4_ca_S8": H.ConvSpec(512, 512, 7, 3, 1, 64, 8, 8, 8, "CA", S=8),
       # ResNet-18 stage-4 shortcut: 1x1 stride-2 pconv from plan (4,4) at gap 4 to RA(8,8) at gap 8
       "r18_L4_pconv": H.ConvSpec(256, 512, 14, 1, 2, 64, 4, 4, 4, "CA")}



@pytest.mark.parametrize("name,outputs", [("L1_ra", [0]), ("L3_ca", [3]), ("L3_ds", [1]), ("r18_L1_ca_S8", [5]),
                                          ("r18_L4_pconv", [1]), ("r18_L4_ca_S8", [7]),
                                          ("r18_L1_ra_S8", [3])])
def test_resnet_layers_sampled(ctx_hyp, orc_hyp, name, outputs):
    spec = R20[name] if name in R20 else R18[name]
    level = 9 if spec.algo == "CA" else 6      # l+1 = 10 for CAConv, 7 for RAConv (DESIGN R-LEVELS)
    X = synth.image(21, spec.ci, spec.w)
    K = synth.conv_weight(22, spec.co, spec.ci, spec.f)
    j = outputs[0]
    p, outs = gpu_layer(ctx_hyp, spec, X, K, level, 2 ** 42, j, j + 1)
    plan, ref = oracle_layer(orc_hyp, spec, X, K, level, 2 ** 42, outputs)
    assert np.array_equal(to_np(outs[0]), ref[0].data)


def _tap_split_equals_raconv(ctx, spec, level, scale, j, shards):
    """hy_raconv_partial over disjoint tap ranges, states added as integers (what the all-reduce of
    dist.raconv_tap_sharded does across ranks), then hy_raconv_finish: bit-identical to hy_raconv."""
    import paper_2302_02407_b200 as hy
    p = hy.ConvPlan(ctx, spec.ci, spec.co, spec.w, spec.f, spec.s, spec.wp, spec.g, spec.m, spec.d, spec.algo,
                    S=spec.S)
    fin = H.Fmt("RA", spec.n, spec.wp, spec.g, spec.m, spec.d, spec.S)
    X = synth.image(31, spec.ci, spec.w)
    K = synth.conv_weight(32, spec.co, spec.ci, spec.f)
    cts = [ctx.encrypt(SK, 901, i, ctx.encode(v, scale, level), level) for i, v in enumerate(H.pack(X, fin))]
    evks = {r: ctx.keygen_rot(SK, EK, r) for r in p.rots}
    pts = p.encode_weights(K, level)
    want = p.run(evks, cts, level, pts, out_begin=j, out_end=j + 1)[0]
    total = p.partial_state(level)
    for b, e in shards:
        st = p.partial_state(level)
        p.raconv_partial(evks, cts, level, pts, j, b, e, st)
        total += st  # int64 sum, as the all-reduce
    got = p.raconv_finish(evks, level, pts, total, j)
    assert np.array_equal(to_np(got), to_np(want))


@pytest.mark.parametrize("shards", [[(0, 9)], [(0, 5), (5, 9)], [(0, 2), (2, 4), (4, 6), (6, 8), (8, 9), (9, 9)]])
def test_raconv_tap_sharding_toy(ctx_toy, shards):
    # config 1 (BASELINE configs[0]) and an R_g = 2 layer (IR_g mask step)
    _tap_split_equals_raconv(ctx_toy, TOY[0], 2, 2 ** 40, 0, shards)
    _tap_split_equals_raconv(ctx_toy, TOY[3], 2, 2 ** 40, 0, shards)


def test_raconv_tap_sharding_resnet20(ctx_hyp):
    # ResNet-20 stage-3 RAConv (one output ciphertext) at l+1 = 7, taps over 8 "ranks"
    shards = [(0, 2)] + [(t, t + 1) for t in range(2, 9)]
    _tap_split_equals_raconv(ctx_hyp, R20["L3_ra"], 6, 2 ** 42, 0, shards)


def test_block_mini_bit_exact():
    """Alg. 3 block (CAConv -> x^2 -> RAConv) through the C ABI, bit-exact vs the oracle's composition, and its
    decryption = conv2d(conv2d(X, K1)^2, K2) within 2^-10."""
    import paper_2302_02407_b200 as hy
    prm = synth.PARAMS["mini"]
    ctx, o = hy.Context(**prm), oracle.Oracle(**prm)
    n = o.n
    ca_s = H.ConvSpec(4, 4, 4, 3, 1, 4, 1, 1, 2, "CA", n=n)
    ra_s = H.ConvSpec(4, 4, 4, 3, 1, 4, 1, 2, 1, "RA", n=n)
    X = synth.image(70, 4, 4)
    K1, K2 = synth.conv_weight(71, 4, 4, 3), synth.conv_weight(72, 4, 4, 3)
    ca, ra = H.plan_caconv(ca_s, K1), H.plan_raconv(ra_s, K2)
    level = o.nq - 1
    octs = [o.encrypt(SK, 73, i, o.encode(v, 2**40, level)) for i, v in enumerate(H.pack(X, ca.fin))]
    ek = {r: o.keygen_rot(SK, EK, r) for r in H.rotation_amounts(ca, n)}
    rk = {r: o.keygen_rot(SK, EK, r) for r in H.rotation_amounts(ra, n)}
    want = H.run_block_encrypted(o, ca, ra, ek, rk, o.keygen_relin(SK, EK), octs)
    g_ca = hy.ConvPlan(ctx, *[getattr(ca_s, k) for k in ("ci", "co", "w", "f", "s", "wp", "g", "m", "d", "algo")])
    g_ra = hy.ConvPlan(ctx, *[getattr(ra_s, k) for k in ("ci", "co", "w", "f", "s", "wp", "g", "m", "d", "algo")])
    blk = hy.ConvBlock(ctx, g_ca, g_ra)
    mid, ra_level, out_level = blk.levels(level)
    import torch
    cts = [torch.from_numpy(c.data.view(np.int64)).to(ctx.device) for c in octs]
    got = blk.run({r: ctx.keygen_rot(SK, EK, r) for r in g_ca.rots}, {r: ctx.keygen_rot(SK, EK, r) for r in g_ra.rots},
                  ctx.keygen_relin(SK, EK), cts, level, g_ca.encode_weights(K1, level),
                  g_ra.encode_weights(K2, ra_level))
    assert len(got) == len(want)
    for a, b in zip(got, want):
        assert b.level == out_level and np.array_equal(to_np(a), b.data)
    dec = [np.real(o.decode(o.decrypt(SK, b))) for b in want]
    res = H.unpack(dec, ra.fout, 4, 4, 4)
    ref = H.conv2d(H.conv2d(X, K1) ** 2, K2)
    assert np.max(np.abs(res - ref)) / np.max(np.abs(ref)) < 2**-10


@pytest.mark.parametrize("spec", [TOY[0], TOY[5], TOY[7]], ids=["C1_raconv", "dsconv", "prcr_ca"])
def test_toy_layers_bias_bit_exact(ctx_toy, orc_toy, spec):
    """the conv bias (hy_conv_spec.bias, hy_conv_encode_weights' bias plaintexts, AddPt after the layer; DESIGN
    R-BIAS) bit-exact vs the oracle's EncConv with bias, and decrypting to conv2d(X, K) + b within 2^-10"""
    import paper_2302_02407_b200 as hy
    level = orc_toy.nq - 1
    X = synth.image(13, spec.ci, spec.w)
    K = synth.conv_weight(14, spec.co, spec.ci, spec.f)
    b = synth.conv_bias(15, spec.co)
    p = hy.ConvPlan(ctx_toy, spec.ci, spec.co, spec.w, spec.f, spec.s, spec.wp, spec.g, spec.m, spec.d, spec.algo,
                    S=spec.S, bias=True)
    fin = H.Fmt("CA" if spec.algo == "CA" else "RA", spec.n, spec.wp, spec.g, spec.m, spec.d, spec.S)
    cts = [ctx_toy.encrypt(SK, 902, i, ctx_toy.encode(v, 2**40, level), level) for i, v in enumerate(H.pack(X, fin))]
    evks = {r: ctx_toy.keygen_rot(SK, EK, r) for r in p.rots}
    outs = p.run(evks, cts, level, p.encode_weights(K, level, bias=b, bias_scale=2**40))
    o = orc_toy
    plan = H.plan_caconv(spec, K) if spec.algo == "CA" else H.plan_raconv(spec, K)
    octs = [o.encrypt(SK, 902, i, o.encode(v, 2**40, level)) for i, v in enumerate(H.pack(X, plan.fin))]
    oevks = {r: o.keygen_rot(SK, EK, r) for r in H.rotation_amounts(plan, o.n)}
    ref = H.EncConv(o, plan, oevks, bias=b).run(octs)
    for a, r in zip(outs, ref):
        assert np.array_equal(to_np(a), r.data)
    dec = [np.real(o.decode(o.decrypt(SK, r))) for r in ref]
    got = H.unpack(dec, plan.fout, spec.co, spec.wo, spec.wo)
    want = H.conv2d(X, K, spec.s, bias=b)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 2 ** -10


def test_raconv_tap_sharding_with_bias(ctx_toy):
    """hy_raconv_finish adds the bias too: tap-sharded = hy_raconv, bit for bit"""
    import paper_2302_02407_b200 as hy
    spec, level = TOY[0], 2
    p = hy.ConvPlan(ctx_toy, spec.ci, spec.co, spec.w, spec.f, spec.s, spec.wp, spec.g, spec.m, spec.d, spec.algo,
                    bias=True)
    cts = [ctx_toy.encrypt(SK, 903, i, ctx_toy.encode(synth.slots_uniform(50 + i, 2048), 2**40, level), level)
           for i in range(p.n_in)]
    evks = {r: ctx_toy.keygen_rot(SK, EK, r) for r in p.rots}
    pts = p.encode_weights(synth.conv_weight(16, 4, 4, 3), level, bias=synth.conv_bias(17, 4), bias_scale=2**40)
    want = p.run(evks, cts, level, pts)[0]
    total = p.partial_state(level)
    for b_, e_ in [(0, 4), (4, 9)]:
        st = p.partial_state(level)
        p.raconv_partial(evks, cts, level, pts, 0, b_, e_, st)
        total += st
    assert np.array_equal(to_np(p.raconv_finish(evks, level, pts, total, 0)), to_np(want))


@pytest.mark.parametrize("idx", [3, 4, 5], ids=["ra21", "ca_g2", "dsconv"])
def test_toy_layers_limited_keyset_bit_exact(ctx_toy, orc_toy, idx):
    """a limited rotation-key set (DESIGN R-KEYSET): the Slide amounts plus {1, 3 W_p, 7}; every
    RaS / RaS_g / IR_g / combine amount is synthesized as a chain of loaded rotations -- bit-exact vs the oracle's
    composition (the same BFS decomposition), and decrypting to conv2d within 2^-10"""
    import paper_2302_02407_b200 as hy
    spec, level = TOY[idx], orc_toy.nq - 1
    X = synth.image(18, spec.ci, spec.w)
    K = synth.conv_weight(19, spec.co, spec.ci, spec.f)
    plan = H.plan_caconv(spec, K) if spec.algo == "CA" else H.plan_raconv(spec, K)
    amounts = [r % spec.n for r in plan.taps if r % spec.n] + [1, 3 * spec.wp, 7]
    p = hy.ConvPlan(ctx_toy, spec.ci, spec.co, spec.w, spec.f, spec.s, spec.wp, spec.g, spec.m, spec.d, spec.algo)
    p.set_keyset(hy.KeySet(12, amounts))
    ks = H.KeySet(spec.n, amounts)
    assert sum(p.eff_counts.values()) > sum(p.counts.values())   # something is synthesized
    fin = H.Fmt("CA" if spec.algo == "CA" else "RA", spec.n, spec.wp, spec.g, spec.m, spec.d)
    cts = [ctx_toy.encrypt(SK, 904, i, ctx_toy.encode(v, 2**40, level), level) for i, v in enumerate(H.pack(X, fin))]
    outs = p.run({r: ctx_toy.keygen_rot(SK, EK, r) for r in p.rots}, cts, level, p.encode_weights(K, level))
    o = orc_toy
    octs = [o.encrypt(SK, 904, i, o.encode(v, 2**40, level)) for i, v in enumerate(H.pack(X, plan.fin))]
    oevks = {r: o.keygen_rot(SK, EK, r) for r in H.keyset_amounts(plan, ks)}
    ref = H.EncConv(o, plan, oevks, keyset=ks).run(octs)
    for a, r in zip(outs, ref):
        assert np.array_equal(to_np(a), r.data)
    dec = [np.real(o.decode(o.decrypt(SK, r))) for r in ref]
    got = H.unpack(dec, plan.fout, spec.co, spec.wo, spec.wo)
    want = H.conv2d(X, K, spec.s)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 2 ** -10


def test_resnet20_layer_positive_power_keyset(ctx_hyp, orc_hyp):
    """ResNet-20 stage-2 CAConv at N = 2^16 with the Slide keys + positive powers of two loaded: the negative IR_g
    amounts are synthesized; a sampled output bit-exact vs the oracle"""
    import paper_2302_02407_b200 as hy
    spec, level, j = R20["L2_ca"], 9, 1
    K = synth.conv_weight(24, spec.co, spec.ci, spec.f)
    plan = H.plan_caconv(spec, K)
    amounts = [r % spec.n for r in plan.taps if r % spec.n] + [1 << i for i in range(15)]
    p = hy.ConvPlan(ctx_hyp, spec.ci, spec.co, spec.w, spec.f, spec.s, spec.wp, spec.g, spec.m, spec.d, spec.algo)
    p.set_keyset(hy.KeySet(16, amounts))
    ks = H.KeySet(spec.n, amounts)
    assert p.eff_counts["IR_g"] > p.counts["IR_g"]
    X = synth.image(25, spec.ci, spec.w)
    fin = H.Fmt("CA", spec.n, spec.wp, spec.g, spec.m, spec.d)
    cts = [ctx_hyp.encrypt(SK, 905, i, ctx_hyp.encode(v, 2**42, level), level) for i, v in enumerate(H.pack(X, fin))]
    out = p.run({r: ctx_hyp.keygen_rot(SK, EK, r) for r in p.rots}, cts, level, p.encode_weights(K, level),
                out_begin=j, out_end=j + 1)[0]
    o = orc_hyp
    octs = [o.encrypt(SK, 905, i, o.encode(v, 2**42, level)) for i, v in enumerate(H.pack(X, plan.fin))]
    oevks = {r: o.keygen_rot(SK, EK, r) for r in H.keyset_amounts(plan, ks)}
    ref = H.EncConv(o, plan, oevks, keyset=ks).run(octs, [j])[0]
    assert np.array_equal(to_np(out), ref.data)
