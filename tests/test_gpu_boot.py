"""GPU parity of the bootstrapping linear steps (partial; DESIGN R-LINTRANS): complex encoding,
ModRaise and the BSGS diagonal linear transform through the C ABI, bit-exact on every limb against oracle/boot.py,
and CoeffToSlot / SlotToCoeff (dense special-FFT matrices) moving coefficients to slots and back."""
import numpy as np
import pytest

import oracle
import synth
from oracle import boot as B

pytestmark = pytest.mark.gpu
SK, EK = synth.SEED_SK, synth.SEED_EVK


def to_np(t):
    return t.detach().cpu().numpy().view(np.uint64)


def to_dev(a, ctx):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(ctx.device)


_P = {}


def pair(name):
    if name not in _P:
        import paper_2302_02407_b200 as hy
        prm = synth.PARAMS[name]
        _P[name] = (hy.Context(**prm), oracle.Oracle(**prm))
    return _P[name]


@pytest.mark.parametrize("name", ["mini", "toy", "hyp"])
def test_encode_complex(name):
    ctx, o = pair(name)
    z = synth.slots_uniform(1, o.n) + 1j * synth.slots_uniform(2, o.n)
    lv = min(3, o.nq - 1)
    for scale in (2**40, int(o.q[lv])):
        assert np.array_equal(to_np(ctx.encode_complex(z, scale, lv)), o.encode(z, scale, lv).data)


@pytest.mark.parametrize("name", ["mini", "toy", "hyp"])
def test_mod_raise(name):
    ctx, o = pair(name)
    top = o.nq - 1
    z = synth.slots_uniform(3, o.n)
    ct0 = o.level_down(o.encrypt(SK, 7, 1, o.encode(z, 2**40, top)), 0)
    got = to_np(ctx.mod_raise(to_dev(ct0.data, ctx), top))
    assert np.array_equal(got, B.mod_raise(o, ct0, top).data)


def _lintrans_case(ctx, o, ds, bs, seed, level):
    import paper_2302_02407_b200 as hy
    n = o.n
    g = np.random.default_rng(seed)
    dsc = sorted({d % n for d in ds})
    vals = [g.uniform(-1, 1, n) + 1j * g.uniform(-1, 1, n) for _ in dsc]
    lt = hy.LinTrans(ctx, dsc, bs)
    keys = {r: ctx.keygen_rot(SK, EK, r) for r in lt.rots}
    okeys = {r: o.keygen_rot(SK, EK, r) for r in lt.rots}
    z = synth.slots_uniform(seed, n) + 1j * synth.slots_uniform(seed + 1, n)
    oct_ = o.encrypt(SK, 9, seed, o.encode(z, 2**40, level))
    y = lt.apply(keys, to_dev(oct_.data, ctx), level, lt.encode(vals, level))
    want = B.lintrans(o, oct_, dict(zip(dsc, vals)), bs, okeys)
    assert np.array_equal(to_np(y), want.data)
    return lt, want, z, dict(zip(dsc, vals))


@pytest.mark.parametrize("name,ds,bs", [("mini", [0, 1, 3, 9, -1, 64], 4), ("toy", [0, 2, 5, 33, -7, 100, 1023], 8),
                                        ("hyp", [0, 1, 2, 3, 8, 16, -8], 4)])
def test_lintrans_bit_exact(name, ds, bs):
    ctx, o = pair(name)
    lv = o.nq - 1 if name != "hyp" else 9
    lt, want, z, diags = _lintrans_case(ctx, o, ds, bs, 20, lv)
    # and it is the matrix-vector product on the slots
    n = o.n
    j = np.arange(n)
    ref = sum(v * z[(j + d) % n] for d, v in diags.items())
    got = o.decode(o.decrypt(SK, want))
    assert np.max(np.abs(got - ref)) < 2**-18 * np.max(np.abs(ref))


def test_coeff_to_slot_to_coeff_mini():
    """ModRaise of a level-0 ciphertext, CoeffToSlot (V^{-1}, 512 diagonals, bs = 32) and SlotToCoeff (V): bit-exact
    vs the oracle; CoeffToSlot's slots are the raised plaintext's complex-packed coefficients / scale and
    SlotToCoeff returns the raised slots"""
    import paper_2302_02407_b200 as hy
    ctx, o = pair("mini")
    n, top = o.n, o.nq - 1
    V = B.special_fft_matrix(o.N)
    Vi = np.linalg.inv(V)
    ds = list(range(n))
    z = synth.slots_uniform(30, n) * 0.01
    ct0 = o.level_down(o.encrypt(SK, 7, 2, o.encode(z, 2**40, top)), 0)
    up = B.mod_raise(o, ct0, top)
    d_up = ctx.mod_raise(to_dev(ct0.data, ctx), top)
    assert np.array_equal(to_np(d_up), up.data)
    c2s = hy.LinTrans(ctx, ds, 32)
    keys = {r: ctx.keygen_rot(SK, EK, r) for r in c2s.rots}
    okeys = {r: o.keygen_rot(SK, EK, r) for r in c2s.rots}
    y = c2s.apply(keys, d_up, top, c2s.encode(B.diagonals(Vi, ds), top))
    oy = B.lintrans(o, up, dict(zip(ds, B.diagonals(Vi, ds))), 32, okeys)
    assert np.array_equal(to_np(y), oy.data)
    m = np.array(o.crt_coeffs(o.decrypt(SK, up).data, top), dtype=float)
    u = (m[:n] + 1j * m[n:]) / 2**40
    assert np.max(np.abs(o.decode(o.decrypt(SK, oy)) - u)) < 2**-20 * np.max(np.abs(u))
    s2c = hy.LinTrans(ctx, ds, 32)
    w = s2c.apply(keys, y, top - 1, s2c.encode(B.diagonals(V, ds), top - 1))
    ow = B.lintrans(o, oy, dict(zip(ds, B.diagonals(V, ds))), 32, okeys)
    assert np.array_equal(to_np(w), ow.data)
    back = o.decode(o.decrypt(SK, ow))
    assert np.max(np.abs(back - o.decode(o.decrypt(SK, up)))) < 2**-12


def test_bootstrap_small_ring():
    """The whole bootstrapping (DESIGN R-EVALMOD) on the 'boot' chain (N = 2^10, 17 limbs): ModRaise, CoeffToSlot,
    conjugation split, EvalMod (Chebyshev degree 30 of cos(8 s), 3 double angles), recombination, SlotToCoeff --
    every intermediate and the result bit-exact vs oracle/boot.py, and the result decrypts to the input slots within
    2^-10 of max|z|"""
    import math

    import paper_2302_02407_b200 as hy
    from paper_2302_02407_b200.boot import Bootstrapper
    ctx, o = pair("boot")
    n, N, top = o.n, o.N, o.nq - 1
    r, a, bs = 3, 8.0, 32
    K = float(o.q[0]) / 2**40
    V = B.special_fft_matrix(N)
    ds = list(range(n))
    cts_d = B.diagonals(np.linalg.inv(V) / 2, ds)
    stc_d = B.diagonals(K / (2 * math.pi) * V, ds)
    cheb = np.polynomial.chebyshev.chebinterpolate(lambda s: np.cos(a * s), 30)
    cheb[1::2] = 0.0
    lt = hy.LinTrans(ctx, ds, bs)
    keys = {rr: ctx.keygen_rot(SK, EK, rr) for rr in lt.rots}
    okeys = {rr: o.keygen_rot(SK, EK, rr) for rr in lt.rots}
    conj, oconj = ctx.keygen_galois(SK, EK, 2 * N - 1), o.keygen_galois(SK, EK, 2 * N - 1)
    rlk, orlk = ctx.keygen_relin(SK, EK), o.keygen_relin(SK, EK)
    z = synth.slots_uniform(40, n)
    ct0 = o.level_down(o.encrypt(SK, 11, 0, o.encode(z, 2**40, top)), 0)
    bt = Bootstrapper(ctx, cts_d, stc_d, bs, cheb, r, a, keys, conj, rlk)
    got = bt.bootstrap(to_dev(ct0.data, ctx), 2.0**40, top)
    want = B.bootstrap(o, ct0, top, dict(zip(ds, cts_d)), dict(zip(ds, stc_d)), bs, cheb, r, a, okeys, oconj, orlk)
    assert got.level == want.level and got.scale == want.scale
    assert np.array_equal(to_np(got.t), want.data)
    dz = o.decode(o.decrypt(SK, want))
    assert np.max(np.abs(dz - z)) < 2**-10 * np.max(np.abs(z))


def _factorised(N, groups, K):
    import math
    cts = B.sfft_levels(N, groups, inverse=True, scale=0.5)
    stc = B.sfft_levels(N, groups, scale=K / (2 * math.pi))
    bsc = [8 * min((d & -d) for d in D if d) for D in cts]
    bss = [8 * min((d & -d) for d in D if d) for D in stc]
    return cts, stc, (bsc, bss)


def _cheb(a):
    cheb = np.polynomial.chebyshev.chebinterpolate(lambda s: np.cos(a * s), 30)
    cheb[1::2] = 0.0
    return cheb


def test_bootstrap_small_ring_factorised():
    """The whole bootstrap with the factorised special FFT (DESIGN R-SFFT: CoeffToSlot and SlotToCoeff as 2 levels of
    radix-2 butterfly stages each, slots bit-reversed in between) on the 'boot' chain (N = 2^10): every limb of the
    result bit-exact vs oracle/boot.py, and the result decrypts to the input slots within 2^-10 of max|z|"""
    from paper_2302_02407_b200.boot import Bootstrapper, transform_rots
    ctx, o = pair("boot")
    N, top = o.N, o.nq - 1
    r, a = 3, 8.0
    cts, stc, bs = _factorised(N, [4, 5], float(o.q[0]) / 2**40)
    rots = sorted(set(transform_rots(ctx, cts, bs[0])) | set(transform_rots(ctx, stc, bs[1])))
    keys = {rr: ctx.keygen_rot(SK, EK, rr) for rr in rots}
    okeys = {rr: o.keygen_rot(SK, EK, rr) for rr in rots}
    conj, oconj = ctx.keygen_galois(SK, EK, 2 * N - 1), o.keygen_galois(SK, EK, 2 * N - 1)
    rlk, orlk = ctx.keygen_relin(SK, EK), o.keygen_relin(SK, EK)
    z = synth.slots_uniform(42, o.n)
    ct0 = o.level_down(o.encrypt(SK, 13, 0, o.encode(z, 2**40, top)), 0)
    bt = Bootstrapper(ctx, cts, stc, bs, _cheb(a), r, a, keys, conj, rlk)
    assert bt.rots == rots
    got = bt.bootstrap(to_dev(ct0.data, ctx), 2.0**40, top)
    want = B.bootstrap(o, ct0, top, cts, stc, bs, _cheb(a), r, a, okeys, oconj, orlk)
    assert got.level == want.level == top - 14 and got.scale == want.scale
    assert np.array_equal(to_np(got.t), want.data)
    dz = o.decode(o.decrypt(SK, want))
    assert np.max(np.abs(dz - z)) < 2**-10 * np.max(np.abs(z))


def test_bootstrap_set_hyp():
    """Bootstrapping at Set_hyp (N = 2^16, L+1 = 24, h = 192): ModRaise, CoeffToSlot as 3
    factorised levels (32/63/63 diagonals), EvalMod (cos(12 s), degree 30, 4 double angles: ~30 periods for h = 192),
    SlotToCoeff as 3 levels -- 17 levels, ending at L' = 6, with the transforms' 38 rotation keys, one
    conjugation and one relinearisation key (48 + 2).  Every limb of the result bit-exact vs oracle/boot.py
    (the oracle's part takes ~2 minutes), and it decrypts to the input slots within 2^-9 of max|z|."""
    from paper_2302_02407_b200.boot import Bootstrapper, transform_rots
    ctx, o = pair("hyp")
    N, top = o.N, o.nq - 1
    r, a = 4, 12.0
    cts, stc, bs = _factorised(N, [5, 5, 5], float(o.q[0]) / 2**42)
    rots = sorted(set(transform_rots(ctx, cts, bs[0])) | set(transform_rots(ctx, stc, bs[1])))
    keys = {rr: ctx.keygen_rot(SK, EK, rr) for rr in rots}
    okeys = {rr: o.keygen_rot(SK, EK, rr) for rr in rots}
    conj, oconj = ctx.keygen_galois(SK, EK, 2 * N - 1), o.keygen_galois(SK, EK, 2 * N - 1)
    rlk, orlk = ctx.keygen_relin(SK, EK), o.keygen_relin(SK, EK)
    z = synth.slots_uniform(44, o.n)
    ct0 = o.level_down(o.encrypt(SK, 15, 0, o.encode(z, 2**42, top)), 0)
    got = Bootstrapper(ctx, cts, stc, bs, _cheb(a), r, a, keys, conj, rlk).bootstrap(to_dev(ct0.data, ctx), 2.0**42,
                                                                                     top)
    want = B.bootstrap(o, ct0, top, cts, stc, bs, _cheb(a), r, a, okeys, oconj, orlk)
    assert got.level == want.level == 6 and got.scale == want.scale
    assert np.array_equal(to_np(got.t), want.data)
    dz = o.decode(o.decrypt(SK, want))
    assert np.max(np.abs(dz - z)) < 2**-9 * np.max(np.abs(z))


def test_block_chain_set_hyp():
    """Bootstrapping chaining conv blocks end to end at Set_hyp: ResNet-20 stage-1 shapes (16
    channels, 32 x 32, CA(1,2) -> RA(2,1) -> CA(1,2)), y = RAConv(CAConv(x)^2) + x at L' = 6 -> level 3, bootstrap back
    to L' (BlockChain.refresh), a second block; the result decrypts to the plaintext recursion
    Y1 = conv(conv(X, K1)^2, K2) + X, Y2 = conv(conv(Y1, K3)^2, K4) + Y1 within 2^-8 of max|Y2|."""
    import paper_2302_02407_b200 as hy
    from oracle import hyphen as H
    from paper_2302_02407_b200.boot import CT, BlockChain, Bootstrapper, transform_rots
    ctx, o = pair("hyp")
    N, n, top = o.N, o.n, o.nq - 1
    cts, stc, bs = _factorised(N, [5, 5, 5], float(o.q[0]) / 2**42)
    rots = sorted(set(transform_rots(ctx, cts, bs[0])) | set(transform_rots(ctx, stc, bs[1])))
    rlk = ctx.keygen_relin(SK, EK)
    bt = Bootstrapper(ctx, cts, stc, bs, _cheb(12.0), 4, 12.0, {r: ctx.keygen_rot(SK, EK, r) for r in rots},
                      ctx.keygen_galois(SK, EK, 2 * N - 1), rlk)
    ca_s = H.ConvSpec(16, 16, 32, 3, 1, 32, 1, 1, 2, "CA", n=n)
    ra_s = H.ConvSpec(16, 16, 32, 3, 1, 32, 1, 2, 1, "RA", n=n)
    X = synth.image(90, 16, 32)
    Ks = [synth.conv_weight(91 + i, 16, 16, 3) * 0.3 for i in range(4)]
    fin = H.plan_caconv(ca_s, Ks[0]).fin
    fout = H.plan_raconv(ra_s, Ks[1]).fout
    assert fin == fout  # the block's output format is its input's: the shortcut adds slot by slot
    g_ca = hy.ConvPlan(ctx, 16, 16, 32, 3, 1, 32, 1, 1, 2, "CA")
    g_ra = hy.ConvPlan(ctx, 16, 16, 32, 3, 1, 32, 1, 2, 1, "RA")
    blk = hy.ConvBlock(ctx, g_ca, g_ra)
    L = 6
    _, ra_level, out_level = blk.levels(L)
    ca_keys = {r: ctx.keygen_rot(SK, EK, r) for r in g_ca.rots}
    ra_keys = {r: ctx.keygen_rot(SK, EK, r) for r in g_ra.rots}
    xs = H.pack(X, fin)
    assert len(xs) == 1
    chain = BlockChain(ctx, bt)
    x = CT(ctx.encrypt(SK, 31, 0, ctx.encode(xs[0], 2**42, L), L), L, 2.0**42)
    x = chain.block(blk, ca_keys, ra_keys, g_ca.encode_weights(Ks[0], L), g_ra.encode_weights(Ks[1], ra_level), x)
    assert x.level == out_level
    x = chain.refresh(x)
    assert x.level == L
    x = chain.block(blk, ca_keys, ra_keys, g_ca.encode_weights(Ks[2], L), g_ra.encode_weights(Ks[3], ra_level), x)
    dec = np.real(ctx.decode(ctx.decrypt(SK, x.t, x.level), x.level, x.scale))
    res = H.unpack([dec], fout, 16, 32, 32)
    Y1 = H.conv2d(H.conv2d(X, Ks[0]) ** 2, Ks[1]) + X
    Y2 = H.conv2d(H.conv2d(Y1, Ks[2]) ** 2, Ks[3]) + Y1
    assert np.max(np.abs(res - Y2)) < 2**-8 * np.max(np.abs(Y2))


def test_resnet20_convs_end_to_end():
    """The ResNet-20 conv stack end to end under encryption at Set_hyp (boot.ResNet20Convs: stem + square, 9 blocks
    y = RAConv(CAConv(x)^2) + s(x) with dsconv / pconv at the stage boundaries, a bootstrap after each of the first 8
    blocks): the 64 x 8 x 8 result decrypts to the plaintext network (oracle conv2d) within 2^-7 of its max."""
    import paper_2302_02407_b200 as hy
    from oracle import hyphen as H
    from paper_2302_02407_b200.boot import CT, BlockChain, Bootstrapper, ResNet20Convs, transform_rots
    ctx, o = pair("hyp")
    N, n = o.N, o.n
    cts, stc, bs = _factorised(N, [5, 5, 5], float(o.q[0]) / 2**42)
    rots = sorted(set(transform_rots(ctx, cts, bs[0])) | set(transform_rots(ctx, stc, bs[1])))
    bt = Bootstrapper(ctx, cts, stc, bs, _cheb(12.0), 4, 12.0, {r: ctx.keygen_rot(SK, EK, r) for r in rots},
                      ctx.keygen_galois(SK, EK, 2 * N - 1), ctx.keygen_relin(SK, EK))
    shapes = [((16, 3), 3)] + [((16, 16), 3)] * 6 + [((32, 16), 3), ((32, 32), 3), ((32, 16), 1)] + \
        [((32, 32), 3)] * 4 + [((64, 32), 3), ((64, 64), 3), ((64, 32), 1)] + [((64, 64), 3)] * 4
    Ws = [synth.conv_weight(200 + i, co, ci, f) * (0.5) for i, ((co, ci), f) in enumerate(shapes)]
    net = ResNet20Convs(ctx, BlockChain(ctx, bt), Ws, lambda r: ctx.keygen_rot(SK, EK, r))
    X = synth.image(300, 3, 32)
    spec = ResNet20Convs.SPECS
    fin = H.plan_caconv(H.ConvSpec(*spec["stem"], n=n), Ws[0]).fin
    xs = H.pack(X, fin)
    assert len(xs) == 1
    L = net.input_level
    y = net.run(CT(ctx.encrypt(SK, 32, 0, ctx.encode(xs[0], 2**42, L), L), L, 2.0**42))
    fout = H.plan_raconv(H.ConvSpec(*spec["s3_ra"], n=n), Ws[-1]).fout
    res = H.unpack([np.real(ctx.decode(ctx.decrypt(SK, y.t, y.level), y.level, y.scale))], fout, 64, 8, 8)
    it = iter(Ws)
    Y = H.conv2d(X, next(it)) ** 2
    for ca, ra, sc in ResNet20Convs.BLOCKS:
        Kc, Kr = next(it), next(it)
        stride = spec[ca][4]
        main = H.conv2d(H.conv2d(Y, Kc, stride) ** 2, Kr)
        Y = main + (H.conv2d(Y, next(it), 2) if sc else Y)
    assert res.shape == Y.shape
    assert np.max(np.abs(res - Y)) < 2**-7 * np.max(np.abs(Y))
