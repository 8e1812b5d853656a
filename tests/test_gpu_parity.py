"""GPU parity: every RNS-CKKS step of the CUDA path vs the CPU oracle, bit-exact
on every limb, through the C ABI (paper_2302_02407_b200 binding)."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

SK = synth.SEED_SK
EK = synth.SEED_EVK


def to_np(t):
    return t.detach().cpu().numpy().view(np.uint64)


def to_dev(a, ctx):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).to(ctx.device)


def evk_dev(e, ctx):
    """an oracle key (one uint64 per word) -> the library's packed device key"""
    return ctx.evk_pack(to_dev(e, ctx))


@pytest.fixture(scope="module", params=["toy", "mini", "hyp"])
def pair(request):
    import paper_2302_02407_b200 as hy
    prm = synth.PARAMS[request.param]
    return request.param, hy.Context(**prm), oracle.Oracle(**prm)


def rand_limbs(o, seed, chain):
    g = np.random.default_rng(seed)
    return np.stack([g.integers(0, int(o.moduli[t]), o.N, dtype=np.uint64) for t in chain])


def test_moduli(pair):
    _, ctx, o = pair
    assert ctx.moduli == [int(x) for x in o.moduli]
    assert ctx.alpha == o.alpha


def test_ntt_forward_inverse(pair):
    _, ctx, o = pair
    chain = list(range(o.nq + o.np_))
    a = rand_limbs(o, 1, chain)
    A = to_np(ctx.ntt(to_dev(a, ctx), chain))
    want = np.stack([o.ntt(a[t], t) for t in chain])
    assert np.array_equal(A, want)
    back = to_np(ctx.ntt(to_dev(A, ctx), chain, inverse=True))
    assert np.array_equal(back, a)
    # ragged batch with repeated primes
    ch2 = [0, 0, chain[-1], 1]
    b = rand_limbs(o, 2, ch2)
    assert np.array_equal(to_np(ctx.ntt(to_dev(b, ctx), ch2)), np.stack([o.ntt(b[i], t) for i, t in enumerate(ch2)]))


def test_automorph(pair):
    _, ctx, o = pair
    chain = [0, 1]
    a = rand_limbs(o, 3, chain)
    for r in [1, 5, -1, o.n - 3]:
        k = o.galois_elt(r)
        assert ctx.galois_elt(r) == k
        A = np.stack([o.ntt(a[t], t) for t in chain])
        got = to_np(ctx.automorph(to_dev(A, ctx), k))
        want = np.stack([o.ntt(o.automorph_coeff(a[t], t, k), t) for t in chain])
        assert np.array_equal(got, want)


def test_keygen(pair):
    name, ctx, o = pair
    for r in ([1, -7] if name != "hyp" else [3]):
        k = ctx.keygen_rot(SK, EK, r)
        want = o.keygen_rot(SK, EK, r)
        assert np.array_equal(to_np(ctx.evk_unpack(k)), want)
        # packed layout: 6 bytes per word, 3/4 of the unpacked size, equal to packing the oracle's key
        assert k.numel() * 8 == want.nbytes // 4 * 3 == ctx.evk_bytes()
        assert np.array_equal(to_np(k), to_np(evk_dev(want, ctx)))


def test_encode_encrypt_decrypt(pair):
    name, ctx, o = pair
    level = o.nq - 1 if name != "hyp" else 9
    z = synth.slots_uniform(30, o.n)
    scale = 2 ** synth.PARAMS[name]["log_scale"]
    pt = ctx.encode(z, scale, level)
    opt = o.encode(z, scale, level)
    assert np.array_equal(to_np(pt), opt.data)
    ct = ctx.encrypt(SK, 41, 7, pt, level)
    oct_ = o.encrypt(SK, 41, 7, opt)
    assert np.array_equal(to_np(ct), oct_.data)
    dec = ctx.decrypt(SK, ct, level)
    assert np.array_equal(to_np(dec), o.decrypt(SK, oct_).data)


def test_decode(pair):
    """hy_decode (device iNTT + centred CRT + special FFT) vs the oracle's big-int CRT + FFT decode of the same
    limbs (a float result: tolerance), and decode(decrypt(encrypt(encode z))) = z within the encryption noise."""
    name, ctx, o = pair
    level = o.nq - 1 if name != "hyp" else 3
    z = synth.slots_uniform(31, o.n)
    scale = 2 ** synth.PARAMS[name]["log_scale"]
    ct = ctx.encrypt(SK, 41, 8, ctx.encode(z, scale, level), level)
    dec = ctx.decrypt(SK, ct, level)
    got = ctx.decode(dec, level, scale)
    want = o.decode(oracle.Pt(to_np(dec), level, float(scale)))
    assert np.max(np.abs(got - want)) < 1e-9
    assert np.max(np.abs(got - z)) < 2**-20
    assert np.array_equal(ctx.decode(dec, level, scale, n_slots=5), got[:5])


def test_modup_ip_moddown(pair):
    name, ctx, o = pair
    for level in sorted({o.nq - 1, 0, min(5, o.nq - 1)}):
        d = rand_limbs(o, 10 + level, list(range(level + 1)))
        ext = ctx.modup(level, to_dev(d, ctx))
        oext = o.modup_coeff(level, d)
        assert np.array_equal(to_np(ext), oext)
        evk = o.keygen_rot(SK, EK, 1) if name != "hyp" else None
        if evk is not None:
            u = ctx.ks_inner_product(level, ext, evk_dev(evk, ctx))
            ou = o.ks_inner_product(level, oext, evk)
            assert np.array_equal(to_np(u), ou)
        chain = o.ext_chain(level)
        uu = rand_limbs(o, 20 + level, chain)
        assert np.array_equal(to_np(ctx.moddown(level, to_dev(uu, ctx))), o.moddown(level, uu))


def _fresh_ct(ctx, o, name, level, seed):
    z = synth.slots_uniform(seed, o.n)
    scale = 2 ** synth.PARAMS[name]["log_scale"]
    opt = o.encode(z, scale, level)
    oct_ = o.encrypt(SK, 50, seed, opt)
    return to_dev(oct_.data, ctx), oct_


def test_hrot_plain_and_batch(pair):
    name, ctx, o = pair
    level = o.nq - 1
    rs = [1, -1, 9] if name != "hyp" else [5]
    evks = [o.keygen_rot(SK, EK, r) for r in rs]
    d_evks = [evk_dev(e, ctx) for e in evks]
    cts = [_fresh_ct(ctx, o, name, level, 60 + i) for i in range(len(rs))]
    for (dct, oct_), r, e, de in zip(cts, rs, evks, d_evks):
        got = to_np(ctx.hrot(de, dct, level, r))
        assert np.array_equal(got, o.hrot(oct_, e, r).data), r
    outs = ctx.hrot_batch(d_evks, [c[0] for c in cts], level, rs)
    for out, (dct, oct_), r, e in zip(outs, cts, rs, evks):
        assert np.array_equal(to_np(out), o.hrot(oct_, e, r).data)
    # r = 0 and r = n are copies
    assert np.array_equal(to_np(ctx.hrot(d_evks[0], cts[0][0], level, 0)), cts[0][1].data)
    assert np.array_equal(to_np(ctx.hrot(d_evks[0], cts[0][0], level, o.n)), cts[0][1].data)


def test_hrot_hoisted(pair):
    name, ctx, o = pair
    level = o.nq - 1 if name != "hyp" else 9
    rs = [1, 0, -1, 8] if name != "hyp" else [1, 32, -64]
    evks = [o.keygen_rot(SK, EK, r) if o.galois_elt(r) != 1 else None for r in rs]
    dct, oct_ = _fresh_ct(ctx, o, name, level, 70)
    d_evks = [evk_dev(e, ctx) if e is not None else None for e in evks]
    outs = ctx.hrot_hoisted(d_evks, dct, level, rs)
    oo = o.hrot_hoisted(oct_, [e if e is not None else np.zeros(1, np.uint64) for e in evks], rs)
    for a, b in zip(outs, oo):
        assert np.array_equal(to_np(a), b.data)


def test_hrot_sum(pair):
    name, ctx, o = pair
    level = o.nq - 1 if name != "hyp" else 6
    rs = [1, 0, -1, 7] if name != "hyp" else [1, 0, -9]
    evks = [o.keygen_rot(SK, EK, r) if o.galois_elt(r) != 1 else None for r in rs]
    cts = [_fresh_ct(ctx, o, name, level, 80 + i) for i in range(len(rs))]
    got = ctx.hrot_sum([evk_dev(e, ctx) if e is not None else None for e in evks], [c[0] for c in cts], level, rs)
    want = o.hrot_sum([c[1] for c in cts], evks, rs)
    assert np.array_equal(to_np(got), want.data)


def test_pmult_add_rescale(pair):
    name, ctx, o = pair
    level = o.nq - 1 if name != "hyp" else 9
    a = rand_limbs(o, 90, list(range(level + 1)) * 2).reshape(2, level + 1, o.N)
    b = rand_limbs(o, 91, list(range(level + 1)) * 2).reshape(2, level + 1, o.N)
    pts = [rand_limbs(o, 92 + i, list(range(level + 1))) for i in range(3)]
    A, B = oracle.Ct(a, level, 1.0), oracle.Ct(b, level, 1.0)
    da, db = to_dev(a, ctx), to_dev(b, ctx)
    dp = [to_dev(p, ctx) for p in pts]
    assert np.array_equal(to_np(ctx.add(da, db, level)), o.add(A, B).data)
    assert np.array_equal(to_np(ctx.pmult(da, dp[0], level)), o.pmult(A, oracle.Pt(pts[0], level, 1.0)).data)
    acc = ctx.pmult_acc([da, db, da], dp, level)
    want = o.add(o.add(o.pmult(A, oracle.Pt(pts[0], level, 1.0)), o.pmult(B, oracle.Pt(pts[1], level, 1.0))),
                 o.pmult(A, oracle.Pt(pts[2], level, 1.0)))
    assert np.array_equal(to_np(acc), want.data)
    assert np.array_equal(to_np(ctx.rescale(da, level)), o.rescale(A).data)


def test_relin_key_and_mulct(pair):
    """Relinearization key and MulCt (+ relinearization, no rescale) bit-exact vs the oracle, including the
    square (a = b, output aliasing the input) and a batch sharing the key; the rescaled square decodes to z^2."""
    name, ctx, o = pair
    level = o.nq - 1 if name != "hyp" else 9
    rlk = ctx.keygen_relin(SK, EK)
    orlk = o.keygen_relin(SK, EK)
    assert np.array_equal(to_np(ctx.evk_unpack(rlk)), orlk)
    scale = 2 ** synth.PARAMS[name]["log_scale"]
    za, zb = synth.slots_uniform(60, o.n), synth.slots_uniform(61, o.n)
    pa, pb = o.encode(za, scale, level), o.encode(zb, scale, level)
    oa, ob = o.encrypt(SK, 62, 0, pa), o.encrypt(SK, 62, 1, pb)
    a, b = to_dev(oa.data, ctx), to_dev(ob.data, ctx)
    want = o.mulct(oa, ob, orlk)
    assert np.array_equal(to_np(ctx.mulct(rlk, a, b, level)), want.data)
    # batch of squares, in place
    cts = [a.clone(), b.clone(), a.clone()]
    outs = ctx.square_batch(rlk, cts, level, outs=cts)
    wsq = [o.mulct(x, x, orlk) for x in (oa, ob, oa)]
    for g, w in zip(outs, wsq):
        assert np.array_equal(to_np(g), w.data)
    sq = o.rescale(wsq[0])
    zs = np.real(o.decode(o.decrypt(SK, sq)))
    assert np.max(np.abs(zs - za * za)) < 2**-15
    # hy_decode of the unrescaled square: coefficients ~ scale^2, far beyond q_0 (multi-limb centred CRT)
    sq_dec = ctx.decrypt(SK, outs[0], level)
    zq = ctx.decode(sq_dec, level, float(scale) ** 2)
    assert np.max(np.abs(np.real(zq) - za * za)) < 2**-15


@pytest.mark.parametrize("level", [23, 9])
def test_hrot_hoisted_chunked(level):
    """Hoisted batch longer than the workspace's key-switch batch (4 -> chunks of 4 and 1 sharing one ModUp):
    bit-exact vs the oracle at both conv and full level."""
    import paper_2302_02407_b200 as hy
    prm = synth.PARAMS["hyp"]
    ctx, o = hy.Context(**prm, max_batch=4), oracle.Oracle(**prm)
    rs = [1, 2, -3, 7, 100]
    evks = [o.keygen_rot(SK, EK, r) for r in rs]
    dct, oct_ = _fresh_ct(ctx, o, "hyp", level, 71)
    outs = ctx.hrot_hoisted([evk_dev(e, ctx) for e in evks], dct, level, rs)
    oo = o.hrot_hoisted(oct_, evks, rs)
    for a, b in zip(outs, oo):
        assert np.array_equal(to_np(a), b.data)


def test_encode_batch_device(pair):
    """Batched device encoding (hy_encode_batch: double-double special FFT on the GPU) = the oracle's encoder
    (binary128 DFT), bit-exact, for random, sparse weight-like, 0/1-mask and zero slot vectors, at a power-of-two
    and a prime scale."""
    name, ctx, o = pair
    level = o.nq - 1 if name != "hyp" else 9
    g = np.random.default_rng(77)
    z = np.zeros((5, o.n))
    z[0] = synth.slots_uniform(32, o.n)
    z[1, g.choice(o.n, o.n // 16, replace=False)] = g.normal(0, 0.1, o.n // 16)  # sparse, weight-like
    z[2, ::4] = 1.0                                                               # mask
    z[3, : o.n // 3] = synth.slots_uniform(33, o.n // 3)
    for scale in (2 ** synth.PARAMS[name]["log_scale"], o.q[level]):
        got = to_np(ctx.encode_batch(z, scale, level))
        for i in range(len(z)):
            assert np.array_equal(got[i], o.encode(z[i], scale, level).data), (scale, i)


@pytest.mark.parametrize("level", [1, 2, 9, 23])
def test_rescale_fused_levels(level):
    """Rescale at N = 2^16 runs as a centred ModDown by q_l (inverse row pass, fused column kernel, row kernel with
    the epilogue): bit-exact vs the oracle's big-int-pinned rescale at the lowest, conv and full levels, on random
    residues (both centring branches taken); the conv-layer tests cover the batched calls."""
    ctx, o = _hyp_pair()
    cts = [rand_limbs(o, 300 + level * 10 + k, list(range(level + 1)) * 2).reshape(2, level + 1, o.N)
           for k in range(3)]
    for a in cts:
        assert np.array_equal(to_np(ctx.rescale(to_dev(a, ctx), level)), o.rescale(oracle.Ct(a, level, 1.0)).data)


def test_rescale_batch_and_mulct_batch():
    """hy_rescale_batch, hy_pmult_batch and hy_mulct_batch (bootstrapping's lockstep EvalMod): every item bit-exact vs
    the oracle's rescale / PMult / MulCt of that item; an output aliasing another item's input is rejected (HY_E_ARG)"""
    import paper_2302_02407_b200 as hy
    ctx, o = _hyp_pair()
    level = 9
    cts = [rand_limbs(o, 700 + k, list(range(level + 1)) * 2).reshape(2, level + 1, o.N) for k in range(5)]
    outs = ctx.rescale_batch([to_dev(a, ctx) for a in cts], level)
    for a, got in zip(cts, outs):
        assert np.array_equal(to_np(got), o.rescale(oracle.Ct(a, level, 1.0)).data)
    d = [to_dev(a, ctx) for a in cts[:2]]
    with pytest.raises(hy.HyError):
        ctx.rescale_batch(d, level, outs=[d[1][:, :level].contiguous(), d[0]])
    pt = rand_limbs(o, 799, list(range(level + 1)))
    pm = ctx.pmult_batch([to_dev(a, ctx) for a in cts], to_dev(pt, ctx), level)
    for a, got in zip(cts, pm):
        assert np.array_equal(to_np(got), o.pmult(oracle.Ct(a, level, 1.0), oracle.Pt(pt, level, 1.0)).data)
    with pytest.raises(hy.HyError):
        ctx.pmult_batch(d, to_dev(pt, ctx), level, outs=[d[1], d[1].clone()])
    rlk, orlk = ctx.keygen_relin(SK, EK), o.keygen_relin(SK, EK)
    z = [synth.slots_uniform(80 + k, o.n) for k in range(3)]
    ocs = [o.encrypt(SK, 4, 40 + k, o.encode(z[k], 2**42, level)) for k in range(3)]
    dcs = [to_dev(c.data, ctx) for c in ocs]
    got = ctx.mulct_batch(rlk, [dcs[0], dcs[1], dcs[2]], [dcs[1], dcs[1], dcs[0]], level)
    for g, (x, y) in zip(got, [(0, 1), (1, 1), (2, 0)]):
        assert np.array_equal(to_np(g), o.mulct(ocs[x], ocs[y], orlk).data)


_HYP = {}


def _hyp_pair():
    if not _HYP:
        import paper_2302_02407_b200 as hy
        prm = synth.PARAMS["hyp"]
        _HYP["p"] = (hy.Context(**prm), oracle.Oracle(**prm))
    return _HYP["p"]


def test_pack48_wire_format():
    """hy_pack48 / hy_unpack48: word x at bytes [6x, 6x+6) little-endian (checked against a numpy byte view),
    round trip exact, and the packed keys use the same layout."""
    ctx, o = _hyp_pair()
    level = 3
    a = rand_limbs(o, 5, list(range(level + 1)) * 2).reshape(2, level + 1, o.N)
    d = to_dev(a, ctx)
    packed = to_np(ctx.pack48(d))
    want = a.reshape(-1).view(np.uint8).reshape(-1, 8)[:, :6].reshape(-1)
    assert np.array_equal(packed.view(np.uint8), want)
    back = ctx.unpack48(ctx.pack48(d), ctx.empty(*d.shape))
    assert np.array_equal(to_np(back), a)
    k = ctx.keygen_rot(SK, EK, 3)
    assert np.array_equal(to_np(ctx.pack48(ctx.evk_unpack(k))), to_np(k).reshape(-1))


def test_bench_configuration_sampled():
    """The C2 bench workload in the bench's launch configuration (workspace for 64 key switches per launch, level
    23): 66 plain rotations r_i = i + 1 (a full chunk of 64 and a ragged chunk of 2) and 70 hoisted rotations of one
    ciphertext; sampled outputs bit-exact vs the oracle (device keys, themselves bit-exact with the oracle's)."""
    import paper_2302_02407_b200 as hy
    prm = synth.PARAMS["hyp"]
    _, o = _hyp_pair()
    ctx = hy.Context(**prm, max_batch=64)
    level = 23
    n_rot = 66
    rs = [i + 1 for i in range(n_rot)]
    keys = [ctx.keygen_rot(SK, EK, r) for r in rs]
    cts = [_fresh_ct(ctx, o, "hyp", level, 400 + i) for i in range(n_rot)]
    outs = ctx.hrot_batch(keys, [c[0] for c in cts], level, rs)
    for i in (0, 33, 63, 65):
        okey = to_np(ctx.evk_unpack(keys[i])).reshape(o.dnum, 2, o.nq + o.np_, o.N)
        assert np.array_equal(to_np(outs[i]), o.hrot(cts[i][1], okey, rs[i]).data), i
    hrs = [i + 1 for i in range(70)]
    hkeys = keys + [ctx.keygen_rot(SK, EK, r) for r in hrs[n_rot:]]
    hout = ctx.hrot_hoisted(hkeys, cts[0][0], level, hrs)
    sample = (0, 63, 69)
    okeys = [to_np(ctx.evk_unpack(hkeys[i])).reshape(o.dnum, 2, o.nq + o.np_, o.N) for i in sample]
    want = o.hrot_hoisted(cts[0][1], okeys, [hrs[i] for i in sample])
    for i, w in zip(sample, want):
        assert np.array_equal(to_np(hout[i]), w.data), i


def test_level_down(pair):
    """level_down keeps the first l'+1 limbs of both polynomials (reduction mod Q_l'), decrypts to the same
    message, and refuses to raise the level."""
    import paper_2302_02407_b200 as hy
    name, ctx, o = pair
    level = o.nq - 1 if name != "hyp" else 9
    a = rand_limbs(o, 95, list(range(level + 1)) * 2).reshape(2, level + 1, o.N)
    for nl in (level, level - 1, 0):
        got = to_np(ctx.level_down(to_dev(a, ctx), level, nl))
        assert np.array_equal(got, a[:, : nl + 1])
    z = synth.slots_uniform(34, o.n)
    scale = 2 ** synth.PARAMS[name]["log_scale"]
    ct = ctx.encrypt(SK, 41, 9, ctx.encode(z, scale, level), level)
    low = ctx.level_down(ct, level, 1)
    assert np.max(np.abs(np.real(ctx.decode(ctx.decrypt(SK, low, 1), 1, scale)) - z)) < 2**-20
    with pytest.raises(hy.HyError):
        ctx.level_down(low, 1, 2)


def test_error_paths():
    """Status codes at the C ABI (include/hyphen.h): checked on the host before any launch."""
    import ctypes as C

    import paper_2302_02407_b200 as hy
    ctx, o = _hyp_pair()
    L = hy.lib()
    level = 3
    ct = ctx.empty(*ctx.ct_shape(level))
    ct.zero_()
    key = ctx.keygen_rot(SK, EK, 1)

    def code(fn):
        with pytest.raises(hy.HyError) as e:
            fn()
        return e.value.code

    assert code(lambda: ctx.rescale(ctx.empty(*ctx.ct_shape(0)), 0, out=ctx.empty(*ctx.ct_shape(0)))) == 3  # EXHAUSTED
    assert code(lambda: ctx.hrot(key, ct, level, 1, out=ct)) == 1                       # in place: ARG
    assert code(lambda: ctx.hrot(key, ct, o.nq, 1)) == 1                                # level out of range: ARG
    assert code(lambda: ctx.decode(ct[0], level, 2.0**42, n_slots=o.N)) == 5            # > N/2 slots: CAPACITY
    assert code(lambda: ctx.pack48(ctx.empty(6))) == 1                                  # not a multiple of 4: ARG
    assert code(lambda: ctx.level_down(ct, level, level + 1)) == 2                      # raise: LEVEL_MISMATCH
    # a rotation without its key: MISSING_KEY
    outs = (C.c_void_p * 1)(ctx.empty(*ctx.ct_shape(level)).data_ptr())
    keys = (C.c_void_p * 1)(0)
    cts = (C.c_void_p * 1)(ct.data_ptr())
    rs = (C.c_int32 * 1)(5)
    rc = L.hy_hrot_batch(ctx._c, keys, cts, level, rs, 1, outs, ctx._stream())
    assert rc == 8, L.hy_last_error()
    # r = 0 needs no key; an empty batch is a no-op
    assert L.hy_hrot_batch(ctx._c, keys, cts, level, (C.c_int32 * 1)(0), 1, outs, ctx._stream()) == 0
    assert L.hy_hrot_batch(ctx._c, keys, cts, level, rs, 0, outs, ctx._stream()) == 0


def test_hrot_sum_long_batch():
    """Lazy HRotSum over 66 ciphertexts with a 64-item workspace (one full SUM launch of 64 items, whose running
    FP64 sums are re-centred every 32 items, and a ragged chunk of 2): bit-exact vs the oracle."""
    import paper_2302_02407_b200 as hy
    prm = synth.PARAMS["hyp"]
    _, o = _hyp_pair()
    ctx = hy.Context(**prm, max_batch=64)
    level, n = 2, 66
    rs = [1] * n
    okey = o.keygen_rot(SK, EK, 1)
    key = evk_dev(okey, ctx)
    cts = [_fresh_ct(ctx, o, "hyp", level, 500 + i) for i in range(n)]
    got = ctx.hrot_sum([key] * n, [c[0] for c in cts], level, rs)
    want = o.hrot_sum([c[1] for c in cts], [okey] * n, rs)
    assert np.array_equal(to_np(got), want.data)


@pytest.mark.parametrize("level", [0, 1, 5, 12, 23])
def test_hrot_random_levels(level):
    """Plain batch, hoisted and lazy-sum HRot at levels from 0 (one limb, one digit of one limb) to the full chain,
    with random rotation amounts of both signs (including |r| > n/2): bit-exact vs the oracle."""
    ctx, o = _hyp_pair()
    g = np.random.default_rng(1000 + level)
    rs = [int(x) for x in g.integers(1, o.n, 3) * g.choice([-1, 1], 3)]
    okeys = [o.keygen_rot(SK, EK, r) for r in rs]
    keys = [evk_dev(k, ctx) for k in okeys]
    cts = [_fresh_ct(ctx, o, "hyp", level, 600 + 10 * level + i) for i in range(3)]
    outs = ctx.hrot_batch(keys, [c[0] for c in cts], level, rs)
    for out, (dct, oct_), r, k in zip(outs, cts, rs, okeys):
        assert np.array_equal(to_np(out), o.hrot(oct_, k, r).data), (level, r)
    hout = ctx.hrot_hoisted(keys, cts[0][0], level, rs)
    for a, b in zip(hout, o.hrot_hoisted(cts[0][1], okeys, rs)):
        assert np.array_equal(to_np(a), b.data), level
    s = ctx.hrot_sum(keys, [c[0] for c in cts], level, rs)
    assert np.array_equal(to_np(s), o.hrot_sum([c[1] for c in cts], okeys, rs).data), level


def test_prot(pair):
    """PRot = the oracle's coefficient-domain automorphism of the plaintext (the EncConv reference), bit-exact;
    decodes to the left-rotated slots; r = 0 copies."""
    name, ctx, o = pair
    level = min(2, o.nq - 1)
    z = synth.slots_uniform(35, o.n)
    scale = 2 ** synth.PARAMS[name]["log_scale"]
    pt = ctx.encode(z, scale, level)
    opt = to_np(pt)
    for r in (0, 1, -3, o.n // 2 + 5):
        got = to_np(ctx.prot(pt, level, r))
        k = o.galois_elt(r)
        want = np.stack([o.ntt(o.automorph_coeff(o.intt(opt[i], i), i, k), i) for i in range(level + 1)]) \
            if r % o.n else opt
        assert np.array_equal(got, want), r
    zr = np.real(ctx.decode(ctx.prot(pt, level, 3), level, scale))
    assert np.max(np.abs(zr - np.roll(z, -3))) < 2**-20


def test_add_pt_and_scale_check(pair):
    """hy_add_pt: (c0 + pt, c1) bit-exact vs the oracle's AddPt, in place and out of place; mismatched scales are
    HY_E_SCALE_MISMATCH (12)"""
    import paper_2302_02407_b200 as hy
    name, ctx, o = pair
    level = o.nq - 1 if name != "hyp" else 5
    a = rand_limbs(o, 110, list(range(level + 1)) * 2).reshape(2, level + 1, o.N)
    p = rand_limbs(o, 111, list(range(level + 1)))
    want = o.add_pt(oracle.Ct(a, level, 2.0**40), oracle.Pt(p, level, 2.0**40)).data
    da, dp = to_dev(a, ctx), to_dev(p, ctx)
    assert np.array_equal(to_np(ctx.add_pt(da, 2.0**40, dp, 2.0**40, level)), want)
    ctx.add_pt(da, 2.0**40, dp, 2.0**40, level, out=da)
    assert np.array_equal(to_np(da), want)
    with pytest.raises(hy.HyError) as e:
        ctx.add_pt(da, 2.0**40, dp, 2.0**41, level)
    assert e.value.code == 12


def test_coeff_wire_format_and_sizes(pair):
    """hy_export_coeff / hy_import_coeff (coefficient domain, limbs q_0.. then p_0..) = the oracle's
    iNTT / NTT, round trip exact; hy_ct_bytes / hy_pt_bytes; unreduced imports are HY_E_ARG"""
    import paper_2302_02407_b200 as hy
    name, ctx, o = pair
    chain = list(range(o.nq)) + list(range(o.nq, o.nq + o.np_))
    a = rand_limbs(o, 120, chain)
    coeff = ctx.export_coeff(to_dev(a, ctx), chain)
    assert np.array_equal(coeff, np.stack([o.intt(a[i], t) for i, t in enumerate(chain)]))
    back = ctx.import_coeff(coeff, chain)
    assert np.array_equal(to_np(back), a)
    bad = coeff.copy()
    bad[0, 0] = int(o.moduli[0])
    with pytest.raises(hy.HyError) as e:
        ctx.import_coeff(bad, chain)
    assert e.value.code == 1
    lv = min(3, o.nq - 1)
    assert ctx.ct_bytes(lv) == 2 * (lv + 1) * o.N * 8
    assert ctx.pt_bytes(lv) == (lv + 1) * o.N * 8 and ctx.pt_bytes(lv, True) == (lv + 1 + o.np_) * o.N * 8
    assert ctx.ct_bytes(o.nq) == 0


def test_ctx_and_batch_argument_checks():
    """K < alpha special primes is HY_E_ARG at context creation; an hrot_batch output overlapping
    another item's input is HY_E_ARG"""
    import paper_2302_02407_b200 as hy
    prm = dict(synth.PARAMS["mini"])
    prm["p_bits"] = [48]          # alpha = 2 > K = 1
    with pytest.raises(hy.HyError) as e:
        hy.Context(**prm)
    assert e.value.code == 1
    ctx, o = _hyp_pair()
    level = 2
    key = ctx.keygen_rot(SK, EK, 1)
    a, b = ctx.zeros(*ctx.ct_shape(level)), ctx.zeros(*ctx.ct_shape(level))
    with pytest.raises(hy.HyError) as e:
        ctx.hrot_batch([key, key], [a, b], level, [1, 1], outs=[b, ctx.empty(*ctx.ct_shape(level))])
    assert e.value.code == 1
