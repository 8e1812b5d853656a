"""Encrypted HyPHEN layers on the CPU oracle: decrypt(conv(enc x)) vs conv2d within
2^-10 relative error (BASELINE north_star), at the toy parameter set (N = 2^12)."""
import numpy as np
import pytest

import oracle
import synth
from oracle import hyphen as H

SK, EK = synth.SEED_SK, synth.SEED_EVK


def run_encrypted(o, spec, seed, level):
    X = synth.image(seed, spec.ci, spec.w)
    K = synth.conv_weight(seed + 1, spec.co, spec.ci, spec.f)
    plan = H.plan_caconv(spec, K) if spec.algo == "CA" else H.plan_raconv(spec, K)
    scale = 2 ** 40
    cts = [o.encrypt(SK, 900, i, o.encode(v, scale, level)) for i, v in enumerate(H.pack(X, plan.fin))]
    evks = {r: o.keygen_rot(SK, EK, r) for r in H.rotation_amounts(plan, o.n)}
    outs = H.EncConv(o, plan, evks).run(cts)
    dec = [np.real(o.decode(o.decrypt(SK, c))) for c in outs]
    got = H.unpack(dec, plan.fout, spec.co, spec.wo, spec.wo)
    want = H.conv2d(X, K, spec.s)
    return got, want, outs, plan


@pytest.mark.parametrize("spec", [
    H.ConvSpec(4, 4, 8, 3, 1, 8, 1, 1, 1, "RA", n=2048),   # BASELINE config 1
    H.ConvSpec(4, 4, 8, 3, 1, 8, 1, 1, 1, "CA", n=2048),
    H.ConvSpec(8, 8, 8, 3, 1, 8, 1, 1, 2, "CA", n=2048),   # R_g = 2 (e = 2)
    H.ConvSpec(8, 8, 8, 3, 1, 8, 1, 2, 1, "RA", n=2048),   # RaS_g + IR_g over R_g
    H.ConvSpec(8, 8, 4, 3, 1, 8, 2, 2, 4, "CA", n=2048),   # gap 2: RaS_g + mask + IR_g over C_g
    H.ConvSpec(4, 8, 8, 3, 2, 8, 1, 1, 2, "CA", n=2048),   # dsconv: gap 1 -> 2
    H.ConvSpec(64, 8, 6, 3, 1, 8, 1, 1, 1, "CA", n=2048, S=2),   # PRCR CAConv (full family)
    H.ConvSpec(8, 64, 6, 3, 1, 8, 1, 1, 1, "RA", n=2048, S=2),   # PRCR RAConv
], ids=["C1_raconv", "caconv_11", "caconv_12", "raconv_21", "caconv_g2", "dsconv", "prcr_ca", "prcr_ra"])
def test_encrypted_conv_matches_conv2d(orc_toy, spec):
    o = orc_toy
    got, want, outs, plan = run_encrypted(o, spec, 5, o.nq - 1)
    err = np.max(np.abs(got - want)) / np.max(np.abs(want))
    assert err < 2 ** -10, err
    used = 1 + (1 if plan.mask is not None else 0)
    assert outs[0].level == o.nq - 1 - used
    assert all(abs(c.scale - 2 ** 40) < 1e-6 * 2 ** 40 for c in outs)


def test_encrypted_block_mini():
    """Alg. 3 block (CAConv -> MulCt square + relinearization + rescale -> RAConv) on encrypted data at the mini
    parameter set: decrypts to conv2d(conv2d(X, K1)^2, K2) within 2^-10 relative (north star)."""
    o = oracle.Oracle(**synth.PARAMS["mini"])
    n = o.n
    ca_s = H.ConvSpec(4, 4, 4, 3, 1, 4, 1, 1, 2, "CA", n=n)
    ra_s = H.ConvSpec(4, 4, 4, 3, 1, 4, 1, 2, 1, "RA", n=n)
    X = synth.image(70, 4, 4)
    K1 = synth.conv_weight(71, 4, 4, 3)
    K2 = synth.conv_weight(72, 4, 4, 3)
    ca, ra = H.plan_caconv(ca_s, K1), H.plan_raconv(ra_s, K2)
    level = o.nq - 1
    cts = [o.encrypt(synth.SEED_SK, 73, i, o.encode(v, 2**40, level)) for i, v in enumerate(H.pack(X, ca.fin))]
    ek = {r: o.keygen_rot(synth.SEED_SK, synth.SEED_EVK, r) for r in H.rotation_amounts(ca, n)}
    rk = {r: o.keygen_rot(synth.SEED_SK, synth.SEED_EVK, r) for r in H.rotation_amounts(ra, n)}
    rlk = o.keygen_relin(synth.SEED_SK, synth.SEED_EVK)
    outs = H.run_block_encrypted(o, ca, ra, ek, rk, rlk, cts)
    dec = [np.real(o.decode(o.decrypt(synth.SEED_SK, c))) for c in outs]
    got = H.unpack(dec, ra.fout, 4, 4, 4)
    want = H.conv2d(H.conv2d(X, K1) ** 2, K2)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 2**-10


# ---------------------------------------------------------------------------------------------------------------
# Pins of the oracle's conv2d (the reference every layer test decrypts against), VERDICT r01 "weak" 1.
def test_conv2d_matches_torch():
    """oracle conv2d = torch.nn.functional.conv2d (cross-correlation, zero padding (f-1)/2, stride s, bias): an
    independent implementation, f in {1, 3}, s in {1, 2}, even and odd image sizes, several channel counts."""
    import torch
    import torch.nn.functional as F
    g = np.random.default_rng(17)
    for ci, co, w, f, s in [(1, 1, 4, 3, 2), (3, 16, 32, 3, 1), (16, 32, 32, 3, 2), (16, 32, 32, 1, 2),
                            (4, 4, 7, 3, 2), (8, 4, 5, 3, 1), (2, 3, 9, 1, 1), (5, 2, 6, 5, 1)]:
        X = g.uniform(-1, 1, (ci, w, w))
        K = g.normal(0, 1, (co, ci, f, f))
        b = g.uniform(-1, 1, co)
        want = F.conv2d(torch.from_numpy(X)[None], torch.from_numpy(K), torch.from_numpy(b), stride=s,
                        padding=(f - 1) // 2)[0].numpy()
        got = H.conv2d(X, K, s, bias=b)
        assert got.shape == want.shape
        assert np.max(np.abs(got - want)) < 1e-12


def _golden_fig2d():
    import os
    taps, pos = {}, {}
    path = os.path.join(os.path.dirname(__file__), "golden", "fig2d_stride2.txt")
    for line in open(path):
        line = line.split("#")[0].split()
        if not line:
            continue
        if line[0] == "pos":
            for it in line[1:]:
                o, rc = it.split(":")
                pos[o] = tuple(int(x) for x in rc.split(","))
        else:
            taps[line[0]] = [tuple(it.split(":")) for it in line[1:]]
    return taps, pos


def test_conv2d_fig2d_stride2_worked_example():
    """Fig. 2(d): with one-hot image a_i and one-hot filter k_t, the stride-2 pad-1 conv2d output is
    one-hot at exactly the output the figure pairs (k_t, a_i) with, and zero where the figure's filter slot is 0;
    outputs c1..c4 are the even grid positions, i.e. Y[row/2, col/2]."""
    taps, pos = _golden_fig2d()
    for k, pairs in taps.items():
        t = int(k[1:]) - 1
        K = np.zeros((1, 1, 3, 3))
        K[0, 0, t // 3, t % 3] = 1.0
        listed = {}
        for o, a in pairs:
            listed[a] = o
        for i in range(16):
            X = np.zeros((1, 4, 4))
            X[0, i // 4, i % 4] = 1.0
            Y = H.conv2d(X, K, 2)[0]
            assert Y.shape == (2, 2)
            want = np.zeros((2, 2))
            if f"a{i + 1}" in listed:
                r, c = pos[listed[f"a{i + 1}"]]
                assert r % 2 == 0 and c % 2 == 0
                want[r // 2, c // 2] = 1.0
            # outputs the figure shows for this tap hold only the listed inputs
            for o, (r, c) in pos.items():
                if o in listed.values() and f"a{i + 1}" not in listed:
                    assert Y[r // 2, c // 2] == 0.0
            if f"a{i + 1}" in listed:
                assert np.array_equal(Y, want), (k, i)
    # and every output position of the figure receives k1 only from a6 (the rest reads the padding)
    K = np.zeros((1, 1, 3, 3))
    K[0, 0, 0, 0] = 1.0
    X = np.arange(1, 17, dtype=float).reshape(1, 4, 4)
    assert np.array_equal(H.conv2d(X, K, 2)[0], np.array([[0.0, 0.0], [0.0, 6.0]]))


@pytest.mark.parametrize("spec", [H.ConvSpec(4, 4, 8, 3, 1, 8, 1, 1, 1, "RA", n=2048),
                                  H.ConvSpec(4, 8, 8, 3, 2, 8, 1, 1, 2, "CA", n=2048)], ids=["C1_raconv", "dsconv"])
def test_encrypted_conv_with_bias(orc_toy, spec):
    """AddPt of the bias plaintexts after the layer (DESIGN R-BIAS): decrypts to conv2d(X, K) + b within 2^-10"""
    o = orc_toy
    level = o.nq - 1
    X = synth.image(8, spec.ci, spec.w)
    K = synth.conv_weight(9, spec.co, spec.ci, spec.f)
    b = synth.conv_bias(10, spec.co)
    plan = H.plan_caconv(spec, K) if spec.algo == "CA" else H.plan_raconv(spec, K)
    cts = [o.encrypt(SK, 900, i, o.encode(v, 2**40, level)) for i, v in enumerate(H.pack(X, plan.fin))]
    evks = {r: o.keygen_rot(SK, EK, r) for r in H.rotation_amounts(plan, o.n)}
    outs = H.EncConv(o, plan, evks, bias=b).run(cts)
    dec = [np.real(o.decode(o.decrypt(SK, c))) for c in outs]
    got = H.unpack(dec, plan.fout, spec.co, spec.wo, spec.wo)
    want = H.conv2d(X, K, spec.s, bias=b)
    assert np.max(np.abs(got - want)) / np.max(np.abs(want)) < 2 ** -10
