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
