"""Pins of the bootstrapping linear steps in the oracle (oracle/boot.py, partial), CPU only:
ModRaise decrypts to m + q_0 I with a small integer polynomial I (big-int check); the BSGS linear transform decrypts
to the plaintext matrix-vector product M z; the special-FFT matrix is the encoder's embedding (decode of a known
coefficient vector), and CoeffToSlot / SlotToCoeff built from it move coefficients to slots and back."""
import numpy as np
import pytest

import oracle
import synth
from oracle import boot as B

SK, EK = synth.SEED_SK, synth.SEED_EVK


@pytest.fixture(scope="module")
def mini():
    return oracle.Oracle(**synth.PARAMS["mini"])


def test_special_fft_matrix_is_the_embedding(mini):
    o = mini
    V = B.special_fft_matrix(o.N)
    g = np.random.default_rng(3)
    m = g.integers(-1000, 1000, o.N)
    pt = oracle.Pt(o.coeffs_to_pt(m, o.nq - 1), o.nq - 1, 1.0)
    z = o.decode(pt)
    u = m[: o.n] + 1j * m[o.n:]
    assert np.max(np.abs(V @ u - z)) < 1e-9 * np.max(np.abs(z))


def test_mod_raise(mini):
    o = mini
    z = synth.slots_uniform(5, o.n)
    ct0 = o.level_down(o.encrypt(SK, 7, 0, o.encode(z, 2**40, o.nq - 1)), 0)
    up = B.mod_raise(o, ct0, o.nq - 1)
    m0 = o.crt_coeffs(o.decrypt(SK, ct0).data, 0)
    m1 = o.crt_coeffs(o.decrypt(SK, up).data, o.nq - 1)
    q0 = int(o.q[0])
    I = [(b - a) // q0 for a, b in zip(m0, m1)]
    assert all((b - a) % q0 == 0 for a, b in zip(m0, m1))
    assert max(abs(x) for x in I) <= (o.h + 1) // 2 + 1


def _rand_diag_matrix(n, ds, seed):
    g = np.random.default_rng(seed)
    M = np.zeros((n, n), complex)
    j = np.arange(n)
    for d in ds:
        M[j, (j + d) % n] = g.uniform(-1, 1, n) + 1j * g.uniform(-1, 1, n)
    return M


def test_lintrans_is_matrix_product(mini):
    o = mini
    n = o.n
    ds = [0, 1, 2, 5, 7, 9, n - 1, n - 8, 64]
    M = _rand_diag_matrix(n, ds, 11)
    bs = 4
    dsc = sorted(d % n for d in ds)
    diags = dict(zip(dsc, B.diagonals(M, dsc)))
    need = sorted({d % bs for d in dsc if d % bs} | {(d // bs) * bs for d in dsc if d // bs})
    evks = {r: o.keygen_rot(SK, EK, r) for r in need}
    z = synth.slots_uniform(12, n) + 1j * synth.slots_uniform(13, n)
    lv = o.nq - 1
    ct = o.encrypt(SK, 8, 0, o.encode(z, 2**40, lv))
    y = B.lintrans(o, ct, diags, bs, evks)
    assert y.level == lv - 1 and abs(y.scale - 2**40) < 1e-3
    got = o.decode(o.decrypt(SK, y))
    want = M @ z
    assert np.max(np.abs(got - want)) < 2**-18 * np.max(np.abs(want))


def test_coeff_to_slot_and_back(mini):
    """CoeffToSlot = V^{-1} on the slots (dense, n diagonals, bs = 32): the slots become the complex-packed
    coefficients / scale; SlotToCoeff = V brings the slots back"""
    o = mini
    n = o.n
    V = B.special_fft_matrix(o.N)
    Vi = np.linalg.inv(V)
    ds = list(range(n))
    bs = 32
    need = sorted({d % bs for d in ds if d % bs} | {(d // bs) * bs for d in ds if d // bs})
    evks = {r: o.keygen_rot(SK, EK, r) for r in need}
    z = synth.slots_uniform(14, n)
    lv = o.nq - 1
    pt = o.encode(z, 2**40, lv)
    ct = o.encrypt(SK, 9, 0, pt)
    c2s = B.lintrans(o, ct, dict(zip(ds, B.diagonals(Vi, ds))), bs, evks)
    m = np.array(o.crt_coeffs(pt.data, lv), dtype=float)
    u = (m[:n] + 1j * m[n:]) / 2**40
    got = o.decode(o.decrypt(SK, c2s))
    assert np.max(np.abs(got - u)) < 2**-20 * max(1.0, np.max(np.abs(u)))
    s2c = B.lintrans(o, c2s, dict(zip(ds, B.diagonals(V, ds))), bs, evks)
    back = o.decode(o.decrypt(SK, s2c))
    assert np.max(np.abs(back - z)) < 2**-15


@pytest.mark.slow
def test_oracle_bootstrap_recovers_slots():
    """DESIGN R-EVALMOD end to end on the oracle ('boot' chain, N = 2^10): a level-0 ciphertext bootstrapped to a
    higher level decrypts to the same slots within 2^-10 of max|z|, and every EvalMod stage matches its plaintext
    function (the scaled sine of t / (Delta K))"""
    import math
    o = oracle.Oracle(**synth.PARAMS["boot"])
    n, N, top = o.n, o.N, o.nq - 1
    r, a, bs = 3, 8.0, 32
    K = float(o.q[0]) / 2**40
    V = B.special_fft_matrix(N)
    ds = list(range(n))
    cheb = np.polynomial.chebyshev.chebinterpolate(lambda s: np.cos(a * s), 30)
    cheb[1::2] = 0.0
    need = sorted({d % bs for d in ds if d % bs} | {(d // bs) * bs for d in ds if d // bs})
    evks = {rr: o.keygen_rot(SK, EK, rr) for rr in need}
    z = synth.slots_uniform(41, n)
    ct0 = o.level_down(o.encrypt(SK, 12, 0, o.encode(z, 2**40, top)), 0)
    out = B.bootstrap(o, ct0, top, dict(zip(ds, B.diagonals(np.linalg.inv(V) / 2, ds))),
                      dict(zip(ds, B.diagonals(K / (2 * math.pi) * V, ds))), bs, cheb, r, a, evks,
                      o.keygen_galois(SK, EK, 2 * N - 1), o.keygen_relin(SK, EK))
    assert out.level >= 1
    got = o.decode(o.decrypt(SK, out))
    assert np.max(np.abs(got - z)) < 2**-10 * np.max(np.abs(z))


def _dense(D, n):
    M = np.zeros((n, n), complex)
    j = np.arange(n)
    for d, v in D.items():
        M[j, (j + d) % n] += v
    return M


@pytest.mark.parametrize("N,groups", [(16, [1, 2]), (64, [2, 3]), (256, [3, 2, 2]), (1024, [3, 3, 3]), (1024, [4, 5])])
def test_sfft_levels_factorise_the_embedding(N, groups):
    """DESIGN R-SFFT pinned to the plain definition: the levels of the forward factorisation, applied in order to a
    bit-reversed vector, multiply to V P (V = special_fft_matrix, itself pinned to the embedding above; P the bit
    reversal); the inverse levels multiply to P V^{-1}; each level has the diagonal count of its stages' offsets"""
    n = N // 2
    V = B.special_fft_matrix(N)
    P = np.eye(n)[B.bit_reverse_perm(n)]
    fwd = B.sfft_levels(N, groups)
    inv = B.sfft_levels(N, groups, inverse=True, scale=0.5)
    Mf, Mi = np.eye(n), np.eye(n)
    for D in fwd:
        Mf = _dense(D, n) @ Mf
    for D in inv:
        Mi = _dense(D, n) @ Mi
    assert np.abs(Mf - V @ P).max() < 1e-12
    assert np.abs(Mi - 0.5 * P @ np.linalg.inv(V)).max() < 1e-12
    at = 0
    for g, D in zip(groups, fwd):
        offs = {(m << at) % n for m in range(-(2 ** g - 1), 2 ** g)}
        assert set(D) == offs
        at += g


def test_bit_reverse_perm():
    assert list(B.bit_reverse_perm(8)) == [0, 4, 2, 6, 1, 5, 3, 7]
    assert list(B.bit_reverse_perm(1)) == [0]


def test_diag_mul_is_matmul():
    """the product of two matrices given by their diagonals equals dense matmul (random diagonals, wrap-around)"""
    n = 16
    rng = np.random.default_rng(5)
    A = {d: rng.normal(size=n) + 1j * rng.normal(size=n) for d in (0, 1, 5, 15)}
    Bm = {d: rng.normal(size=n) + 1j * rng.normal(size=n) for d in (0, 3, 14)}
    assert np.abs(_dense(B.diag_mul(A, Bm, n), n) - _dense(A, n) @ _dense(Bm, n)).max() < 1e-12


def test_product_sfft_levels_match_oracle():
    """the product's own (vectorised) factorisation gives the oracle's diagonals to the last bit, so bench.py (which
    may not import oracle/) times the transforms the parity tests check"""
    from paper_2302_02407_b200 import boot as PB
    for N, groups in ((64, [2, 3]), (1024, [4, 5]), (4096, [4, 4, 3])):
        for inv in (False, True):
            a = B.sfft_levels(N, groups, inv, 0.5)
            b = PB.sfft_levels(N, groups, inv, 0.5)
            for x, y in zip(a, b):
                assert sorted(x) == sorted(y)
                for d in x:
                    assert np.array_equal(x[d], y[d])


def test_oracle_bootstrap_factorised_recovers_slots():
    """the whole bootstrap with the factorised transforms (2 CoeffToSlot + 2 SlotToCoeff levels, DESIGN R-SFFT) on
    the 'boot' chain decrypts to the input slots within 2^-10 of max|z|"""
    import math
    o = oracle.Oracle(**synth.PARAMS["boot"])
    N, top = o.N, o.nq - 1
    r, a = 3, 8.0
    K = float(o.q[0]) / 2**40
    cts = B.sfft_levels(N, [4, 5], inverse=True, scale=0.5)
    stc = B.sfft_levels(N, [4, 5], scale=K / (2 * math.pi))
    bsc = [8 * min((d & -d) for d in D if d) for D in cts]
    bss = [8 * min((d & -d) for d in D if d) for D in stc]
    cheb = np.polynomial.chebyshev.chebinterpolate(lambda s: np.cos(a * s), 30)
    cheb[1::2] = 0.0
    need = set()
    for D, bs in list(zip(cts, bsc)) + list(zip(stc, bss)):
        need |= {d % bs for d in D if d % bs} | {(d // bs) * bs for d in D if d // bs}
    evks = {rr: o.keygen_rot(SK, EK, rr) for rr in sorted(need)}
    z = synth.slots_uniform(41, o.n)
    ct0 = o.level_down(o.encrypt(SK, 12, 0, o.encode(z, 2**40, top)), 0)
    out = B.bootstrap(o, ct0, top, cts, stc, (bsc, bss), cheb, r, a, evks, o.keygen_galois(SK, EK, 2 * N - 1),
                      o.keygen_relin(SK, EK))
    assert out.level == top - 14
    got = o.decode(o.decrypt(SK, out))
    assert np.max(np.abs(got - z)) < 2**-10 * np.max(np.abs(z))
