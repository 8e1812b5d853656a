"""Pins of the CPU oracle against things other than itself (CPU only).

Every test here checks oracle/ against a published value, a closed form, an
independent library (sympy / mpmath / Python big ints) or brute force.
"""
import math
import os

import mpmath
import numpy as np
import pytest
import sympy

import oracle
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _centre(v, Q):
    v %= Q
    return v - Q if v > Q // 2 else v


# ---------------------------------------------------------------- Philox
def test_philox_kat():
    rows = [l.split() for l in open(os.path.join(GOLD, "philox4x32_10_kat.txt")) if l.strip() and not l.startswith("#")]
    assert len(rows) == 3
    for r in rows:
        v = [int(x, 16) for x in r]
        out = oracle.philox4x32_10(v[4:6], v[0:4])
        assert [int(x) for x in out] == v[6:10]


# ---------------------------------------------------------------- primes / roots
@pytest.mark.parametrize("pset", ["toy", "mini", "hyp"])
def test_primes(pset):
    prm = synth.PARAMS[pset]
    o = oracle.Oracle(**prm)
    N = o.N
    bits = prm["q_bits"] + prm["p_bits"]
    mods = [int(x) for x in o.moduli]
    assert len(set(mods)) == len(mods)
    for i, (q, b) in enumerate(zip(mods, bits)):
        assert sympy.isprime(q)
        assert q % (2 * N) == 1
        assert q < 2 ** b
        # largest unused such prime below 2^b (DESIGN R-PRIMES)
        x = q + 2 * N
        while x < 2 ** b:
            assert not (sympy.isprime(x) and x not in mods[:i]), (pset, i, x)
            x += 2 * N
        # psi: primitive 2N-th root, smallest such
        psi = int(o.psi[i])
        assert pow(psi, N, q) == q - 1
        assert pow(psi, 2 * N, q) == 1
    # smallest primitive root: brute force on the toy set
    if pset == "toy":
        for i, q in enumerate(mods):
            psi = int(o.psi[i])
            roots = {pow(psi, e, q) for e in range(1, 2 * N, 2)}
            assert psi == min(roots)


def test_is_prime_vs_sympy():
    rng = np.random.default_rng(7)
    for _ in range(300):
        n = int(rng.integers(2, 2**62)) | 1
        assert oracle.is_prime(n) == sympy.isprime(n)
    for n in [2, 3, 4, 561, 1105, 2**61 - 1, 3215031751, 3825123056546413051]:
        assert oracle.is_prime(n) == sympy.isprime(n)


# ---------------------------------------------------------------- NTT
@pytest.fixture(scope="module")
def orc_tiny():
    return oracle.Oracle(log_n=5, q_bits=[40, 40], p_bits=[40], dnum=2, h=8)


def _br(x, bits):
    return int(format(x, f"0{bits}b")[::-1], 2)


def test_ntt_direct_evaluation(orc_tiny):
    o = orc_tiny
    rng = np.random.default_rng(1)
    for t, q in enumerate(o.moduli):
        q = int(q)
        a = rng.integers(0, q, size=o.N, dtype=np.uint64)
        A = o.ntt(a, t)
        psi = int(o.psi[t])
        for k in range(o.N):
            e = 2 * _br(k, o.log_n) + 1
            want = sum(int(a[i]) * pow(psi, e * i, q) for i in range(o.N)) % q
            assert int(A[k]) == want


def test_ntt_schoolbook_product(orc_mini):
    o = orc_mini
    rng = np.random.default_rng(2)
    N = o.N
    for t in [0, 3, o.nq]:
        q = int(o.moduli[t])
        a = rng.integers(0, q, size=N, dtype=np.uint64)
        b = rng.integers(0, q, size=N, dtype=np.uint64)
        c = o.intt((o.ntt(a, t).astype(object) * o.ntt(b, t).astype(object) % q).astype(np.uint64), t)
        # schoolbook negacyclic product, vectorised over one operand
        ai, bi = [int(x) for x in a], [int(x) for x in b]
        want = [0] * N
        for i in range(N):
            if ai[i] == 0:
                continue
            for j in range(N):
                k = i + j
                if k < N:
                    want[k] += ai[i] * bi[j]
                else:
                    want[k - N] -= ai[i] * bi[j]
        assert [int(x) for x in c] == [w % q for w in want]


def test_ntt_roundtrip_hyp(orc_hyp):
    o = orc_hyp
    rng = np.random.default_rng(3)
    for t in range(o.nq + o.np_):
        q = int(o.moduli[t])
        a = rng.integers(0, q, size=o.N, dtype=np.uint64)
        assert np.array_equal(o.intt(o.ntt(a, t), t), a)


# ---------------------------------------------------------------- encode / decode
def test_encode_matches_mpmath_definition(orc_tiny):
    """m_k = round(Delta * (2/N) Re sum_j z_j zeta^{-5^j k}), zeta = e^{i pi/N}: direct 60-digit evaluation."""
    o = orc_tiny
    mpmath.mp.dps = 60
    rng = np.random.default_rng(4)
    z = rng.uniform(-1, 1, o.n) + 1j * rng.uniform(-1, 1, o.n)
    scale = 2**30 + 7
    m = o.encode_coeffs(z, scale)
    zeta = mpmath.exp(1j * mpmath.pi / o.N)
    for k in range(o.N):
        s = mpmath.mpf(0)
        for j in range(o.n):
            s += mpmath.re(mpmath.mpc(z[j].real, z[j].imag) * zeta ** (-(pow(5, j, 2 * o.N)) * k))
        x = mpmath.mpf(scale) * 2 * s / o.N
        want = int(mpmath.floor(x + mpmath.mpf("0.5"))) if x >= 0 else -int(mpmath.floor(-x + mpmath.mpf("0.5")))
        assert int(m[k]) == want


def test_decode_eval_matches_mpmath(orc_tiny):
    o = orc_tiny
    mpmath.mp.dps = 40
    rng = np.random.default_rng(5)
    m = rng.integers(-1000, 1000, o.N).astype(np.float64)
    z = o.eval_slots(m)
    zeta = mpmath.exp(1j * mpmath.pi / o.N)
    for j in range(o.n):
        e = pow(5, j, 2 * o.N)
        want = sum(mpmath.mpf(int(m[k])) * zeta ** (e * k) for k in range(o.N))
        assert abs(complex(want) - z[j]) < 1e-9 * max(1.0, abs(complex(want)))


def test_encode_decode_integer_roundtrip(orc_mini):
    """encode(decode(m)) == m exactly for random integer m, |m_k| < 2^20 (scale 1)."""
    o = orc_mini
    m = synth.int_coeffs(6, o.N, 2**20 - 1)
    z = o.eval_slots(m.astype(np.float64))
    assert np.array_equal(o.encode_coeffs(z, 1), m)


def test_encode_tie_rule(orc_tiny):
    """constant slot vector c: m_0 = Delta*c exactly, others 0; half-integers round away from zero."""
    o = orc_tiny
    for c, scale, want0 in [(0.5, 1, 1), (-0.5, 1, -1), (1.5, 1, 2), (0.25, 4, 1), (-2.5, 1, -3)]:
        m = o.encode_coeffs(np.full(o.n, c), scale)
        assert int(m[0]) == want0
        assert not np.any(m[1:])


# ---------------------------------------------------------------- automorphism / rotation direction
def test_rotation_is_left_roll(orc_mini):
    """decode(kappa_{5^r}(m)) == roll(decode(m), -r): CRot rotates LEFT."""
    o = orc_mini
    z = synth.slots_uniform(8, o.n)
    m = o.encode_coeffs(z, 2**30)
    q0 = int(o.moduli[0])
    limb = (m % q0).astype(np.uint64)
    for r in [1, 3, o.n - 1, 17, 0]:
        k = o.galois_elt(r)
        rl = o.automorph_coeff(limb, 0, k)
        mr = np.array([_centre(int(x), q0) for x in rl], np.float64)
        zr = o.eval_slots(mr) / 2**30
        assert np.max(np.abs(zr - np.roll(z, -r))) < 1e-6


def test_automorphism_group_laws(orc_mini):
    o = orc_mini
    rng = np.random.default_rng(9)
    a = rng.integers(0, int(o.moduli[1]), o.N, dtype=np.uint64)
    k1, k2 = o.galois_elt(5), o.galois_elt(11)
    assert np.array_equal(o.automorph_coeff(o.automorph_coeff(a, 1, k1), 1, k2),
                          o.automorph_coeff(a, 1, (k1 * k2) % (2 * o.N)))
    assert o.galois_elt(o.n) == 1 and o.galois_elt(0) == 1
    assert np.array_equal(o.automorph_coeff(a, 1, 1), a)


# ---------------------------------------------------------------- keys / encryption
def test_secret_and_errors(orc_hyp):
    o = orc_hyp
    s = o.secret(synth.SEED_SK)
    assert int(np.count_nonzero(s)) == 192
    assert set(np.unique(s)) <= {-1, 0, 1}
    assert np.array_equal(s, o.secret(synth.SEED_SK))
    e = o.cbd(11, oracle.DOM_ENC_E, 0)
    assert np.max(np.abs(e)) <= 21
    assert abs(e.mean()) < 0.1 and abs(e.var() - 10.5) < 0.3   # CBD(21): variance 21/2
    # CBD draw = popcount difference of the first two Philox words
    w = oracle.philox4x32_10([11, 0], [5, 0, 0, oracle.DOM_ENC_E << 24])
    assert e[5] == bin(int(w[0]) & 0x1FFFFF).count("1") - bin(int(w[1]) & 0x1FFFFF).count("1")


def test_decrypt_encrypt_is_m_plus_e(orc_mini):
    o = orc_mini
    level = o.nq - 1
    z = synth.slots_uniform(10, o.n)
    pt = o.encode(z, 2**40, level)
    ct = o.encrypt(synth.SEED_SK, 77, 5, pt)
    m2 = o.decrypt(synth.SEED_SK, ct)
    e = o.cbd(77, oracle.DOM_ENC_E, 5)
    for i in range(level + 1):
        q = int(o.moduli[i])
        diff = (o.intt(m2.data[i], i).astype(object) - o.intt(pt.data[i], i).astype(object)) % q
        assert [_centre(int(x), q) for x in diff] == [int(x) for x in e]
    assert np.max(np.abs(o.decode(m2) - z)) < 1e-9


# ---------------------------------------------------------------- ModUp / ModDown / rescale (big-int CRT)
def _lift(limbs_coeff, mods, x):
    """CRT lift of coefficient x over the given moduli, in [0, prod)."""
    return sympy.ntheory.modular.crt(mods, [int(l[x]) for l in limbs_coeff])[0]


def test_modup_identity(orc_mini):
    """lift(d~_j) = d + u*D_j with 0 <= u < alpha_j (fast BConv without correction)."""
    o = orc_mini
    level = o.nq - 1
    rng = np.random.default_rng(12)
    d = np.stack([rng.integers(0, q, o.N, dtype=np.uint64) for q in o.q[: level + 1]])
    ext = o.modup_coeff(level, d)
    chain = o.ext_chain(level)
    mods = [int(o.moduli[t]) for t in chain]
    for j in range(o.n_digits(level)):
        lo, hi = j * o.alpha, min((j + 1) * o.alpha, level + 1)
        Dj = math.prod(o.q[lo:hi])
        coeff = [o.intt(ext[j][u], chain[u]) for u in range(len(chain))]
        for x in range(0, o.N, 37):
            L = _lift(coeff, mods, x)
            dj = sympy.ntheory.modular.crt(o.q[lo:hi], [int(d[i][x]) for i in range(lo, hi)])[0]
            assert (L - dj) % Dj == 0
            assert 0 <= (L - dj) // Dj < hi - lo


def test_moddown_identity(orc_mini):
    """out*P == U - ut_P (mod Q_l) with ut_P = sum_k z_k (P/p_k) exactly, z_k = [U (P/p_k)^{-1}]_{p_k} taken in
    (-p_k/2, p_k/2] (DESIGN R-MODDOWN, centred), so |ut_P| < K P / 2 and ut_P == U (mod P); and the rounding error
    ut_P / P has mean ~0 over the sampled coefficients (no floor-style bias)."""
    o = orc_mini
    level = 3
    chain = o.ext_chain(level)
    rng = np.random.default_rng(13)
    u = np.stack([rng.integers(0, int(o.moduli[t]), o.N, dtype=np.uint64) for t in chain])
    out = o.moddown(level, u)
    P = math.prod(o.p)
    Q = math.prod(o.q[: level + 1])
    uc = [o.intt(u[i], chain[i]) for i in range(len(chain))]
    oc = [o.intt(out[i], i) for i in range(level + 1)]
    mods = [int(o.moduli[t]) for t in chain]
    errs = []
    for x in range(0, o.N, 41):
        U = _lift(uc, mods, x)
        Ot = _lift(oc, o.q[: level + 1], x)
        r = (U - Ot * P) % (Q * P)
        r = r - Q * P if r > (Q * P) // 2 else r  # == ut_P, centred
        want = 0
        for pk in o.p:
            pk = int(pk)
            z = (U % pk) * pow(P // pk, -1, pk) % pk
            z = z - pk if z > (pk - 1) // 2 else z
            want += z * (P // pk)
        assert r == want
        assert r % P == U % P and abs(r) < o.np_ * P // 2
        errs.append(r / P)
    assert abs(np.mean(errs)) < 0.5


def test_rescale_is_exact_rounding(orc_mini):
    o = orc_mini
    level = o.nq - 1
    rng = np.random.default_rng(14)
    ct = oracle.Ct(np.stack([np.stack([rng.integers(0, q, o.N, dtype=np.uint64) for q in o.q[: level + 1]])
                             for _ in range(2)]), level, 2.0**80)
    out = o.rescale(ct)
    assert out.level == level - 1 and out.scale == 2.0**80 / o.q[level]
    Q = math.prod(o.q[: level + 1])
    Qm = Q // o.q[level]
    for p in range(2):
        cc = [o.intt(ct.data[p][i], i) for i in range(level + 1)]
        oc = [o.intt(out.data[p][i], i) for i in range(level)]
        for x in range(0, o.N, 29):
            C = _lift(cc, o.q[: level + 1], x)
            want = (2 * C + o.q[level]) // (2 * o.q[level])  # round(C / q_l), q_l odd => no ties
            assert _lift(oc, o.q[:level], x) == want % Qm


def test_pmult_add_limbwise(orc_mini):
    o = orc_mini
    level = 2
    rng = np.random.default_rng(15)
    mk = lambda: np.stack([np.stack([rng.integers(0, q, o.N, dtype=np.uint64) for q in o.q[: level + 1]]) for _ in range(2)])
    a, b = oracle.Ct(mk(), level, 1.0), oracle.Ct(mk(), level, 1.0)
    pt = oracle.Pt(np.stack([rng.integers(0, q, o.N, dtype=np.uint64) for q in o.q[: level + 1]]), level, 3.0)
    s, m = o.add(a, b), o.pmult(a, pt)
    for p in range(2):
        for i in range(level + 1):
            q = o.q[i]
            for x in (0, 1, o.N - 1, 333):
                assert int(s.data[p, i, x]) == (int(a.data[p, i, x]) + int(b.data[p, i, x])) % q
                assert int(m.data[p, i, x]) == int(a.data[p, i, x]) * int(pt.data[i, x]) % q
    assert m.scale == 3.0


# ---------------------------------------------------------------- key switching
def _dec_coeffs(o, ct):
    m = o.decrypt(synth.SEED_SK, ct)
    return o.crt_coeffs(m.data, ct.level)


@pytest.fixture(scope="module")
def ks_setup(orc_mini):
    o = orc_mini
    level = o.nq - 1
    z = synth.slots_uniform(20, o.n)
    ct = o.encrypt(synth.SEED_SK, 21, 0, o.encode(z, 2**40, level))
    rs = [1, 5, -3]
    evks = [o.keygen_rot(synth.SEED_SK, synth.SEED_EVK, r) for r in rs]
    return o, level, z, ct, rs, evks


def _ks_bound(o, level):
    """|e_ks| <= beta*alpha*21*N*max_j D_j / P + K*(h+1)   (DESIGN R-KSBOUND)"""
    beta = o.n_digits(level)
    Dmax = max(math.prod(o.q[j * o.alpha: min((j + 1) * o.alpha, level + 1)]) for j in range(beta))
    return beta * o.alpha * 21 * o.N * Dmax / math.prod(o.p) + o.np_ * (o.h + 1)


def test_hrot_decrypt_identity(ks_setup):
    o, level, z, ct, rs, evks = ks_setup
    Q = math.prod(o.q[: level + 1])
    m = _dec_coeffs(o, ct)
    bound = _ks_bound(o, level)
    for r, evk in zip(rs, evks):
        rot = o.hrot(ct, evk, r)
        mr = _dec_coeffs(o, rot)
        # kappa(dec(ct)) in the coefficient domain over the integers
        k = o.galois_elt(r)
        km = [0] * o.N
        for i in range(o.N):
            e = i * k % (2 * o.N)
            if e < o.N:
                km[e] = m[i]
            else:
                km[e - o.N] = -m[i]
        err = max(abs(_centre(a - b, Q)) for a, b in zip(mr, km))
        assert err <= bound, (r, err, bound)
        zr = o.decode(o.decrypt(synth.SEED_SK, rot))
        assert np.max(np.abs(zr - np.roll(z, -r))) < 2**-20


def test_hoisted_and_sum_variants(ks_setup):
    o, level, z, ct, rs, evks = ks_setup
    plain = [o.hrot(ct, e, r) for e, r in zip(evks, rs)]
    hoisted = o.hrot_hoisted(ct, evks, rs)
    for p, h, r in zip(plain, hoisted, rs):
        assert not np.array_equal(p.data, h.data)  # several correct results (DESIGN R-HROT)
        zr = o.decode(o.decrypt(synth.SEED_SK, h))
        assert np.max(np.abs(zr - np.roll(z, -r))) < 2**-20
    # lazy sum vs sum of plain rotations; r = 0 term included without key switching
    cts = [ct, ct, ct, ct]
    rr = rs + [0]
    ee = evks + [None]
    s = o.hrot_sum(cts, ee, rr)
    want = np.roll(z, -rs[0]) + np.roll(z, -rs[1]) + np.roll(z, -rs[2]) + z
    zs = o.decode(o.decrypt(synth.SEED_SK, s))
    assert np.max(np.abs(zs - want)) < 2**-19
    acc = plain[0]
    for p in plain[1:]:
        acc = o.add(acc, p)
    acc = o.add(acc, ct)
    assert not np.array_equal(acc.data, s.data)


def test_keygen_structure(orc_mini):
    """b_j + a_j s == e_j + g_j kappa(s) (mod every prime) with g_j = P on digit j's q-limbs."""
    o = orc_mini
    r = 7
    k = o.galois_elt(r)
    evk = o.keygen_rot(synth.SEED_SK, synth.SEED_EVK, r)
    s = [int(x) for x in o.secret(synth.SEED_SK)]
    ks_ = [0] * o.N
    for i in range(o.N):
        e = i * k % (2 * o.N)
        if e < o.N:
            ks_[e] = s[i]
        else:
            ks_[e - o.N] = -s[i]
    P = math.prod(o.p)
    for j in range(o.dnum):
        e = [int(x) for x in o.cbd(synth.SEED_EVK, oracle.DOM_EVK_E, (k << 8) | j)]
        for t in range(o.nq + o.np_):
            q = int(o.moduli[t])
            b = o.intt(evk[j, 0, t], t)
            a = o.intt(evk[j, 1, t], t)
            # a*s negacyclic via NTT of the oracle (already pinned by the schoolbook test)
            s_ntt = o.ntt(np.array([x % q for x in s], np.uint64), t)
            a_s = o.intt((evk[j, 1, t].astype(object) * s_ntt.astype(object) % q).astype(np.uint64), t)
            g = P % q if (t < o.nq and j * o.alpha <= t < (j + 1) * o.alpha) else 0
            for x in range(0, o.N, 53):
                assert (int(b[x]) + int(a_s[x])) % q == (e[x] + g * ks_[x]) % q
        del a


def test_set_hyp_sizes(orc_hyp):
    """Ctxt 10 MB / Ptxt 5 MB at the post-bootstrap level, Evk 168 MB."""
    o = orc_hyp
    g = dict(l.split() for l in open(os.path.join(GOLD, "set_hyp_sizes.txt")) if l.strip() and not l.startswith("#"))
    assert o.N == 2 ** int(g["log_n"]) and o.nq == int(g["l_plus_1"]) and o.dnum == int(g["dnum"])
    limb = o.N * 8
    post_boot_limbs = 10
    assert 2 * post_boot_limbs * limb == int(g["ctxt_mib_post_boot"]) * 2**20
    assert post_boot_limbs * limb == int(g["ptxt_mib_post_boot"]) * 2**20
    assert o.dnum * 2 * (o.nq + o.np_) * limb == int(g["evk_mib"]) * 2**20
    # P:1243 multiplies the MiB-exact key size by 66 in decimal units: 66 x 168 MB = 11.09 GB
    assert abs(int(g["n_evk_resnet18"]) * int(g["evk_mib"]) / 1000 - float(g["evk_gb_resnet18"])) < 0.05


# ---------------------------------------------------------------- MulCt + relinearization
def _negacyclic_square(s):
    """s^2 in Z[X]/(X^N + 1) by schoolbook over the nonzero coefficients (plain integers)."""
    N = len(s)
    nz = [(i, v) for i, v in enumerate(s) if v]
    out = [0] * N
    for i, a in nz:
        for j, b in nz:
            k = i + j
            if k < N:
                out[k] += a * b
            else:
                out[k - N] -= a * b
    return out


def test_relin_key_structure(orc_mini):
    """Relinearization key (DESIGN R-RELIN): b_j + a_j s == e_j + g_j s^2 (mod every prime), s^2 by schoolbook,
    g_j = P on digit j's q-limbs (R-EVK), e_j drawn with object id j (Galois element 0)."""
    o = orc_mini
    rlk = o.keygen_relin(synth.SEED_SK, synth.SEED_EVK)
    s = [int(x) for x in o.secret(synth.SEED_SK)]
    s2 = _negacyclic_square(s)
    P = math.prod(o.p)
    for j in range(o.dnum):
        e = [int(x) for x in o.cbd(synth.SEED_EVK, oracle.DOM_EVK_E, j)]
        for t in range(o.nq + o.np_):
            q = int(o.moduli[t])
            b = o.intt(rlk[j, 0, t], t)
            s_ntt = o.ntt(np.array([x % q for x in s], np.uint64), t)
            a_s = o.intt((rlk[j, 1, t].astype(object) * s_ntt.astype(object) % q).astype(np.uint64), t)
            g = P % q if (t < o.nq and j * o.alpha <= t < (j + 1) * o.alpha) else 0
            for x in range(0, o.N, 37):
                assert (int(b[x]) + int(a_s[x])) % q == (e[x] + g * s2[x]) % q


def test_mulct_decrypts_to_product(orc_mini):
    """dec(MulCt(a, b)) = dec(a) * dec(b) (negacyclic, mod Q) up to the key-switch error of relinearizing
    d2 (R-KSBOUND); the rescaled square decodes to the slot-wise square (AESPA x^2)."""
    o = orc_mini
    level = o.nq - 1
    Q = math.prod(o.q[: level + 1])
    rlk = o.keygen_relin(synth.SEED_SK, synth.SEED_EVK)
    za, zb = synth.slots_uniform(40, o.n), synth.slots_uniform(41, o.n)
    a = o.encrypt(synth.SEED_SK, 42, 0, o.encode(za, 2**40, level))
    b = o.encrypt(synth.SEED_SK, 42, 1, o.encode(zb, 2**40, level))
    ab = o.mulct(a, b, rlk)
    # dec(a) * dec(b): product of the decrypted plaintexts in the NTT domain (NTT product = schoolbook,
    # pinned above), back to centred integer coefficients by CRT
    ma, mb = o.decrypt(synth.SEED_SK, a), o.decrypt(synth.SEED_SK, b)
    prod = np.array([[int(x) * int(y) % o.q[i] for x, y in zip(ma.data[i], mb.data[i])] for i in range(level + 1)],
                    dtype=object).astype(np.uint64)
    want = o.crt_coeffs(prod, level)
    got = _dec_coeffs(o, ab)
    err = max(abs(_centre(x - y, Q)) for x, y in zip(got, want))
    assert err <= _ks_bound(o, level), err
    sq = o.square(a, rlk)
    assert sq.level == level - 1
    assert np.max(np.abs(np.real(o.decode(o.decrypt(synth.SEED_SK, sq))) - za * za)) < 2**-20
