"""Oracle for CKKS bootstrapping -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import this (see oracle/__init__.py).

* mod_raise: ModRaise, the first step of bootstrapping: a level-0 ciphertext (mod q_0) is read as integer
  polynomials with centred coefficients in (-q_0/2, q_0/2] and reduced mod q_0..q_l.  Plain definition: iNTT of
  limb 0, centred lift, reduction, NTT -- each step the textbook one (oracle/ckks_oracle.c transforms).
* lintrans: the homomorphic diagonal linear transform y = M x of CoeffToSlot / SlotToCoeff, step by step as
  DESIGN R-LINTRANS fixes it: diag_d[j] = M[j][(j + d) mod n]; d = g bs + b; the baby steps Rot_b(x) as one hoisted
  HRot batch, inner_g = sum_b PMult(Rot_b(x), Enc(Rot_{-g bs}(diag_{g bs + b}), scale q_l)), y = HRotSum over the
  giant steps g bs (one ModDown), then Rescale.
* special_fft_matrix: the canonical embedding restricted to CKKS's complex packing, V[j][k] = zeta^{k 5^j}
  (zeta = exp(i pi / N)), so that the slots of a plaintext with coefficients m are V (m_k + i m_{k+n})_k / scale
  (DESIGN R-ENCODE).  CoeffToSlot is V^{-1} on the slots, SlotToCoeff is V.
* sfft_stage / diag_mul / sfft_levels: V factorised into radix-2 butterfly stages (three diagonals each) grouped
  into a few levels (DESIGN R-SFFT), so that CoeffToSlot / SlotToCoeff at N = 2^16 take 3 levels and ~42 rotation keys
  (48 rotation keys) instead of n = 2^15 dense diagonals.  Pinned in tests/test_oracle_boot.py against the
  dense V and V^{-1} (products of the levels, bit reversal), and the product of two diagonal matrices against dense
  matmul.
* eval_chebyshev / eval_mod / bootstrap: EvalMod and the whole bootstrap in the operation order DESIGN R-EVALMOD fixes.
"""
from __future__ import annotations

import numpy as np

from . import Ct


def mod_raise(o, ct: Ct, level: int) -> Ct:
    assert ct.level == 0
    q0 = int(o.q[0])
    out = np.empty((2, level + 1, o.N), np.uint64)
    for p in range(2):
        v = o.intt(ct.data[p, 0], 0).astype(object)
        cen = np.where(v > (q0 - 1) // 2, v - q0, v)
        for i in range(level + 1):
            qi = int(o.q[i])
            out[p, i] = o.ntt(np.array([int(x) % qi for x in cen], dtype=np.uint64), i)
    return Ct(out, level, ct.scale)


def diagonals(M: np.ndarray, ds) -> list:
    """diag_d[j] = M[j][(j + d) mod n] for each d in ds (ascending canonical order)"""
    n = M.shape[0]
    j = np.arange(n)
    return [M[j, (j + d) % n] for d in ds]


def lintrans(o, ct: Ct, diags: dict, bs: int, evks: dict) -> Ct:
    """y = M x with M given by its nonzero diagonals {d: diag_d}; evks: rotation amount (mod n) -> key."""
    n = o.n
    level = ct.level
    terms = {}
    for d, v in diags.items():
        d %= n
        terms[(d // bs, d % bs)] = np.asarray(v)
    babies = sorted({b for _, b in terms})
    giants = sorted({g for g, _ in terms})
    nz = [b for b in babies if b]
    rot = dict(zip(nz, o.hrot_hoisted(ct, [evks[b] for b in nz], nz))) if nz else {}
    rot[0] = ct
    inner = []
    for g in giants:
        acc = None
        for b in babies:
            if (g, b) not in terms:
                continue
            # Rot_{-g bs}(diag): v[j] = diag[j - g bs]
            pt = o.encode(np.roll(terms[(g, b)], g * bs), int(o.q[level]), level)
            t = o.pmult(rot[b], pt)
            acc = t if acc is None else o.add(acc, t)
        inner.append(acc)
    rs = [(g * bs) % n for g in giants]
    keys = [evks[r] if r else None for r in rs]
    return o.rescale(o.hrot_sum(inner, keys, rs))


def special_fft_matrix(N: int) -> np.ndarray:
    n = N // 2
    M2 = 2 * N
    rot = np.array([pow(5, j, M2) for j in range(n)], dtype=object)
    k = np.arange(n, dtype=object)
    e = np.outer(rot, k) % M2
    return np.exp(1j * np.pi * e.astype(np.float64) / N)


# --------------------------------------------------------------------------- the special FFT, factorised
# DESIGN R-SFFT.  V (special_fft_matrix) is evaluated by the radix-2 "special FFT": bit-reverse the input, then for
# len = 2, 4, ..., n, every block of len slots takes the butterfly (x_j, x_{j+len/2}) -> (x_j + w x_{j+len/2},
# x_j - w x_{j+len/2}) with w = zeta^{(5^j mod 4 len) N / (2 len)} (zeta = exp(i pi / N)), j < len / 2.  Each stage
# is a matrix with three diagonals (offsets 0, +len/2, -len/2 mod n); the dense V never has to be formed.


def sfft_stage(N: int, length: int, inverse: bool = False) -> dict:
    """the butterfly stage of half-length h = length / 2 as diagonals {d: diag_d} (diag_d[j] = S[j][(j + d) mod n]);
    inverse: the stage's inverse, (a, b) -> ((a + b) / 2, (a - b) / (2 w))"""
    n, h = N // 2, length // 2
    d0 = np.zeros(n, complex)
    dp = np.zeros(n, complex)
    dm = np.zeros(n, complex)
    for p in range(n):
        j = p % length
        jj = j if j < h else j - h
        e = (pow(5, jj, 4 * length) * (N // (2 * length))) % (2 * N)
        w = np.exp(1j * np.pi * e / N)
        if j < h:  # output p = x_p + w x_{p+h}   (inverse: (x_p + x_{p+h}) / 2)
            d0[p], dp[p] = (0.5, 0.5) if inverse else (1.0, w)
        else:      # output p = x_{p-h} - w x_p   (inverse: (x_{p-h} - x_p) / (2 w))
            dm[p], d0[p] = (0.5 / w, -0.5 / w) if inverse else (1.0, -w)
    out = {0: d0}
    for d, v in ((h % n, dp), ((n - h) % n, dm)):
        out[d] = out[d] + v if d in out else v
    return out


def diag_mul(A: dict, B: dict, n: int) -> dict:
    """the diagonals of the matrix product A B: (A B)[j][j + d] = sum_{a + b = d} A_a[j] B_b[j + a]"""
    out = {}
    j = np.arange(n)
    for a, va in A.items():
        for b, vb in B.items():
            d = (a + b) % n
            t = va * vb[(j + a) % n]
            out[d] = out[d] + t if d in out else t
    return out


def bit_reverse_perm(n: int) -> np.ndarray:
    bits = n.bit_length() - 1
    return np.array([int(format(k, f"0{bits}b")[::-1], 2) if bits else 0 for k in range(n)])


def sfft_levels(N: int, groups, inverse: bool = False, scale: complex = 1.0) -> list:
    """V = S_n ... S_4 S_2 P (P the bit reversal), grouped into len(groups) levels of consecutive stages
    (groups = stages per level, low half-lengths first, sum = log2 n).  Forward (SlotToCoeff): the levels in the
    order they are applied to a bit-reversed slot vector, [S_{2^g0} ... S_2, ...] -> scale V P.  Inverse
    (CoeffToSlot): the order they are applied to the slots, [S_n^{-1} ..., ..., ... S_2^{-1}] -> scale P V^{-1}
    (output in bit-reversed slot order).  scale multiplies the first level applied."""
    n = N // 2
    assert sum(groups) == n.bit_length() - 1
    lens, at = [], 1
    for g in groups:
        lens.append([2 ** (at + k) for k in range(g)])
        at += g
    levels = []
    for ls in lens:
        M = None
        for length in ls:  # later stages on the left
            S = sfft_stage(N, length, inverse)
            M = S if M is None else (diag_mul(S, M, n) if not inverse else diag_mul(M, S, n))
        levels.append(M)
    if inverse:
        levels = levels[::-1]
    levels[0] = {d: v * scale for d, v in levels[0].items()}
    return levels


# --------------------------------------------------------------------------- EvalMod and the whole bootstrap
# DESIGN R-EVALMOD fixes the operation sequence; the Chebyshev coefficients and the linear-transform matrices are
# inputs (data) of both implementations, like conv weights.
CHEB_SCHEDULE = [  # (k, m, n): T_k = 2 T_m T_n - T_|m-n|, every even k <= 30 at depth <= 5
    (2, 1, 1), (4, 2, 2), (8, 4, 4), (16, 8, 8), (6, 4, 2), (10, 8, 2), (12, 8, 4), (14, 8, 6),
    (18, 16, 2), (20, 16, 4), (22, 16, 6), (24, 16, 8), (26, 16, 10), (28, 16, 12), (30, 16, 14)]


def _const(o, c, scale, level):
    return o.encode(np.full(o.n, float(c)), int(round(scale)), level)


def _monomial(o, sign, level):
    """the plaintext sign * X^{N/2} (scale 1): multiplication by sign * i on every slot"""
    import oracle as _o
    cf = np.zeros(o.N, np.int64)
    cf[o.N // 2] = sign
    return _o.Pt(o.coeffs_to_pt(cf, level), level, 1.0)


def _down(o, ct, level):
    return ct if ct.level == level else o.level_down(ct, level)


def _sub(o, a: Ct, b: Ct) -> Ct:
    """a - b limbwise mod q (plain definition)"""
    out = np.empty_like(a.data)
    for p in range(2):
        for i in range(a.level + 1):
            q = np.uint64(o.q[i])
            out[p, i] = (a.data[p, i] + (q - b.data[p, i]) % q) % q
    return Ct(out, a.level, a.scale)


def _add_const(o, ct, c):
    return o.add_pt(ct, _const(o, c, ct.scale, ct.level))


def _mul(o, a, b, rlk):
    lv = min(a.level, b.level)
    return o.rescale(o.mulct(_down(o, a, lv), _down(o, b, lv), rlk))


def _rescaled_to(o, t: Ct, target: float) -> Ct:
    """t brought to scale `target` (one level): PMult by the constant 1 encoded at the integer scale
    round(q_l target / t.scale), then rescale by q_l -- how terms of different scales are aligned before they are
    added (DESIGN R-EVALMOD)"""
    S = float(o.q[t.level]) * target / t.scale
    return o.rescale(o.pmult(t, _const(o, 1.0, S, t.level)))


def eval_chebyshev(o, s: Ct, cheb, rlk, target: float) -> Ct:
    """sum_k cheb[k] T_k(s) for even k (DESIGN R-EVALMOD): T_k = 2 T_m T_n - T_|m-n| by CHEB_SCHEDULE, T_|m-n| first
    brought to the product's scale (_rescaled_to) and level; each term c_k T_k a PMult by the constant c_k encoded at
    round(q_l target / scale(T_k)) and a rescale (every term then at scale ~ target); the terms aligned to the lowest
    level and summed in increasing k; then c_0 added at the sum's scale."""
    T = {1: s}
    for k, m, n in CHEB_SCHEDULE:
        p = _mul(o, T[m], T[n], rlk)
        p = o.add(p, p)
        d = abs(m - n)
        if d == 0:
            T[k] = _add_const(o, p, -1.0)
        else:
            T[k] = _sub(o, p, _down(o, _rescaled_to(o, T[d], p.scale), p.level))
    terms = []
    for k in range(2, len(cheb), 2):
        if cheb[k] == 0:
            continue
        t = T[k]
        S = float(o.q[t.level]) * target / t.scale
        terms.append(o.rescale(o.pmult(t, _const(o, cheb[k], S, t.level))))
    lv = min(t.level for t in terms)
    acc = None
    for t in terms:
        t = _down(o, t, lv)
        acc = t if acc is None else o.add(acc, t)
    return _add_const(o, acc, cheb[0])


def eval_mod(o, s: Ct, cheb, r: int, rlk) -> Ct:
    """cos(a s) by the Chebyshev series, then r double angles cos(2x) = 2 cos(x)^2 - 1"""
    c = eval_chebyshev(o, s, cheb, rlk, s.scale)
    for _ in range(r):
        sq = _mul(o, c, c, rlk)
        c = _add_const(o, o.add(sq, sq), -1.0)
    return c


def bootstrap(o, ct: Ct, level: int, cts_diags: dict, stc_diags: dict, bs: int, cheb, r: int, a: float,
              evks: dict, conj_key, rlk) -> Ct:
    """ModRaise -> CoeffToSlot -> (Re, Im) split by conjugation -> EvalMod -> recombine -> SlotToCoeff
    (DESIGN R-EVALMOD).  cts_diags: the diagonals of V^{-1} / 2, stc_diags those of (K / 2 pi) V, with
    K = q_0 / scale -- or their factorised forms (lists of levels, bs a tuple of two lists (CoeffToSlot, SlotToCoeff):
    sfft_levels, DESIGN R-SFFT; the slots
    between them in bit-reversed order, which the slot-wise EvalMod does not see); cheb: the coefficients of cos(a s) on [-1, 1].  The CoeffToSlot output is scaled by
    alpha1 = 2 pi / (K 2^r a) with a constant PMult (a constant encodes into one coefficient, exactly to 2^-27,
    where alpha1 folded into the diagonals would keep only ~15 bits of them)."""
    K = float(o.q[0]) / ct.scale
    alpha1 = 2.0 * np.pi / (K * (2 ** r) * a)
    beta1 = -np.pi / (2.0 * (2 ** r) * a)
    bs_c, bs_s = bs if isinstance(bs, tuple) else (bs, bs)
    up = mod_raise(o, ct, level)
    y = lintrans_levels(o, up, cts_diags, bs_c, evks)
    # alpha1's constant is encoded at scale q_l q_{l-1} / scale(y): s_re / s_im leave at the EvalMod scale q_{l-1}
    # (DESIGN R-EVALMOD), which the squarings then keep near the primes they rescale by
    y = o.rescale(o.pmult(y, _const(o, alpha1, float(o.q[y.level]) * float(o.q[y.level - 1]) / y.scale, y.level)))
    yc = o.hrot_galois(y, conj_key, 2 * o.N - 1)
    s_re = _add_const(o, o.add(y, yc), beta1)
    s_im = _add_const(o, o.pmult(_sub(o, y, yc), _monomial(o, -1, y.level)), beta1)
    e_re = eval_mod(o, s_re, cheb, r, rlk)
    e_im = eval_mod(o, s_im, cheb, r, rlk)
    z = o.add(e_re, o.pmult(e_im, _monomial(o, 1, e_im.level)))
    del K
    return lintrans_levels(o, z, stc_diags, bs_s, evks)


def lintrans_levels(o, ct: Ct, levels, bs, evks: dict) -> Ct:
    """one dense transform ({d: diag}, bs an int) or a factorised one (a list of {d: diag} levels applied in order,
    bs a list), one lintrans (one level) each (DESIGN R-SFFT)"""
    if isinstance(levels, dict):
        return lintrans(o, ct, levels, bs, evks)
    for D, b in zip(levels, bs):
        ct = lintrans(o, ct, D, b, evks)
    return ct
