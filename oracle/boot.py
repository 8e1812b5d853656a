"""Oracle for the linear steps of CKKS bootstrapping (partial) -- TEST INFRASTRUCTURE.

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
EvalMod (the approximate modular reduction between them) is not built.
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
