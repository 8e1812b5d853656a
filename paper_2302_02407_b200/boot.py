"""CKKS bootstrapping on the B200 engine at small ring sizes (DESIGN
R-LINTRANS, R-EVALMOD): ModRaise -> CoeffToSlot -> conjugation split -> EvalMod (Chebyshev series of cos(a s) and
r double angles: the scaled sine of the modular reduction) -> recombination -> SlotToCoeff.

Every homomorphic step is a C-ABI call into libhyphen.so (hy_mod_raise, hy_lintrans_apply, hy_hrot_galois,
hy_mulct, hy_pmult, hy_rescale, hy_add, hy_sub, hy_add_pt, hy_level_down); this module only sequences them and tracks
the scales (as ConvBlock sequences a residual block).  The CoeffToSlot / SlotToCoeff matrices and the Chebyshev
coefficients are inputs, like conv weights.  The dense transforms need n = N/2 diagonals, so this runs at N <= 2^12;
the N = 2^16 special FFT would need its level-budgeted radix factorisation (not built).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# T_k = 2 T_m T_n - T_|m-n| for every even k <= 30 at depth <= 5 (DESIGN R-EVALMOD)
CHEB_SCHEDULE = [(2, 1, 1), (4, 2, 2), (8, 4, 4), (16, 8, 8), (6, 4, 2), (10, 8, 2), (12, 8, 4), (14, 8, 6),
                 (18, 16, 2), (20, 16, 4), (22, 16, 6), (24, 16, 8), (26, 16, 10), (28, 16, 12), (30, 16, 14)]


@dataclass
class CT:
    t: object          # device tensor [2][level+1][N]
    level: int
    scale: float


class Bootstrapper:
    def __init__(self, ctx, cts_diags, stc_diags, bs: int, cheb, r: int, a: float, evks: dict, conj_key, rlk):
        """cts_diags / stc_diags: the n diagonals of V^{-1}/2 and of (K/2pi) V (ascending d); cheb: Chebyshev
        coefficients of cos(a s) on [-1, 1] (odd ones zero); evks: rotation amount -> key (the transforms' baby and
        giant steps); conj_key: the Galois key of k = 2N - 1; rlk: the relinearization key."""
        from . import LinTrans
        self.ctx, self.bs, self.cheb, self.r, self.a = ctx, bs, list(cheb), r, a
        self.evks, self.conj_key, self.rlk = evks, conj_key, rlk
        self.q = ctx.moduli
        n = ctx.n
        self.cts = LinTrans(ctx, list(range(n)), bs)
        self.stc = LinTrans(ctx, list(range(n)), bs)
        self._cts_diags, self._stc_diags = cts_diags, stc_diags
        self._pts = {}
        self._consts = {}

    # ---- helpers (each one C-ABI call, scales tracked as the oracle's Ct does)
    def _const(self, c, scale, level):
        """the constant plaintext c at integer scale round(scale), encoded once and kept on the device (so that a
        bootstrap issues only device work and can be captured in a CUDA graph)"""
        key = (float(c), int(round(scale)), level)
        if key not in self._consts:
            self._consts[key] = self.ctx.encode(np.full(self.ctx.n, float(c)), key[1], level)
        return self._consts[key], float(key[1])

    def _monomial(self, sign, level):
        key = ("X^{N/2}", sign, level)
        if key not in self._consts:
            cf = np.zeros(self.ctx.N, np.int64)
            cf[self.ctx.N // 2] = sign
            self._consts[key] = self.ctx.pt_from_coeffs(cf, level)
        return self._consts[key]

    def _down(self, x: CT, level):
        return x if x.level == level else CT(self.ctx.level_down(x.t, x.level, level), level, x.scale)

    def _pmult(self, x: CT, pt, pt_scale):
        return CT(self.ctx.pmult(x.t, pt, x.level), x.level, x.scale * pt_scale)

    def _rescale(self, x: CT):
        return CT(self.ctx.rescale(x.t, x.level), x.level - 1, x.scale / self.q[x.level])

    def _add(self, a: CT, b: CT):
        return CT(self.ctx.add(a.t, b.t, a.level), a.level, a.scale)

    def _sub(self, a: CT, b: CT):
        return CT(self.ctx.sub(a.t, b.t, a.level), a.level, a.scale)

    def _add_const(self, x: CT, c):
        pt, s = self._const(c, x.scale, x.level)
        return CT(self.ctx.add_pt(x.t, x.scale, pt, s, x.level), x.level, x.scale)

    def _mul(self, a: CT, b: CT):
        lv = min(a.level, b.level)
        a, b = self._down(a, lv), self._down(b, lv)
        return self._rescale(CT(self.ctx.mulct(self.rlk, a.t, b.t, lv), lv, a.scale * b.scale))

    def _rescaled_to(self, x: CT, target):
        pt, s = self._const(1.0, float(self.q[x.level]) * target / x.scale, x.level)
        return self._rescale(self._pmult(x, pt, s))

    def _lintrans(self, lt, diags, x: CT):
        key = (id(lt), x.level)
        if key not in self._pts:
            self._pts[key] = lt.encode(diags, x.level)
        q = self.q[x.level]
        return CT(lt.apply(self.evks, x.t, x.level, self._pts[key]), x.level - 1, (x.scale * q) / q)

    # ---- the steps
    def eval_chebyshev(self, s: CT, target: float) -> CT:
        T = {1: s}
        for k, m, n in CHEB_SCHEDULE:
            p = self._mul(T[m], T[n])
            p = self._add(p, p)
            d = abs(m - n)
            if d == 0:
                T[k] = self._add_const(p, -1.0)
            else:
                T[k] = self._sub(p, self._down(self._rescaled_to(T[d], p.scale), p.level))
        terms = []
        for k in range(2, len(self.cheb), 2):
            if self.cheb[k] == 0:
                continue
            t = T[k]
            pt, sc = self._const(self.cheb[k], float(self.q[t.level]) * target / t.scale, t.level)
            terms.append(self._rescale(self._pmult(t, pt, sc)))
        lv = min(t.level for t in terms)
        acc = None
        for t in terms:
            t = self._down(t, lv)
            acc = t if acc is None else self._add(acc, t)
        return self._add_const(acc, self.cheb[0])

    def eval_mod(self, s: CT) -> CT:
        c = self.eval_chebyshev(s, s.scale)
        for _ in range(self.r):
            sq = self._mul(c, c)
            c = self._add_const(self._add(sq, sq), -1.0)
        return c

    def bootstrap(self, ct0, scale: float, level: int) -> CT:
        """a level-0 ciphertext at `scale` -> a ciphertext of the same slots at a higher level"""
        ctx = self.ctx
        K = float(self.q[0]) / scale
        alpha1 = 2.0 * math.pi / (K * (2 ** self.r) * self.a)
        beta1 = -math.pi / (2.0 * (2 ** self.r) * self.a)
        up = CT(ctx.mod_raise(ct0, level), level, scale)
        y = self._lintrans(self.cts, self._cts_diags, up)
        pt, s = self._const(alpha1, float(self.q[y.level]), y.level)
        y = self._rescale(self._pmult(y, pt, s))
        yc = CT(ctx.hrot_galois(self.conj_key, y.t, y.level, 2 * ctx.N - 1), y.level, y.scale)
        s_re = self._add_const(self._add(y, yc), beta1)
        d = self._sub(y, yc)
        s_im = self._add_const(CT(ctx.pmult(d.t, self._monomial(-1, d.level), d.level), d.level, d.scale), beta1)
        e_re = self.eval_mod(s_re)
        e_im = self.eval_mod(s_im)
        ie = CT(ctx.pmult(e_im.t, self._monomial(1, e_im.level), e_im.level), e_im.level, e_im.scale)
        z = self._add(e_re, ie)
        return self._lintrans(self.stc, self._stc_diags, z)
