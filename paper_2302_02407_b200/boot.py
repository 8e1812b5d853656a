"""CKKS bootstrapping on the B200 engine at small ring sizes (DESIGN
R-LINTRANS, R-EVALMOD): ModRaise -> CoeffToSlot -> conjugation split -> EvalMod (Chebyshev series of cos(a s) and
r double angles: the scaled sine of the modular reduction) -> recombination -> SlotToCoeff.

Every homomorphic step is a C-ABI call into libhyphen.so (hy_mod_raise, hy_lintrans_apply, hy_hrot_galois,
hy_mulct, hy_pmult, hy_rescale, hy_add, hy_sub, hy_add_pt, hy_level_down); this module only sequences them and tracks
the scales (as ConvBlock sequences a residual block).  The CoeffToSlot / SlotToCoeff matrices and the Chebyshev
coefficients are inputs, like conv weights.  Dense transforms need n = N/2 diagonals (small rings only);
at N = 2^16 the transforms are factorised into 3 levels of radix-2 butterfly stages (sfft_levels, DESIGN R-SFFT).
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
    def __init__(self, ctx, cts_diags, stc_diags, bs, cheb, r: int, a: float, evks, conj_key, rlk):
        """cts_diags / stc_diags: the n diagonals of V^{-1}/2 and of (K/2pi) V (ascending d, bs an int), or their
        factorised forms (lists of {d: diag} levels, bs a list per transform pair: sfft_levels, DESIGN R-SFFT); cheb:
        Chebyshev coefficients of cos(a s) on [-1, 1] (odd ones zero); evks: rotation amount -> key (the transforms'
        baby and giant steps, `transform_rots`); conj_key: the Galois key of k = 2N - 1; rlk: the relinearization
        key."""
        self.ctx, self.cheb, self.r, self.a = ctx, list(cheb), r, a
        self.evks, self.conj_key, self.rlk = evks, conj_key, rlk
        self.q = ctx.moduli
        self.cts = _levels(ctx, cts_diags, bs[0] if isinstance(bs, (list, tuple)) else bs)
        self.stc = _levels(ctx, stc_diags, bs[1] if isinstance(bs, (list, tuple)) else bs)
        self._pts = {}
        self._consts = {}

    @property
    def rots(self):
        """every rotation amount the two transforms need a key for"""
        return sorted({r for lt, _ in self.cts + self.stc for r in lt.rots})

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

    def _lintrans(self, levels, x: CT):
        for lt, diags in levels:
            key = (id(lt), x.level)
            if key not in self._pts:
                self._pts[key] = lt.encode(diags, x.level)
            q = self.q[x.level]
            x = CT(lt.apply(self.evks, x.t, x.level, self._pts[key]), x.level - 1, (x.scale * q) / q)
        return x

    def _mul_many(self, As, Bs):
        """pairwise MulCt + rescale of several ciphertext pairs in lockstep: one batched key switch (hy_mulct_batch;
        each item bit-identical to its own hy_mulct)"""
        lv = min(x.level for x in As + Bs)
        # every pair at the level its own _mul would use (a batch must not pull a pair lower than that)
        assert all(min(a.level, b.level) == lv for a, b in zip(As, Bs))
        As, Bs = [self._down(a, lv) for a in As], [self._down(b, lv) for b in Bs]
        outs = self.ctx.mulct_batch(self.rlk, [a.t for a in As], [b.t for b in Bs], lv)
        res = self.ctx.rescale_batch(outs, lv)
        return [CT(r, lv - 1, a.scale * b.scale / self.q[lv]) for r, a, b in zip(res, As, Bs)]

    # ---- the steps
    def _rescaled_to_many(self, xs, target):
        """_rescaled_to of ciphertexts in lockstep (equal levels and scales): one constant, one batched PMult
        (hy_pmult_batch) and one batched rescale; each item bit-identical to its own _rescaled_to"""
        x0 = xs[0]
        pt, s = self._const(1.0, float(self.q[x0.level]) * target / x0.scale, x0.level)
        return self._pmult_rescale_many(xs, pt, s)

    def _pmult_rescale_many(self, xs, pt, s):
        return self._pmult_rescale_groups([(xs, pt, s)])[0]

    def _pmult_rescale_groups(self, groups):
        """[(cts, pt, pt_scale)] -> [[rescale(ct (.) pt)]]: one batched PMult per group (one plaintext each), then
        one batched rescale per level over every group's products; each item bit-identical to its own PMult +
        rescale"""
        prods = [self.ctx.pmult_batch([x.t for x in xs], pt, xs[0].level) for xs, pt, _ in groups]
        by_level = {}
        for gi, (xs, _, _) in enumerate(groups):
            for ii, x in enumerate(xs):
                by_level.setdefault(x.level, []).append((gi, ii))
        res = [[None] * len(xs) for xs, _, _ in groups]
        for lv, idx in by_level.items():
            outs = self.ctx.rescale_batch([prods[gi][ii] for gi, ii in idx], lv)
            for (gi, ii), o in zip(idx, outs):
                xs, _, s = groups[gi]
                res[gi][ii] = CT(o, lv - 1, xs[ii].scale * s / self.q[lv])
        return res

    def eval_chebyshev_many(self, xs, targets):
        """eval_chebyshev of several ciphertexts in lockstep (the real and imaginary parts): the same operation
        sequence per item as eval_chebyshev, every MulCt, scale alignment and coefficient product batched over the
        items (their levels and scales are equal step by step)"""
        assert all(t == targets[0] for t in targets) and all(x.scale == xs[0].scale for x in xs)
        target = targets[0]
        T = {1: list(xs)}
        # the schedule in waves of entries whose operands are ready (depth by depth: T2 | T4 | T8, T6 |
        # T16, T10, T12, T14 | T18 .. T30); a wave's MulCts share one level, so all of them, for every item, run as ONE
        # batched MulCt + rescale -- 5 sequential key-switch steps instead of 15, each item's operations unchanged
        todo = list(CHEB_SCHEDULE)
        while todo:
            wave = [e for e in todo if all(v in T for v in (e[1], e[2], abs(e[1] - e[2])) if v)]
            todo = [e for e in todo if e not in wave]
            ni = len(xs)
            prods = self._mul_many([a for _, m, _ in wave for a in T[m]], [b for _, _, n in wave for b in T[n]])
            ps = {k: [self._add(p, p) for p in prods[w * ni:(w + 1) * ni]] for w, (k, _, _) in enumerate(wave)}
            # the scale alignments of T_|m-n| (one constant per entry), rescaled together level by level
            al_entries = [(k, abs(m - n)) for k, m, n in wave if m != n]
            groups = []
            for k, d in al_entries:
                x0 = T[d][0]
                pt, sc = self._const(1.0, float(self.q[x0.level]) * ps[k][0].scale / x0.scale, x0.level)
                groups.append((T[d], pt, sc))
            als = dict(zip([k for k, _ in al_entries], self._pmult_rescale_groups(groups)))
            for k, m, n in wave:
                if m == n:
                    T[k] = [self._add_const(p, -1.0) for p in ps[k]]
                else:
                    T[k] = [self._sub(p, self._down(a, p.level)) for p, a in zip(ps[k], als[k])]
        groups = []
        for k in range(2, len(self.cheb), 2):
            if self.cheb[k] == 0:
                continue
            t0 = T[k][0]
            pt, sc = self._const(self.cheb[k], float(self.q[t0.level]) * target / t0.scale, t0.level)
            groups.append((T[k], pt, sc))
        terms = self._pmult_rescale_groups(groups)
        lv = min(x[0].level for x in terms)
        outs = []
        for i in range(len(xs)):
            acc = None
            for x in terms:
                x = self._down(x[i], lv)
                acc = x if acc is None else self._add(acc, x)
            outs.append(self._add_const(acc, self.cheb[0]))
        return outs

    def eval_mod_many(self, xs):
        cs = self.eval_chebyshev_many(xs, [x.scale for x in xs])
        for _ in range(self.r):
            sqs = self._mul_many(cs, cs)
            cs = [self._add_const(self._add(sq, sq), -1.0) for sq in sqs]
        return cs

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
        y = self._lintrans(self.cts, up)
        # alpha1 brings the slots to the EvalMod scale: the next prime q_{l-1} (R-EVALMOD), so that the squarings
        # of the Chebyshev series and the double angles keep the scale near the primes they rescale by
        pt, s = self._const(alpha1, float(self.q[y.level]) * float(self.q[y.level - 1]) / y.scale, y.level)
        y = self._rescale(self._pmult(y, pt, s))
        yc = CT(ctx.hrot_galois(self.conj_key, y.t, y.level, 2 * ctx.N - 1), y.level, y.scale)
        s_re = self._add_const(self._add(y, yc), beta1)
        d = self._sub(y, yc)
        s_im = self._add_const(CT(ctx.pmult(d.t, self._monomial(-1, d.level), d.level), d.level, d.scale), beta1)
        e_re, e_im = self.eval_mod_many([s_re, s_im])  # the two parts in lockstep (batched MulCts)
        ie = CT(ctx.pmult(e_im.t, self._monomial(1, e_im.level), e_im.level), e_im.level, e_im.scale)
        z = self._add(e_re, ie)
        return self._lintrans(self.stc, z)


def _levels(ctx, diags, bs):
    """[(LinTrans, diagonal values in ascending d)] of one dense transform (a list of n diagonals) or of a factorised
    one (a list of {d: diag} dicts, bs a list)"""
    from . import LinTrans
    if isinstance(diags, (list, tuple)) and diags and isinstance(diags[0], dict):
        out = []
        for D, b in zip(diags, bs):
            ds = sorted(D)
            out.append((LinTrans(ctx, ds, b), [D[d] for d in ds]))
        return out
    return [(LinTrans(ctx, list(range(ctx.n)), bs), diags)]


def transform_rots(ctx, diags, bs) -> list:
    """rotation amounts the transform (dense or factorised, as Bootstrapper takes it) needs keys for"""
    return sorted({r for lt, _ in _levels(ctx, diags, bs) for r in lt.rots})


# ---- the special FFT factorised into levels (DESIGN R-SFFT; host-side data of the transforms, like conv weights)
def sfft_levels(N: int, groups, inverse: bool = False, scale: complex = 1.0) -> list:
    """The CKKS special FFT V (slots = V (m_k + i m_{k+n})_k) as radix-2 butterfly stages of half-length h
    = 1, 2, ..., n/2 -- (x_j, x_{j+h}) -> (x_j + w x_{j+h}, x_j - w x_{j+h}), w = zeta^{(5^j mod 4 len) N / (2 len)},
    len = 2h -- on a bit-reversed input, grouped into len(groups) levels of consecutive stages; each level a dict
    {offset d: diag_d} with diag_d[j] = M[j][(j + d) mod n].  Forward: the levels of S_n ... S_2 in application order
    (SlotToCoeff on bit-reversed slots); inverse: those of P V^{-1} (CoeffToSlot, output bit-reversed).  `scale`
    multiplies the first level applied."""
    n = N // 2
    assert sum(groups) == n.bit_length() - 1
    rot = np.empty(n, np.int64)
    r = 1
    for j in range(n):
        rot[j] = r
        r = (r * 5) % (2 * N)
    p = np.arange(n)

    def stage(length):
        h = length // 2
        j = p % length
        first = j < h
        jj = np.where(first, j, j - h)
        e = ((rot[jj] % (4 * length)) * (N // (2 * length))) % (2 * N)
        w = np.exp(1j * np.pi * e / N)
        if inverse:
            d0 = np.where(first, 0.5, -0.5 / w)
            dp = np.where(first, 0.5, 0.0)
            dm = np.where(first, 0.0, 0.5 / w)
        else:
            d0 = np.where(first, 1.0, -w)
            dp = np.where(first, w, 0.0)
            dm = np.where(first, 0.0, 1.0)
        out = {0: d0.astype(complex)}
        for d, v in ((h % n, dp), ((n - h) % n, dm)):
            out[d] = out[d] + v if d in out else v.astype(complex)
        return out

    def mul(A, B):  # diagonals of A B
        out = {}
        for a, va in A.items():
            for b, vb in B.items():
                d = (a + b) % n
                t = va * np.roll(vb, -a)
                out[d] = out[d] + t if d in out else t
        return out

    levels, at = [], 1
    for g in groups:
        M = None
        for k in range(g):
            S = stage(2 ** (at + k))
            M = S if M is None else (mul(M, S) if inverse else mul(S, M))
        levels.append(M)
        at += g
    if inverse:
        levels = levels[::-1]
    levels[0] = {d: v * scale for d, v in levels[0].items()}
    return levels


def level_bs(diags) -> int:
    """baby-step size of a factorised level: 8 x the smallest nonzero offset step, so its offsets m 2^a (|m| < 32)
    split into <= 8 baby and <= 8 giant rotations"""
    n_min = min((d & -d) for d in diags if d) if any(diags) else 1
    return 8 * n_min


class BlockChain:
    """ResNet-style conv blocks chained through bootstrapping at Set_hyp (bootstrapping "to chain
    blocks end to end"): y = RAConv(CAConv(x)^2) + x -- the ConvBlock (Alg. 3, the AESPA square between the
    two convs) plus the identity shortcut, whose ciphertext is first brought to the block's output scale
    and level -- and then `refresh`: the scale set to the bootstrapper's input scale (one level), ModRaise ...
    SlotToCoeff back to L' (R-SFFT, R-EVALMOD).  Only sequencing and scale bookkeeping here; every step is a C-ABI
    call."""

    def __init__(self, ctx, bt: Bootstrapper, boot_scale: float = 2.0**42):
        self.ctx, self.bt, self.boot_scale = ctx, bt, boot_scale
        self.top = ctx.n_q - 1

    def block(self, blk, ca_keys, ra_keys, ca_pts, ra_pts, x: CT, shortcut=()) -> CT:
        """y = RAConv(CAConv(x)^2) + s(x), s the identity or (a stride-2 block) the convs `shortcut` = [(ConvPlan,
        keys, weight pts at its input level), ...] applied in order; the shortcut branch is brought to the main
        branch's scale and level"""
        bt = self.bt
        mid, _, out_level = blk.levels(x.level)
        y = blk.run(ca_keys, ra_keys, bt.rlk, [x.t], x.level, ca_pts, ra_pts)
        assert len(y) == 1
        ys = x.scale * x.scale / bt.q[mid]  # CAConv and RAConv keep the scale; the square makes it s^2 / q_mid
        xs = [x.t]
        lv = x.level
        for plan, keys, pts in shortcut:
            xs, lv = plan.run(keys, xs, lv, pts), plan.out_level(lv)
        sc = bt._down(bt._rescaled_to(CT(xs[0], lv, x.scale), ys), out_level)
        return bt._add(CT(y[0], out_level, ys), sc)

    def refresh(self, x: CT) -> CT:
        bt = self.bt
        x = bt._down(bt._rescaled_to(x, self.boot_scale), 0)
        return bt.bootstrap(x.t, x.scale, self.top)


class ResNet20Convs:
    """The ResNet-20 (CIFAR-10) conv stack run end to end under encryption at Set_hyp through BlockChain (SURVEY 8(f)
    row 4): stem conv + square (+ a 1x1 identity RAConv for the format), then 3 stages of 3 blocks y = RAConv(CAConv(x)^2) + s(x) -- the first block of
    stages 2 and 3 a stride-2 CAConv (dsconv, R-DSCONV) with a 1x1 stride-2 conv (pconv, then a 1x1 identity RAConv
    for the format) on the shortcut -- with a
    bootstrap after every block but the last.  Layer shapes and plans as bench.R20_LAYERS (2D-gap
    (1,2) / (2,4) / (4,8)); no average pooling / FC (outside the conv path).  weights: the 21 conv kernels in order
    (stem, then per block CAConv, RAConv [, pconv])."""

    SPECS = {  # (ci, co, w, f, stride, wp, gap, m, d, algo)
        "stem": (3, 16, 32, 3, 1, 32, 1, 1, 2, "CA"),
        "s1_ca": (16, 16, 32, 3, 1, 32, 1, 1, 2, "CA"), "s1_ra": (16, 16, 32, 3, 1, 32, 1, 2, 1, "RA"),
        "s2_ds": (16, 32, 32, 3, 2, 32, 1, 1, 2, "CA"), "s2_pc": (16, 32, 32, 1, 2, 32, 1, 1, 2, "CA"),
        "s2_ca": (32, 32, 16, 3, 1, 32, 2, 2, 4, "CA"), "s2_ra": (32, 32, 16, 3, 1, 32, 2, 4, 2, "RA"),
        "s3_ds": (32, 64, 16, 3, 2, 32, 2, 2, 4, "CA"), "s3_pc": (32, 64, 16, 1, 2, 32, 2, 2, 4, "CA"),
        "s3_ca": (64, 64, 8, 3, 1, 32, 4, 4, 8, "CA"), "s3_ra": (64, 64, 8, 3, 1, 32, 4, 8, 4, "RA"),
        # the pconv shortcut leaves RA(2d, 2m) (8 ciphertexts, R-DSCONV); a 1x1 RAConv with identity weights turns
        # it into the block output's CA(m, d) (1 ciphertext) so that the two branches add slot by slot
        "s2_id": (32, 32, 16, 1, 1, 32, 2, 4, 2, "RA"), "s3_id": (64, 64, 8, 1, 1, 32, 4, 8, 4, "RA"),
        # the same after the stem: its RA(2,1) output (8 ciphertexts) into the first block's CA(1,2)
        "s1_id": (16, 16, 32, 1, 1, 32, 1, 2, 1, "RA"),
    }
    # blocks: (CAConv, RAConv, shortcut conv or None)
    BLOCKS = [("s1_ca", "s1_ra", None)] * 3 + [("s2_ds", "s2_ra", ("s2_pc", "s2_id"))] + \
        [("s2_ca", "s2_ra", None)] * 2 + [("s3_ds", "s3_ra", ("s3_pc", "s3_id"))] + [("s3_ca", "s3_ra", None)] * 2

    def __init__(self, ctx, chain: BlockChain, weights, keyfn, level: int = 6):
        from . import ConvBlock, ConvPlan
        self.ctx, self.chain, self.level = ctx, chain, level
        self.plans = {k: ConvPlan(ctx, *v) for k, v in self.SPECS.items()}
        self.keys = {}
        for p in self.plans.values():
            for r in p.rots:
                if r not in self.keys:
                    self.keys[r] = keyfn(r)
        w = iter(weights)
        # the stem, its square and the identity RAConv into CA(1,2) as one ConvBlock; the client encrypts above L'
        # so that they land on L' (a fresh ciphertext may start at any level; every block then starts at L', the
        # level a bootstrap returns to)
        self.stem = ConvBlock(ctx, self.plans["stem"], self.plans["s1_id"])
        self.input_level = next(lv for lv in range(level, ctx.n_q) if self.stem.levels(lv)[2] == level)
        _, id_level, _ = self.stem.levels(self.input_level)
        self.stem_pts = self.plans["stem"].encode_weights(next(w), self.input_level)
        self.id_pts = self.plans["s1_id"].encode_weights(np.eye(16).reshape(16, 16, 1, 1), id_level)
        self.blocks = []
        lv = level
        for ca, ra, sc in self.BLOCKS:
            blk = ConvBlock(ctx, self.plans[ca], self.plans[ra])
            _, ra_level, _ = blk.levels(lv)
            cap = self.plans[ca].encode_weights(next(w), lv)
            rap = self.plans[ra].encode_weights(next(w), ra_level)
            scp = []
            if sc:
                pc, idn = self.plans[sc[0]], self.plans[sc[1]]
                co = self.SPECS[sc[1]][1]
                scp = [(pc, pc.encode_weights(next(w), lv)),
                       (idn, idn.encode_weights(np.eye(co).reshape(co, co, 1, 1), pc.out_level(lv)))]
            self.blocks.append((blk, cap, rap, scp, lv))

    def run(self, x: CT) -> CT:
        """x: the packed image, encrypted at self.input_level"""
        bt = self.chain.bt
        mid, _, out = self.stem.levels(x.level)
        # the stem conv, its activation (AESPA square), the identity RAConv (format only)
        y = self.stem.run(self.keys, self.keys, bt.rlk, [x.t], x.level, self.stem_pts, self.id_pts)
        y = CT(y[0], out, x.scale * x.scale / bt.q[mid])
        for i, (blk, cap, rap, scp, lv) in enumerate(self.blocks):
            assert y.level == lv
            y = self.chain.block(blk, self.keys, self.keys, cap, rap, y, shortcut=[(p, self.keys, w) for p, w in scp])
            if i + 1 < len(self.blocks):
                y = self.chain.refresh(y)
        return y
