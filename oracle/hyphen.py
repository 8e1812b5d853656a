"""HyPHEN convolution layers, oracle side -- TEST INFRASTRUCTURE ONLY.

Plain numpy statement of the paper's data formats and convolution algorithms
(P:n = PAPER.md line n), the plans they imply (rotation amounts, weight and
mask plaintext slot vectors), a float slot simulator that runs a plan on
cleartext vectors, and the encrypted execution of the same plan on the CKKS
oracle (oracle.Oracle).  Shares no code with the CUDA product.

Formats: pi_CA = {C_a, H, W, R_g, C_g}, pi_RA = {R_a, H, W, C_g, R_g};
2D gap packing: C_g (m multiplexed channels) and R_g (d duplicates)
live inside the stride gap and swap roles at every convolution.

Concrete slot layout (reading R-LAYOUT; the paper's figures are lost):
  W_p  physical image width (power of two, >= logical width), I = W_p^2
  g    cumulative stride gap, logical pixel (h, w) anchored at (h g, w g)
  cell kappa in [0, m d) = (g_c, g_r, e_idx) low->high: offset g_c + g_r W_p + e_idx I,
       e = m d / g^2 extra image sub-blocks per channel block
  B = e I slots per channel block, c_n = n / B blocks
  slot(b, h, w, kappa) = b B + e_idx I + (h g + g_r) W_p + (w g + g_c)
  CA(m, d): mu = kappa % m (C_g), rho = kappa // m (R_g); ct i holds channel i c_n m + b m + mu
  RA(m, d): mu = kappa // d (C_g), rho = kappa % d (R_g); ct i holds channel i m + mu, every block
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


def ilog2(x: int) -> int:
    v = int(x).bit_length() - 1
    assert 1 << v == x, f"{x} is not a power of two"
    return v


# --------------------------------------------------------------------------- formats
@dataclass(frozen=True)
class Fmt:
    kind: str    # "CA" or "RA"
    n: int       # slots
    wp: int      # physical width W_p
    g: int       # gap
    m: int       # |C_g|
    d: int       # |R_g|
    S: int = 1   # PRCR row segments |S|; 1 = plain rows

    @property
    def I(self):
        return self.wp * self.wp

    @property
    def F(self):
        """slots per row segment (the PRCR fragment size)."""
        return self.I // self.S

    @property
    def e(self):
        e = self.m * self.d // (self.g * self.g)
        assert e >= 1 and e * self.g * self.g == self.m * self.d, "m d must be a multiple of g^2"
        return e

    @property
    def B(self):
        return self.e * self.I

    @property
    def cn(self):
        cn = self.n // self.B
        assert cn >= 1 and cn * self.B == self.n
        return cn

    def stride(self, bit: int) -> int:
        """slot distance of kappa bit `bit` (g_c bits, then g_r bits, then e bits)."""
        lg = ilog2(self.g)
        if bit < lg:
            return 1 << bit
        if bit < 2 * lg:
            return self.wp << (bit - lg)
        return self.I << (bit - 2 * lg)

    def decompose(self):
        """per slot: block b, logical pixel (h, w), cell kappa (rows stay at their natural positions
        under PRCR; only the channel occupying each row segment changes)."""
        s = np.arange(self.n)
        b, r = s // self.B, s % self.B
        e_idx, pr, pc = r // self.I, (r % self.I) // self.wp, r % self.wp
        h, gr, w, gc = pr // self.g, pr % self.g, pc // self.g, pc % self.g
        kappa = gc + self.g * (gr + self.g * e_idx)
        return b, h, w, kappa

    def segment(self):
        """global row-segment position G = b S + s of every slot (PRCR; requires e = 1)."""
        s = np.arange(self.n)
        return s // self.F

    def mu_rho(self, kappa):
        if self.kind == "CA":
            return kappa % self.m, kappa // self.m
        return kappa // self.d, kappa % self.d

    def channel(self, i: int):
        """channel held by every slot of ciphertext i (before the `< C` cut).
        pi_CA' (CA, S > 1, PRCR): ciphertexts come in families of S; member im of family k holds, at
        global segment G, row segment (G mod S) of channel k c_n S m + ((G + im) mod c_n S) m + mu --
        the fragments are organised circularly, so member im sees the family's weight
        plaintext rotated by im fragments (PRot)."""
        b, h, w, kappa = self.decompose()
        mu, _ = self.mu_rho(kappa)
        if self.kind == "CA":
            if self.S > 1:
                assert self.e == 1, "PRCR needs e = 1"
                fam, im = divmod(i, self.S)
                G = self.segment()
                return fam * self.cn * self.S * self.m + ((G + im) % (self.cn * self.S)) * self.m + mu
            return i * self.cn * self.m + b * self.m + mu
        return i * self.m + mu

    def n_ct(self, c: int) -> int:
        if self.kind == "CA" and self.S > 1:
            return self.S * -(-c // (self.cn * self.S * self.m))
        per = self.cn * self.m if self.kind == "CA" else self.m
        return -(-c // per)


def pack(X: np.ndarray, fmt: Fmt) -> list[np.ndarray]:
    """tensor [C][H][W] -> slot vectors in format fmt (zero padding elsewhere)."""
    C, H, W = X.shape
    b, h, w, kappa = fmt.decompose()
    valid = (h < H) & (w < W)
    out = []
    for i in range(fmt.n_ct(C)):
        ch = fmt.channel(i)
        v = np.zeros(fmt.n)
        ok = valid & (ch < C)
        v[ok] = X[ch[ok], h[ok], w[ok]]
        out.append(v)
    return out


def unpack(vs: list[np.ndarray], fmt: Fmt, C: int, H: int, W: int, rep: int = 0) -> np.ndarray:
    """slot vectors -> tensor, reading replica `rep` (R_g / R_a index 0 by default)."""
    b, h, w, kappa = fmt.decompose()
    mu, rho = fmt.mu_rho(kappa)
    X = np.full((C, H, W), np.nan)
    sel = (rho == rep) & (h < H) & (w < W)
    if fmt.kind == "RA":
        sel &= b == 0
    for i, v in enumerate(vs):
        ch = fmt.channel(i)
        ok = sel & (ch < C)
        X[ch[ok], h[ok], w[ok]] = v[ok]
    return X


def conv2d(X: np.ndarray, K: np.ndarray, stride: int = 1, bias=None) -> np.ndarray:
    """cross-correlation with zero padding (f-1)/2 (Fig. 2(a); Alg. 1)."""
    C, H, W = X.shape
    O, C2, f, _ = K.shape
    assert C2 == C
    pad = (f - 1) // 2
    Xp = np.zeros((C, H + 2 * pad, W + 2 * pad))
    Xp[:, pad:pad + H, pad:pad + W] = X
    Ho, Wo = (H + stride - 1) // stride, (W + stride - 1) // stride
    Y = np.zeros((O, Ho, Wo))
    for o in range(O):
        for c in range(C):
            for j1 in range(f):
                for j2 in range(f):
                    Y[o] += K[o, c, j1, j2] * Xp[c, j1:j1 + H:stride, j2:j2 + W:stride][:Ho, :Wo]
    if bias is not None:
        Y += np.asarray(bias)[:, None, None]
    return Y


# --------------------------------------------------------------------------- plans
@dataclass
class ConvSpec:
    ci: int
    co: int
    w: int          # input logical width (== height)
    f: int
    s: int          # stride 1 or 2
    wp: int         # physical width
    g: int          # input gap
    m: int          # CA: |C_g| of the input; RA: |C_g| of the input (m' = d of the CA stage)
    d: int
    algo: str       # "CA" or "RA"
    n: int = 32768
    S: int = 1      # PRCR segments |S|; 1 = no PRCR

    @property
    def pad(self):
        return (self.f - 1) // 2

    def check_prcr(self):
        """PRCR needs whole rows per segment: S | W_p / g, stride 1, and e = m d / g^2 = 1 (DESIGN R-PRCR)."""
        if self.S > 1:
            assert self.s == 1 and (self.wp // self.g) % self.S == 0, "PRCR: S must divide W_p / g, stride 1"
            assert self.m * self.d == self.g * self.g, "PRCR: needs e = 1"
            assert self.wp // self.g >= self.w + self.pad, "PRCR: needs >= pad zero rows/columns of padding"

    @property
    def wo(self):
        return (self.w + self.s - 1) // self.s


@dataclass
class Plan:
    """Everything a conv needs besides the ciphertexts: rotation amounts, weight and mask slot vectors."""
    spec: ConvSpec
    fin: Fmt
    fout: Fmt
    taps: list                 # rotation amount r_t per tap t = j1 f + j2 (Alg. 1 line 4, in slots)
    weights: dict              # CA: (j, i, t) -> vec ; RA: (o, i, t) -> vec (inversely rotated, Alg. 2)
    n_in: int
    n_groups: int              # CA: SISO output groups; RA: output cts
    n_out: int
    ras: list = field(default_factory=list)        # RaS over C_a (CA)
    ras_g: list = field(default_factory=list)      # RaS_g
    mask: np.ndarray | None = None                 # IR_g mask (0/1)
    ir_g: list = field(default_factory=list)       # IR_g replication rotations
    combine: int | None = None                     # dsconv: rotation merging two groups
    counts: dict = field(default_factory=dict)

    def wkey(self, grp: int, i: int, t: int):
        """(stored weight key, PRot amount) used for SISO group / output `grp`, input ct i, tap t.
        Without PRCR every (grp, i, t) has its own plaintext and no PRot.  With PRCR a family
        of S ciphertexts shares one plaintext P holding, per slot, the filter value of the channel at
        that global row segment (no pixel masks); the effective weight is PRot(P, shift) with
          CA input member im:  shift = r_t + im F   (P indexed by the source slot of the tap),
          RA output member im: shift = im F - r_t   (the inverse rotation of Alg. 2 folded in).
        Out-of-image sources read the zero padding; invalid output pixels are zeroed by the mask step
        (DESIGN R-PRCR)."""
        S = self.spec.S
        if S == 1:
            return (grp, i, t), 0
        if self.spec.algo == "CA":
            return (grp, i // S, t), self.taps[t] + (i % S) * self.fin.F
        return (grp // S, i, t), (grp % S) * self.fout.F - self.taps[t]

    def effective(self, grp: int, i: int, t: int):
        """the slot vector actually multiplied with (rotated) input i for group/output grp, tap t."""
        key, sh = self.wkey(grp, i, t)
        return rot(self.weights[key], sh)


def _tap(j1, j2, spec: ConvSpec, g: int):
    return (j1 - spec.pad) * g * spec.wp + (j2 - spec.pad) * g


def plan_caconv(spec: ConvSpec, K: np.ndarray, with_weights: bool = True) -> Plan:
    """CAConv: pi_CA(m, d) -> pi_RA.  SISO = Slide_f (hoisted) + MulFilter&Sum_f (Alg. 1),
    then RaS over C_a (cyclic, replicates), RaS_g over C_g, IR_g (mask + rotations).
    Stride 2 (dsconv/pconv, Fig. 2(d)): valid outputs at even pixels; IR_g merges two SISO groups
    into the doubled gap (DESIGN R-DSCONV)."""
    assert spec.algo == "CA" and spec.s in (1, 2)
    spec.check_prcr()
    fin = Fmt("CA", spec.n, spec.wp, spec.g, spec.m, spec.d, spec.S)
    lg = ilog2(spec.g)
    if spec.s == 1:
        fout = Fmt("RA", spec.n, spec.wp, spec.g, spec.d, spec.m, spec.S)
    else:
        assert spec.m == spec.g, "dsconv IR needs m == g (DESIGN R-DSCONV)"
        fout = Fmt("RA", spec.n, spec.wp, 2 * spec.g, 2 * spec.d, 2 * spec.m)
    cn, m, d = fin.cn, spec.m, spec.d
    n_in = fin.n_ct(spec.ci)
    n_groups = -(-spec.co // d)
    if spec.s == 2:
        n_groups += n_groups % 2
    b, h, w, kappa = fin.decompose()
    mu, rho = fin.mu_rho(kappa)
    taps = [_tap(j1, j2, spec, spec.g) for j1 in range(spec.f) for j2 in range(spec.f)]
    weights = {}
    if spec.s == 1:
        out_ok = (h < spec.wo) & (w < spec.wo)
    else:
        out_ok = (h % 2 == 0) & (w % 2 == 0) & (h // 2 < spec.wo) & (w // 2 < spec.wo)
    for j in range(n_groups if with_weights else 0):
        if spec.s == 1:
            o = j * d + rho
        else:
            # new ct J = j // 2 holds 2d channels; mu' = rho_low + 2^lg * (j & 1) + 2^(lg+1) * rho_high
            rho_lo, rho_hi = rho % spec.g, rho // spec.g
            mu_new = rho_lo + (spec.g * (j & 1)) + (2 * spec.g) * rho_hi
            o = (j // 2) * (2 * d) + mu_new
        if spec.S == 1:
            for i in range(n_in):
                c = i * cn * m + b * m + mu
                for t, (j1, j2) in enumerate((a, bb) for a in range(spec.f) for bb in range(spec.f)):
                    sh, sw = h + j1 - spec.pad, w + j2 - spec.pad
                    ok = out_ok & (sh >= 0) & (sh < spec.w) & (sw >= 0) & (sw < spec.w) & (c < spec.ci) & (o < spec.co)
                    v = np.zeros(spec.n)
                    v[ok] = K[o[ok], c[ok], j1, j2]
                    weights[(j, i, t)] = v
        else:
            # PRCR: one plaintext per family k in source coordinates: slot q holds the filter value of the
            # channel at global segment G(q) of member 0, i.e. k c_n S m + G m + mu (DESIGN R-PRCR)
            for k in range(n_in // spec.S):
                c = k * cn * spec.S * m + fin.segment() * m + mu
                ok = (c < spec.ci) & (o < spec.co)
                for t, (j1, j2) in enumerate((a, bb) for a in range(spec.f) for bb in range(spec.f)):
                    v = np.zeros(spec.n)
                    v[ok] = K[o[ok], c[ok], j1, j2]
                    weights[(j, k, t)] = v
    p = Plan(spec, fin, fout, taps, weights, n_in, n_groups, 0)
    p.ras = [fin.B << k for k in range(ilog2(cn))]
    p.ras_g = [fin.stride(k) for k in range(ilog2(m))]
    if spec.s == 1:
        p.n_out = n_groups
        if m > 1 or spec.S > 1:
            # IR_g mask (mu = 0); PRCR also zeroes the invalid output pixels here (DESIGN R-PRCR)
            keep = (mu == 0) & (out_ok if spec.S > 1 else True)
            p.mask = keep.astype(np.float64)
            p.ir_g = [-fin.stride(k) for k in range(ilog2(m))]
    else:
        p.n_out = n_groups // 2
        b2, h2, w2, k2 = fout.decompose()
        bits = [k for k in range(ilog2(m))] + [lg, 2 * lg + 1]
        sel = np.ones(spec.n, bool)
        for k in bits:
            sel &= ((k2 >> k) & 1) == 0
        p.mask = sel.astype(np.float64)
        p.combine = -fout.stride(2 * lg + 1)
        p.ir_g = [-fout.stride(k) for k in range(lg + 1)]
    n_slide = len([r for r in taps if r != 0]) * n_in
    p.counts = {"Slide": n_slide, "RaS": len(p.ras) * n_groups, "RaS_g": len(p.ras_g) * n_groups,
                "IR_g": len(p.ir_g) * p.n_out + (p.n_out if p.combine is not None else 0),
                "PMult": n_groups * n_in * spec.f * spec.f}
    return p


def plan_raconv(spec: ConvSpec, K: np.ndarray, with_weights: bool = True) -> Plan:
    """RAConv_Reorder: pi_RA(m', d') -> pi_CA(d', m').  MulFilter&Sum_{c_i} with
    inversely rotated plaintexts W' = Rot(W, -r_t) (DESIGN R-ALG2), then Slide_1&Sum_f as one lazy
    HRotSum, RaS_g and IR_g over the R_g bits of the output format."""
    assert spec.algo == "RA" and spec.s == 1
    spec.check_prcr()
    fin = Fmt("RA", spec.n, spec.wp, spec.g, spec.m, spec.d, spec.S)
    fout = Fmt("CA", spec.n, spec.wp, spec.g, spec.d, spec.m, spec.S)
    m_out, d_out = spec.d, spec.m
    cn = fout.cn
    n_in = fin.n_ct(spec.ci)
    n_out = fout.n_ct(spec.co)
    b, h, w, kappa = fout.decompose()
    mu, rho = fout.mu_rho(kappa)          # rho (R_g of the output) indexes the input's C_g
    taps = [_tap(j1, j2, spec, spec.g) for j1 in range(spec.f) for j2 in range(spec.f)]
    out_ok = (h < spec.wo) & (w < spec.wo)
    weights = {}
    if spec.S == 1:
        for o in range(n_out if with_weights else 0):
            oc = o * cn * m_out + b * m_out + mu
            for i in range(n_in):
                c = i * spec.m + rho
                for t, (j1, j2) in enumerate((a, bb) for a in range(spec.f) for bb in range(spec.f)):
                    sh, sw = h + j1 - spec.pad, w + j2 - spec.pad
                    ok = out_ok & (sh >= 0) & (sh < spec.w) & (sw >= 0) & (sw < spec.w) & (c < spec.ci) & (oc < spec.co)
                    v = np.zeros(spec.n)
                    v[ok] = K[oc[ok], c[ok], j1, j2]
                    weights[(o, i, t)] = np.roll(v, taps[t])   # W' = Rot_{-r_t}(W): W'[p] = W[p - r_t]
    else:
        # PRCR: one plaintext per output family k (member-0 channel view, no pixel masks); the
        # inverse rotation of Alg. 2 and the member's fragment shift become one PRot (DESIGN R-PRCR)
        for k in range(n_out // spec.S if with_weights else 0):
            oc = k * cn * spec.S * m_out + fout.segment() * m_out + mu
            for i in range(n_in):
                c = i * spec.m + rho
                ok = (c < spec.ci) & (oc < spec.co)
                for t, (j1, j2) in enumerate((a, bb) for a in range(spec.f) for bb in range(spec.f)):
                    v = np.zeros(spec.n)
                    v[ok] = K[oc[ok], c[ok], j1, j2]
                    weights[(k, i, t)] = v
    p = Plan(spec, fin, fout, taps, weights, n_in, n_out, n_out)
    p.ras_g = [fout.stride(ilog2(m_out) + k) for k in range(ilog2(d_out))]
    if d_out > 1 or spec.S > 1:
        keep = (rho == 0) & (out_ok if spec.S > 1 else True)
        p.mask = keep.astype(np.float64)
        p.ir_g = [-s for s in p.ras_g]
    p.counts = {"Slide": len([r for r in taps if r != 0]) * n_out, "RaS": 0, "RaS_g": len(p.ras_g) * n_out,
                "IR_g": len(p.ir_g) * n_out, "PMult": n_out * n_in * spec.f * spec.f}
    return p


# --------------------------------------------------------------------------- float slot simulator
def rot(v, r):
    """left cyclic rotation by r: out[p] = v[p + r]."""
    return np.roll(v, -r)


def bias_slots(plan: Plan, bias) -> list[np.ndarray]:
    """The layer's bias as output-format slot vectors (DESIGN R-BIAS; "BN fused into the conv"): the
    packing, in the output format, of the image B[c][h][w] = b[c] over the wo x wo output pixels.  Adding it to
    the conv's output ciphertexts (AddPt) turns conv2d(X, K) into conv2d(X, K) + b at every valid slot."""
    sp = plan.spec
    B = np.broadcast_to(np.asarray(bias, np.float64)[:, None, None], (sp.co, sp.wo, sp.wo))
    vs = pack(np.ascontiguousarray(B), plan.fout)
    return vs + [np.zeros(plan.fout.n)] * max(0, plan.n_out - len(vs))


def simulate(plan: Plan, xs: list[np.ndarray], bias=None) -> list[np.ndarray]:
    """Run the plan on cleartext slot vectors (exact rotations, float products); bias: added after the layer."""
    outs = _simulate(plan, xs)
    if bias is not None:
        outs = [v + b for v, b in zip(outs, bias_slots(plan, bias))]
    return outs


def _simulate(plan: Plan, xs: list[np.ndarray]) -> list[np.ndarray]:
    sp = plan.spec
    if sp.algo == "CA":
        slid = [[rot(x, r) for r in plan.taps] for x in xs]       # Slide_f per input (hoisted)
        groups = []
        for j in range(plan.n_groups):
            acc = np.zeros(sp.n)
            for i in range(plan.n_in):
                for t in range(len(plan.taps)):
                    acc = acc + slid[i][t] * plan.effective(j, i, t)
            for r in plan.ras:
                acc = acc + rot(acc, r)
            for r in plan.ras_g:
                acc = acc + rot(acc, r)
            groups.append(acc)
        if sp.s == 1:
            outs = []
            for acc in groups:
                if plan.mask is not None:
                    acc = acc * plan.mask
                    for r in plan.ir_g:
                        acc = acc + rot(acc, r)
                outs.append(acc)
            return outs
        outs = []
        for J in range(plan.n_out):
            a = groups[2 * J] * plan.mask
            bb = groups[2 * J + 1] * plan.mask
            y = a + rot(bb, plan.combine)
            for r in plan.ir_g:
                y = y + rot(y, r)
            outs.append(y)
        return outs
    outs = []
    for o in range(plan.n_out):
        accs = [sum(xs[i] * plan.effective(o, i, t) for i in range(plan.n_in)) for t in range(len(plan.taps))]
        out = sum(rot(a, r) for a, r in zip(accs, plan.taps))
        for r in plan.ras_g:
            out = out + rot(out, r)
        if plan.mask is not None:
            out = out * plan.mask
            for r in plan.ir_g:
                out = out + rot(out, r)
        outs.append(out)
    return outs


# --------------------------------------------------------------------------- limited key sets
class KeySet:
    """Loaded rotation keys and the synthesis of the others ("other irregular rotation keys used in
    IR are not loaded; instead, these rotation indices are synthesized using the already loaded key indices").
    Reading (DESIGN R-KEYSET): an amount r is synthesized as the shortest sequence of loaded amounts summing to r
    mod n -- breadth-first search from 0 over Z_n, the loaded amounts as edges in ascending order, FIFO queue,
    the first discovery of a node fixing its parent -- and HRot_r = HRot_{a_k} o ... o HRot_{a_1}."""

    def __init__(self, n: int, amounts):
        self.n = n
        self.loaded = sorted({int(a) % n for a in amounts} - {0})
        parent = {0: None}
        queue = [0]
        h = 0
        while h < len(queue):
            u = queue[h]
            h += 1
            for a in self.loaded:
                v = (u + a) % n
                if v not in parent:
                    parent[v] = (u, a)
                    queue.append(v)
        self.parent = parent

    def steps(self, r: int) -> list:
        v = int(r) % self.n
        out = []
        while v != 0:
            if v not in self.parent:
                raise KeyError(f"rotation {r} cannot be synthesized from the key set")
            u, a = self.parent[v]
            out.append(a)
            v = u
        return out[::-1]


def eff_counts(plan: "Plan", keyset: "KeySet") -> dict:
    """rotation counts with every synthesized rotation counted once per step ("eff. total")."""
    n = plan.fin.n

    def cost(rs):
        return sum(len(keyset.steps(r)) if r % n and r % n not in keyset.loaded else int(r % n != 0) for r in rs)

    c = dict(plan.counts)
    c["RaS"] = cost(plan.ras) * plan.n_groups
    c["RaS_g"] = cost(plan.ras_g) * plan.n_groups
    c["IR_g"] = cost(plan.ir_g) * plan.n_out + (cost([plan.combine]) * plan.n_out if plan.combine is not None else 0)
    return c


def keyset_amounts(plan: "Plan", keyset: "KeySet") -> list:
    """the loaded amounts a plan uses under a key set (Slide taps must be loaded: they are hoisted)."""
    n = plan.fin.n
    need = set()
    for r in plan.taps:
        if r % n:
            assert r % n in keyset.loaded, "Slide amounts must be loaded"
            need.add(r % n)
    for r in plan.ras + plan.ras_g + plan.ir_g + ([plan.combine] if plan.combine is not None else []):
        if r % n == 0:
            continue
        need |= {r % n} if r % n in keyset.loaded else set(keyset.steps(r))
    return sorted(need)


# --------------------------------------------------------------------------- encrypted execution
class EncConv:
    """Runs a plan on oracle ciphertexts.  Weight plaintexts are encoded at scale q_l of the
    level they are consumed at and masks at q_{l-1}, so each rescale returns the scale to
    the ciphertext scale exactly (DESIGN R-SCALE).  evks: rotation amount -> key."""

    def __init__(self, o, plan: Plan, evks: dict, bias=None, keyset: "KeySet | None" = None):
        """bias: optional per-output-channel bias [co], added by AddPt after the layer's last rescale at the
        output ciphertext's level and scale (DESIGN R-BIAS).  keyset: optional limited key set; rotations by
        amounts it does not load are synthesized step by step (DESIGN R-KEYSET)."""
        self.o, self.plan, self.evks, self.bias, self.keyset = o, plan, evks, bias, keyset

    def key(self, r):
        r %= self.o.n
        return self.evks[r]

    def hrot(self, ct, r):
        if r % self.o.n == 0:
            return ct
        if self.keyset is not None and r % self.o.n not in self.keyset.loaded:
            for a in self.keyset.steps(r):
                ct = self.o.hrot(ct, self.key(a), a)
            return ct
        return self.o.hrot(ct, self.key(r), r)

    def ras(self, acc, rs):
        for r in rs:
            acc = self.o.add(acc, self.hrot(acc, r))
        return acc

    def encode(self, v, level):
        return self.o.encode(v, self.o.q[level], level)

    def prot(self, pt, r):
        """PRot: plaintext rotation by r = the automorphism kappa_{5^r} of the plaintext polynomial,
        done the obvious way (iNTT, coefficient map, NTT) limb by limb."""
        import oracle as _o
        if r % self.o.n == 0:
            return pt
        k = self.o.galois_elt(r)
        data = np.stack([self.o.ntt(self.o.automorph_coeff(self.o.intt(pt.data[i], i), i, k), i)
                         for i in range(pt.level + 1)])
        return _o.Pt(data, pt.level, pt.scale)

    def weight(self, wpts, cache, grp, i, t):
        key, pr = self.plan.wkey(grp, i, t)
        if (key, pr) not in cache:
            cache[(key, pr)] = self.prot(wpts[key], pr)
        return cache[(key, pr)]

    def run(self, cts, outputs=None):
        """outputs: optional list of output ciphertext indices to compute (sampling); default all."""
        outs_wanted = list(range(self.plan.n_out)) if outputs is None else list(outputs)
        outs = self._run(cts, outs_wanted)
        if self.bias is None:
            return outs
        bs = bias_slots(self.plan, self.bias)
        res = []
        for j, c in zip(outs_wanted, outs):
            pt = self.o.encode(bs[j], int(round(c.scale)), c.level)
            res.append(self.o.add_pt(c, pt))
        return res

    def _run(self, cts, outs_wanted):
        o, p, sp = self.o, self.plan, self.plan.spec
        level = cts[0].level
        if sp.algo == "CA":
            grp = set(outs_wanted) if sp.s == 1 else {g for J in outs_wanted for g in (2 * J, 2 * J + 1)}
        else:
            grp = set(outs_wanted)
        need = {p.wkey(g, i, t)[0] for g in grp for i in range(p.n_in) for t in range(len(p.taps))}
        wpts = {k: self.encode(v, level) for k, v in p.weights.items() if k in need}
        cache = {}
        if sp.algo == "CA":
            rs = [r for r in p.taps]
            slid = []
            for x in cts:
                nz = [r for r in rs if r % o.n]
                rot_cts = dict(zip(nz, o.hrot_hoisted(x, [self.key(r) for r in nz], nz)))
                slid.append([rot_cts[r] if r % o.n else x for r in rs])
            groups = {}
            for j in sorted(grp):
                acc = None
                for i in range(p.n_in):
                    for t in range(len(rs)):
                        term = o.pmult(slid[i][t], self.weight(wpts, cache, j, i, t))
                        acc = term if acc is None else o.add(acc, term)
                acc = o.rescale(acc)
                acc = self.ras(acc, p.ras)
                acc = self.ras(acc, p.ras_g)
                groups[j] = acc
            if sp.s == 1:
                outs = []
                for j in outs_wanted:
                    acc = groups[j]
                    if p.mask is not None:
                        acc = o.rescale(o.pmult(acc, self.encode(p.mask, acc.level)))
                        acc = self.ras(acc, p.ir_g)
                    outs.append(acc)
                return outs
            outs = []
            for J in outs_wanted:
                lv = groups[2 * J].level
                mpt = self.encode(p.mask, lv)
                a = o.rescale(o.pmult(groups[2 * J], mpt))
                bb = o.rescale(o.pmult(groups[2 * J + 1], mpt))
                y = o.add(a, self.hrot(bb, p.combine))
                outs.append(self.ras(y, p.ir_g))
            return outs
        outs = []
        for oo in outs_wanted:
            accs = []
            for t in range(len(p.taps)):
                acc = None
                for i in range(p.n_in):
                    term = o.pmult(cts[i], self.weight(wpts, cache, oo, i, t))
                    acc = term if acc is None else o.add(acc, term)
                accs.append(acc)
            keys = [self.key(r) if r % o.n else None for r in p.taps]
            out = o.rescale(o.hrot_sum(accs, keys, p.taps))
            out = self.ras(out, p.ras_g)
            if p.mask is not None:
                out = o.rescale(o.pmult(out, self.encode(p.mask, out.level)))
                out = self.ras(out, p.ir_g)
            outs.append(out)
        return outs


def rotation_amounts(plan: Plan, n: int) -> list[int]:
    """distinct non-zero rotation amounts (mod n) the plan needs keys for."""
    rs = set(r % n for r in plan.taps) | set(r % n for r in plan.ras + plan.ras_g + plan.ir_g)
    if plan.combine is not None:
        rs.add(plan.combine % n)
    rs.discard(0)
    return sorted(rs)


# --------------------------------------------------------------------------- fused CA -> x^2 -> RA block
def simulate_block(ca: Plan, ra: Plan, xs: list[np.ndarray]) -> list[np.ndarray]:
    """Alg. 3 on cleartext slot vectors: CAConv, the AESPA activation after its coefficients are
    fused into the neighbouring layers -- a plain square x^2 -- then RAConv."""
    return simulate(ra, [v * v for v in simulate(ca, xs)])


def run_block_encrypted(o, ca: Plan, ra: Plan, ca_evks: dict, ra_evks: dict, rlk, cts):
    """Alg. 3 on ciphertexts: CAConv (all outputs), Square = MulCt + relinearization + rescale
    (one level), RAConv on the squared ciphertexts.  The paper interleaves the loops to bound the
    live ciphertexts (ct_4[l] += MulFilter&Sum(ct_3[j]) as each ct_3[j] is produced); modular sums do not
    depend on that order, so the composition computes the same limbs."""
    mid = EncConv(o, ca, ca_evks).run(cts)
    sq = [o.square(c, rlk) for c in mid]
    return EncConv(o, ra, ra_evks).run(sq)
