"""Stage-by-stage error of the Set_hyp bootstrap (diagnostic): decrypts after CoeffToSlot, after the alpha1 step,
after EvalMod and at the end, against the exact values computed from the ModRaised plaintext."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2302_02407_b200 as hy  # noqa: E402
import synth  # noqa: E402
from oracle import boot as B  # noqa: E402
from paper_2302_02407_b200.boot import CT, Bootstrapper, level_bs, sfft_levels, transform_rots  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "hyp"
DL = 42 if name == "hyp" else 40
r, a = (4, 12.0) if name == "hyp" else (3, 8.0)
groups = [5, 5, 5] if name == "hyp" else [4, 5]
prm = synth.PARAMS[name]
ctx = hy.Context(**prm, device=0)
o = oracle.Oracle(**prm)
SK, EK = synth.SEED_SK, synth.SEED_EVK
N, n, top = ctx.N, ctx.n, ctx.n_q - 1
K = float(ctx.moduli[0]) / 2**DL
cts = sfft_levels(N, groups, inverse=True, scale=0.5)
stc = sfft_levels(N, groups, scale=K / (2 * math.pi))
bs = ([level_bs(D) for D in cts], [level_bs(D) for D in stc])
rots = sorted(set(transform_rots(ctx, cts, bs[0])) | set(transform_rots(ctx, stc, bs[1])))
keys = {rr: ctx.keygen_rot(SK, EK, rr) for rr in rots}
cheb = np.polynomial.chebyshev.chebinterpolate(lambda s: np.cos(a * s), 30)
cheb[1::2] = 0.0
bt = Bootstrapper(ctx, cts, stc, bs, cheb, r, a, keys, ctx.keygen_galois(SK, EK, 2 * N - 1), ctx.keygen_relin(SK, EK))
z = synth.slots_uniform(43, n)
ct0 = o.level_down(o.encrypt(SK, 14, 0, o.encode(z, 2**DL, top)), 0)
d0 = torch.from_numpy(ct0.data.view(np.int64)).cuda()


def dec(x: CT):
    return ctx.decode(ctx.decrypt(SK, x.t, x.level), x.level, x.scale)


up = CT(ctx.mod_raise(d0, top), top, 2.0**DL)
t = np.array(o.crt_coeffs(o.decrypt(SK, oracle.Ct(up.t.cpu().numpy().view(np.uint64), top, 2.0**DL)).data, top),
             dtype=float) / 2**DL
I = np.round(t / K)
print("max|I|", np.abs(I).max(), "max|t/Delta|", np.abs(t).max())
br = B.bit_reverse_perm(n)
u = (t[:n] + 1j * t[n:]) / 2
y = bt._lintrans(bt.cts, up)
got = dec(y)
print("CtS    max err", np.abs(got - u[br]).max(), " max|u|", np.abs(u).max())
alpha1 = 2.0 * math.pi / (K * (2 ** r) * a)
pt, s = bt._const(alpha1, float(bt.q[y.level]) * float(bt.q[y.level - 1]) / y.scale, y.level)
y2 = bt._rescale(bt._pmult(y, pt, s))
print("alpha1 max err", np.abs(dec(y2) - alpha1 * u[br]).max(), " scale", y2.scale)
yc = CT(ctx.hrot_galois(bt.conj_key, y2.t, y2.level, 2 * N - 1), y2.level, y2.scale)
print("conj   max err", np.abs(dec(yc) - np.conj(alpha1 * u[br])).max(), " scale", yc.scale)
sm = bt._add(y2, yc)
print("y+yc   max err", np.abs(dec(sm).real - alpha1 * t[:n][br]).max())
beta1 = -math.pi / (2.0 * (2 ** r) * a)
s_re = bt._add_const(bt._add(y2, yc), beta1)
want_s = alpha1 * t[:n][br] + beta1
print("s_re   max err", np.abs(dec(s_re).real - want_s).max(), " range", want_s.min(), want_s.max())
c = bt.eval_chebyshev(s_re, s_re.scale)
print("cheb   max err", np.abs(dec(c).real - np.cos(a * want_s)).max(), " level", c.level, "scale", c.scale)
for k in range(r):
    sq = bt._mul(c, c)
    c = bt._add_const(bt._add(sq, sq), -1.0)
    print(f"dbl{k}   max err", np.abs(dec(c).real - np.cos(a * 2 ** (k + 1) * want_s)).max(), " level", c.level,
          "scale", c.scale)
m = t - K * I
print("sine vs m: max |K/2pi sin(2pi t/K) - m|", np.abs(K / (2 * math.pi) * np.sin(2 * math.pi * t / K) - m).max())
out = bt.bootstrap(d0, 2.0**DL, top)
print("final  max rel err", np.abs(dec(out) - z).max() / np.abs(z).max(), "level", out.level)
