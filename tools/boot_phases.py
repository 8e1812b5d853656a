"""Device time of each bootstrapping phase at Set_hyp (diagnostic)."""
import os, sys, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2302_02407_b200 as hy, synth
from paper_2302_02407_b200.boot import CT, Bootstrapper, level_bs, sfft_levels, transform_rots
ctx = hy.Context(**synth.PARAMS["hyp"], device=0)
sk, ek = synth.SEED_SK, synth.SEED_EVK
N, top = ctx.N, ctx.n_q - 1
K = float(ctx.moduli[0]) / 2**42
cts = sfft_levels(N, [5, 5, 5], inverse=True, scale=0.5)
stc = sfft_levels(N, [5, 5, 5], scale=K / (2 * math.pi))
bs = ([level_bs(D) for D in cts], [level_bs(D) for D in stc])
rots = sorted(set(transform_rots(ctx, cts, bs[0])) | set(transform_rots(ctx, stc, bs[1])))
cheb = np.polynomial.chebyshev.chebinterpolate(lambda x: np.cos(12.0 * x), 30); cheb[1::2] = 0.0
bt = Bootstrapper(ctx, cts, stc, bs, cheb, 4, 12.0, {r: ctx.keygen_rot(sk, ek, r) for r in rots},
                  ctx.keygen_galois(sk, ek, 2 * N - 1), ctx.keygen_relin(sk, ek))
ct0 = ctx.level_down(ctx.encrypt(sk, 1, 6, ctx.encode(synth.slots_uniform(6, ctx.n), 2**42, top), top), top, 0)
for _ in range(2): bt.bootstrap(ct0, 2.0**42, top)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
# replicate bootstrap() with events
r, a = bt.r, bt.a
Kk = float(bt.q[0]) / 2**42
alpha1 = 2.0 * math.pi / (Kk * (2 ** r) * a); beta1 = -math.pi / (2.0 * (2 ** r) * a)
ev[0].record()
up = CT(ctx.mod_raise(ct0, top), top, 2.0**42)
ev[1].record()
y = bt._lintrans(bt.cts, up)
ev[2].record()
pt, s = bt._const(alpha1, float(bt.q[y.level]) * float(bt.q[y.level - 1]) / y.scale, y.level)
y = bt._rescale(bt._pmult(y, pt, s))
yc = CT(ctx.hrot_galois(bt.conj_key, y.t, y.level, 2 * N - 1), y.level, y.scale)
s_re = bt._add_const(bt._add(y, yc), beta1)
d = bt._sub(y, yc)
s_im = bt._add_const(CT(ctx.pmult(d.t, bt._monomial(-1, d.level), d.level), d.level, d.scale), beta1)
ev[3].record()
e_re, e_im = bt.eval_mod_many([s_re, s_im])
ev[4].record()
ie = CT(ctx.pmult(e_im.t, bt._monomial(1, e_im.level), e_im.level), e_im.level, e_im.scale)
z = bt._add(e_re, ie)
out = bt._lintrans(bt.stc, z)
ev[5].record()
torch.cuda.synchronize()
names = ["ModRaise", "CoeffToSlot", "alpha1+conj split", "EvalMod", "SlotToCoeff"]
for i, nm in enumerate(names):
    print(f"{nm:18s} {ev[i].elapsed_time(ev[i+1]):7.3f} ms")
