"""Key-switch noise per parameter set (diagnostic, DESIGN R-MODDOWN): max slot error of a fresh encryption, a
conjugation and a rotation at a few levels, relative to the scale."""
import sys, numpy as np, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2302_02407_b200 as hy, synth
SK, EK = synth.SEED_SK, synth.SEED_EVK
for name in ("boot", "hyp", "toy"):
    prm = synth.PARAMS[name]
    ctx = hy.Context(**prm, device=0)
    n, N = ctx.n, ctx.N
    z = synth.slots_uniform(7, n)
    for lv in sorted({ctx.n_q - 1, min(19, ctx.n_q - 1), 5 if ctx.n_q > 6 else 1}):
        sc = 2.0 ** prm["log_scale"]
        ct = ctx.encrypt(SK, 3, 9, ctx.encode(z, int(sc), lv), lv)
        e_fresh = np.abs(ctx.decode(ctx.decrypt(SK, ct, lv), lv, sc) - z).max()
        ck = ctx.keygen_galois(SK, EK, 2 * N - 1)
        cc = ctx.hrot_galois(ck, ct, lv, 2 * N - 1)
        e_conj = np.abs(ctx.decode(ctx.decrypt(SK, cc, lv), lv, sc) - np.conj(z)).max()
        rk = ctx.keygen_rot(SK, EK, 1)
        rr = ctx.hrot(rk, ct, lv, 1)
        e_rot = np.abs(ctx.decode(ctx.decrypt(SK, rr, lv), lv, sc) - np.roll(z, -1)).max()
        print(f"{name} level {lv}: fresh {e_fresh:.2e}  conj {e_conj:.2e}  rot {e_rot:.2e}  (x scale: {e_conj*sc:.3g})")
