"""Small invocations of every kernel family for compute-sanitizer (racecheck / synccheck / memcheck):
BASELINE config 1 (toy RAConv 4->4), a toy CAConv and stride-2 dsconv (k_pmult_ring / k_pmult_block, hoisted Slide,
RaS, mask, combine), and at Set_hyp a plain HRot batch, a hoisted pair and a lazy HRotSum at level 23 (the TMA /
mbarrier ring kernels), plus a rescale.  Usage: compute-sanitizer --tool racecheck python tools/sanitize_cases.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2302_02407_b200 as hy  # noqa: E402
import synth  # noqa: E402

SK, EK = synth.SEED_SK, synth.SEED_EVK


def toy():
    prm = synth.PARAMS["toy"]
    ctx = hy.Context(**prm)
    for spec in [(4, 4, 8, 3, 1, 8, 1, 1, 1, "RA", 1), (8, 8, 8, 3, 1, 8, 1, 1, 2, "CA", 1),
                 (4, 8, 8, 3, 2, 8, 1, 1, 2, "CA", 1), (64, 8, 6, 3, 1, 8, 1, 1, 1, "CA", 2),
                 (8, 64, 6, 3, 1, 8, 1, 1, 1, "RA", 2)]:
        p = hy.ConvPlan(ctx, *spec[:10], S=spec[10], bias=True)
        level = 2
        cts = [ctx.encrypt(SK, 9, i, ctx.encode(synth.slots_uniform(i, ctx.n), 2**40, level), level)
               for i in range(p.n_in)]
        evks = {r: ctx.keygen_rot(SK, EK, r) for r in p.rots}
        pts = p.encode_weights(synth.conv_weight(1, spec[1], spec[0], spec[3]), level, bias=np.zeros(spec[1]),
                               bias_scale=2**40)
        p.run(evks, cts, level, pts)
    torch.cuda.synchronize()
    print("toy layers ok")


def hyp():
    prm = synth.PARAMS["hyp"]
    ctx = hy.Context(**prm, max_batch=2)
    level = 23
    rs = [1, -3]
    keys = [ctx.keygen_rot(SK, EK, r) for r in rs]
    cts = [ctx.encrypt(SK, 9, i, ctx.encode(synth.slots_uniform(i, ctx.n), 2**42, level), level) for i in range(2)]
    ctx.hrot_batch(keys, cts, level, rs)
    ctx.hrot_hoisted(keys, cts[0], level, rs)
    ctx.hrot_sum(keys, cts, level, rs)
    ctx.rescale(cts[0], level)
    torch.cuda.synchronize()
    print("hyp key switches ok")


def boot():
    """ModRaise, the BSGS transform (hoisted baby steps, MulFilter&Sum, lazy HRotSum), conjugation, MulCt, and the
    batched MulCt / rescale of the lockstep EvalMod"""
    prm = synth.PARAMS["boot"]
    ctx = hy.Context(**prm)
    top = len(prm["q_bits"]) - 1
    ct = ctx.encrypt(SK, 9, 0, ctx.encode(synth.slots_uniform(1, ctx.n), 2**40, top), top)
    up = ctx.mod_raise(ctx.level_down(ct, top, 0), top)
    lt = hy.LinTrans(ctx, [0, 1, 2, 5, 9, 33], 4)
    keys = {r: ctx.keygen_rot(SK, EK, r) for r in lt.rots}
    g = np.random.default_rng(2)
    y = lt.apply(keys, up, top, lt.encode([g.uniform(-1, 1, ctx.n) + 0j for _ in range(6)], top))
    ctx.hrot_galois(ctx.keygen_galois(SK, EK, 2 * ctx.N - 1), y, top - 1, 2 * ctx.N - 1)
    rlk = ctx.keygen_relin(SK, EK)
    ctx.mulct(rlk, y, y, top - 1)
    # bootstrapping's lockstep EvalMod: batched MulCt and batched rescale
    pr = ctx.mulct_batch(rlk, [y, up[:, : top].contiguous()], [y, y], top - 1)
    pr = ctx.pmult_batch(pr, ctx.encode(np.full(ctx.n, 0.5), 2**40, top - 1), top - 1)
    ctx.rescale_batch(pr, top - 1)
    torch.cuda.synchronize()
    print("boot steps ok")


if __name__ == "__main__":
    toy()
    boot()
    if "--toy-only" not in sys.argv:
        hyp()
