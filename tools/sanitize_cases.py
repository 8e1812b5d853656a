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
    for spec in [(4, 4, 8, 3, 1, 8, 1, 1, 1, "RA"), (8, 8, 8, 3, 1, 8, 1, 1, 2, "CA"), (4, 8, 8, 3, 2, 8, 1, 1, 2, "CA")]:
        p = hy.ConvPlan(ctx, *spec, bias=True)
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


if __name__ == "__main__":
    toy()
    if "--toy-only" not in sys.argv:
        hyp()
