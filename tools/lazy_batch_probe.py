import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
import paper_2302_02407_b200 as hy
prm = synth.PARAMS["hyp"]
ctx = hy.Context(**prm, max_batch=64)
level = 6
rs = [1, 2, 3, 4, 5, 6, 7, 8] * 8
keys = {r: ctx.keygen_rot(synth.SEED_SK, synth.SEED_EVK, r) for r in set(rs)}
cts = [ctx.encrypt(synth.SEED_SK, 1, i, ctx.encode(synth.slots_uniform(i, ctx.n), 2**42, level), level) for i in range(64)]
out = [ctx.empty(*ctx.ct_shape(level)) for _ in range(8)]
def t(fn, k=10):
    for _ in range(3): fn()
    torch.cuda.synchronize(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): fn()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / k
def eight():
    for o in range(8):
        ctx.hrot_sum([keys[r] for r in rs[8*o:8*o+8]], cts[8*o:8*o+8], level, rs[8*o:8*o+8], out[o])
def one():
    ctx.hrot_sum([keys[r] for r in rs], cts, level, rs, out[0])
print("8 x sum(8):", round(t(eight), 3), "ms;  1 x sum(64):", round(t(one), 3), "ms")
