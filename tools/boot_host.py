"""Host vs device time per Set_hyp bootstrap call, batched vs single MulCt in EvalMod (diagnostic); MB=<max_batch>."""
import os, sys, time, math
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import numpy as np, torch
import paper_2302_02407_b200 as hy, synth
from paper_2302_02407_b200.boot import Bootstrapper, level_bs, sfft_levels, transform_rots
ctx = hy.Context(**synth.PARAMS["hyp"], device=0, max_batch=int(os.environ.get("MB", "0")) or None)
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
bt.bootstrap(ct0, 2.0**42, top); torch.cuda.synchronize()
for mode in ("batch", "single", "batch"):
    if mode == "single":
        orig = bt._mul_many
        bt._mul_many = lambda As, Bs: [bt._mul(a, b) for a, b in zip(As, Bs)]
    else:
        bt.__dict__.pop("_mul_many", None)
    for rep in range(3):
        t0 = time.time(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); bt.bootstrap(ct0, 2.0**42, top); t1 = time.time(); e1.record(); torch.cuda.synchronize(); t2 = time.time()
        print(mode, f"host {1e3*(t1-t0):.1f} ms, gpu {e0.elapsed_time(e1):.1f} ms, wall {1e3*(t2-t0):.1f} ms, mem {torch.cuda.memory_allocated()/2**30:.1f} GiB reserved {torch.cuda.memory_reserved()/2**30:.1f}")
