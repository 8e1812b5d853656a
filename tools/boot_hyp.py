"""Time the Set_hyp bootstrap alone (bench.bench_bootstrap_set_hyp) and print its JSON; with --families, also one
bootstrap's device time per kernel family (CUDA events around every launch, so the sum exceeds the wall time)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2302_02407_b200 as hy  # noqa: E402
import synth  # noqa: E402

ctx = hy.Context(**synth.PARAMS["hyp"], device=0, max_batch=int(os.environ.get("HY_BENCH_BATCH", "64")))
args = [a for a in sys.argv[1:] if not a.startswith("--")]
print(json.dumps(bench.bench_bootstrap_set_hyp(ctx, int(args[0]) if args else 3), indent=1))
if "--families" in sys.argv:
    import math

    import numpy as np

    from paper_2302_02407_b200.boot import Bootstrapper, level_bs, sfft_levels, transform_rots
    sk, ek = synth.SEED_SK, synth.SEED_EVK
    N, top = ctx.N, ctx.n_q - 1
    K = float(ctx.moduli[0]) / 2**42
    cts = sfft_levels(N, [5, 5, 5], inverse=True, scale=0.5)
    stc = sfft_levels(N, [5, 5, 5], scale=K / (2 * math.pi))
    bs = ([level_bs(D) for D in cts], [level_bs(D) for D in stc])
    rots = sorted(set(transform_rots(ctx, cts, bs[0])) | set(transform_rots(ctx, stc, bs[1])))
    cheb = np.polynomial.chebyshev.chebinterpolate(lambda x: np.cos(12.0 * x), 30)
    cheb[1::2] = 0.0
    bt = Bootstrapper(ctx, cts, stc, bs, cheb, 4, 12.0, {r: ctx.keygen_rot(sk, ek, r) for r in rots},
                      ctx.keygen_galois(sk, ek, 2 * N - 1), ctx.keygen_relin(sk, ek))
    ct0 = ctx.level_down(ctx.encrypt(sk, 1, 6, ctx.encode(synth.slots_uniform(6, ctx.n), 2**42, top), top), top, 0)
    bt.bootstrap(ct0, 2.0**42, top)
    torch.cuda.synchronize()
    ctx.time_kernels(sum(ctx.FAMILIES.values()))
    bt.bootstrap(ct0, 2.0**42, top)
    torch.cuda.synchronize()
    for fn, fm in ctx.FAMILIES.items():
        ms, n, _ = ctx.kernel_times(fm)
        if n:
            print(f"{fn:8s} {ms:7.3f} ms {n:5d} launches")
    ctx.time_kernels(0)
