"""Time one conv layer (ResNet-18 / ResNet-20 spec from bench.py) with a per-family breakdown, for ncu.

    python tools/prof_layer.py R18 L2_pconv [--ncu]     (--ncu: wrap one run in cudaProfilerStart/Stop)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2302_02407_b200 as hy  # noqa: E402
import synth  # noqa: E402

net, name = sys.argv[1], sys.argv[2]
layers = {n: sp for n, sp, _ in (bench.R18_LAYERS if net == "R18" else bench.R20_LAYERS)}
spec = layers[name]
ctx = hy.Context(**synth.PARAMS["hyp"], max_batch=32)
ci, co, w, f, s, wp, g, m, d, algo = spec[:10]
S = spec[10] if len(spec) > 10 else 1
p = hy.ConvPlan(ctx, ci, co, w, f, s, wp, g, m, d, algo, S=S)
level = bench.CA_LEVEL if algo == "CA" else bench.RA_LEVEL
keys = {r: ctx.keygen_rot(synth.SEED_SK, synth.SEED_EVK, r) for r in p.rots}
pts = p.encode_weights(synth.conv_weight(1, co, ci, f), level)
scale = 2 ** synth.PARAMS["hyp"]["log_scale"]
cts = [ctx.encrypt(synth.SEED_SK, 1, i, ctx.encode(synth.slots_uniform(i, ctx.n), scale, level), level)
       for i in range(p.n_in)]
scr = p.scratch(level)
outs = [ctx.empty(*ctx.ct_shape(p.out_level(level))) for _ in range(p.n_out)]
for _ in range(2):
    p.run(keys, cts, level, pts, scr, outs=outs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
p.run(keys, cts, level, pts, scr, outs=outs)
e1.record()
torch.cuda.synchronize()
ctx.time_kernels(sum(ctx.FAMILIES.values()))
if "--ncu" in sys.argv:
    torch.cuda.cudart().cudaProfilerStart()
p.run(keys, cts, level, pts, scr, outs=outs)
torch.cuda.synchronize()
if "--ncu" in sys.argv:
    torch.cuda.cudart().cudaProfilerStop()
print(f"{net} {name}: {e0.elapsed_time(e1):.3f} ms, weight pts {p.n_pt}, n_in {p.n_in}, n_out {p.n_out}")
for fn, fm in ctx.FAMILIES.items():
    t, n, b = ctx.kernel_times(fm)
    if n:
        print(f"  {fn:8s} {t:8.3f} ms {n:6d} launches {b / t / 1e6 if t else 0:8.1f} GB/s (algorithmic)")
ctx.time_kernels(0)
