"""Run one conv layer (ResNet-18 L1_ca by default) inside a cudaProfilerStart/Stop region for an ncu launch list."""
import sys
import torch
sys.path.insert(0, ".")
import bench, synth
import paper_2302_02407_b200 as hy

which = sys.argv[1] if len(sys.argv) > 1 else "r18:L1_ca"
net, lname = which.split(":")
table = bench.R18_LAYERS if net == "r18" else bench.R20_LAYERS
ctx = hy.Context(**synth.PARAMS["hyp"], max_batch=64)  # as bench.py
name, spec, mult = next(l for l in table if l[0] == lname)
ci, co, w, f, s, wp, g, m, d, algo = spec[:10]
S = spec[10] if len(spec) > 10 else 1
p = hy.ConvPlan(ctx, ci, co, w, f, s, wp, g, m, d, algo, S=S)
level = bench.CA_LEVEL if algo == "CA" else bench.RA_LEVEL
keys = {r: ctx.keygen_rot(3, 5, r) for r in p.rots}
pts = p.encode_weights(synth.conv_weight(7, co, ci, f), level)
cts = [ctx.encrypt(3, 9, i, ctx.encode(synth.slots_uniform(i, ctx.n), 2.0 ** 42, level), level) for i in range(p.n_in)]
outs = [ctx.empty(*ctx.ct_shape(p.out_level(level))) for _ in range(p.n_out)]
scratch = p.scratch(level)
evks = [keys[r] for r in p.rots]
p.run(evks, cts, level, pts, scratch, 0, p.n_out, outs)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
p.run(evks, cts, level, pts, scratch, 0, p.n_out, outs)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
