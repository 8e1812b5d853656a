"""Host issue time vs device time of one conv layer run (is the layer launch-bound?)."""
import sys, time
import torch
sys.path.insert(0, ".")
import bench, synth
import paper_2302_02407_b200 as hy

ctx = hy.Context(**synth.PARAMS["hyp"])
for name, spec, mult in bench.R18_LAYERS[:2] + bench.R20_LAYERS[:3]:
    ci, co, w, f, s, wp, g, m, d, algo = spec[:10]
    S = spec[10] if len(spec) > 10 else 1
    p = hy.ConvPlan(ctx, ci, co, w, f, s, wp, g, m, d, algo, S=S)
    level = bench.CA_LEVEL if algo == "CA" else bench.RA_LEVEL
    keys = {r: ctx.keygen_rot(3, 5, r) for r in p.rots}
    K = synth.conv_weight(7, co, ci, f)
    pts = p.encode_weights(K, level)
    cts = [ctx.encrypt(3, 9, i, ctx.encode(synth.slots_uniform(i, ctx.n), 2.0 ** 42, level), level) for i in range(p.n_in)]
    outs = [ctx.empty(*ctx.ct_shape(p.out_level(level))) for _ in range(p.n_out)]
    scratch = p.scratch(level)
    evks = [keys[r] for r in p.rots]
    for _ in range(2):
        p.run(evks, cts, level, pts, scratch, 0, p.n_out, outs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    p.run(evks, cts, level, pts, scratch, 0, p.n_out, outs)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:10s} issue {1000*(t1-t0):8.2f} ms   device {e0.elapsed_time(e1):8.2f} ms")
    del pts, cts, outs, scratch
    torch.cuda.empty_cache()
