"""Stage-by-stage check of boot.ResNet20Convs against the plaintext network (diagnostic): decrypts after the stem
and after every block and refresh, and prints the error relative to the plaintext value's max."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2302_02407_b200 as hy  # noqa: E402
import synth  # noqa: E402
from oracle import hyphen as H  # noqa: E402
from paper_2302_02407_b200.boot import CT, BlockChain, Bootstrapper, ResNet20Convs, level_bs, sfft_levels, transform_rots  # noqa: E402,E501

SK, EK = synth.SEED_SK, synth.SEED_EVK
ctx = hy.Context(**synth.PARAMS["hyp"], device=0)
N, n = ctx.N, ctx.n
K = float(ctx.moduli[0]) / 2**42
cts = sfft_levels(N, [5, 5, 5], inverse=True, scale=0.5)
stc = sfft_levels(N, [5, 5, 5], scale=K / (2 * math.pi))
bs = ([level_bs(D) for D in cts], [level_bs(D) for D in stc])
rots = sorted(set(transform_rots(ctx, cts, bs[0])) | set(transform_rots(ctx, stc, bs[1])))
cheb = np.polynomial.chebyshev.chebinterpolate(lambda s: np.cos(12.0 * s), 30)
cheb[1::2] = 0.0
bt = Bootstrapper(ctx, cts, stc, bs, cheb, 4, 12.0, {r: ctx.keygen_rot(SK, EK, r) for r in rots},
                  ctx.keygen_galois(SK, EK, 2 * N - 1), ctx.keygen_relin(SK, EK))
shapes = [((16, 3), 3)] + [((16, 16), 3)] * 6 + [((32, 16), 3), ((32, 32), 3), ((32, 16), 1)] + \
    [((32, 32), 3)] * 4 + [((64, 32), 3), ((64, 64), 3), ((64, 32), 1)] + [((64, 64), 3)] * 4
Ws = [synth.conv_weight(200 + i, co, ci, f) * 0.5 for i, ((co, ci), f) in enumerate(shapes)]
chain = BlockChain(ctx, bt)
net = ResNet20Convs(ctx, chain, Ws, lambda r: ctx.keygen_rot(SK, EK, r))
sp = ResNet20Convs.SPECS
X = synth.image(300, 3, 32)
fmt = {k: (H.plan_caconv if v[9] == "CA" else H.plan_raconv)(H.ConvSpec(*v, n=n),
                                                                synth.conv_weight(1, v[1], v[0], v[3]))
       for k, v in sp.items()}
L = net.input_level
x = CT(ctx.encrypt(SK, 32, 0, ctx.encode(H.pack(X, fmt["stem"].fin)[0], 2**42, L), L), L, 2.0**42)


def check(tag, y: CT, f, C, W, ref):
    dec = np.real(ctx.decode(ctx.decrypt(SK, y.t, y.level), y.level, y.scale))
    got = H.unpack([dec], f, C, W, W)
    print(f"{tag:18s} level {y.level:2d} scale 2^{math.log2(y.scale):.2f}  rel err "
          f"{np.max(np.abs(got - ref)) / np.max(np.abs(ref)):.2e}  max|ref| {np.max(np.abs(ref)):.3f}", flush=True)


mid, _, out = net.stem.levels(x.level)
y = net.stem.run(net.keys, net.keys, bt.rlk, [x.t], x.level, net.stem_pts, net.id_pts)
y = CT(y[0], out, x.scale * x.scale / bt.q[mid])
it = iter(Ws)
Y = H.conv2d(X, next(it)) ** 2
check("stem^2 (CA(1,2))", y, fmt["s1_id"].fout, 16, 32, Y)
for i, ((blk, cap, rap, scp, lv), (ca, ra, sc)) in enumerate(zip(net.blocks, ResNet20Convs.BLOCKS)):
    Kc, Kr = next(it), next(it)
    stride = sp[ca][4]
    main = H.conv2d(H.conv2d(Y, Kc, stride) ** 2, Kr)
    Y = main + (H.conv2d(Y, next(it), 2) if sc else Y)
    y = chain.block(blk, net.keys, net.keys, cap, rap, y, shortcut=[(p, net.keys, w) for p, w in scp])
    C, W = sp[ra][1], sp[ra][2]
    check(f"block {i} ({ca})", y, fmt[ra].fout, C, W, Y)
    if i + 1 < len(net.blocks):
        y = chain.refresh(y)
        check(f"  refresh {i}", y, fmt[ra].fout, C, W, Y)
