"""Multi-rank conv layers on the GPU ("G-GPU limbs = 1-GPU limbs, bit-identical").

Two spawned ranks share cuda:0 (gpurun and the round-end tests have one B200; NCCL needs one GPU per rank, so the
collectives run on gloo over host copies -- the same dist.py policy code the NCCL path runs).  Each rank runs its
shard through the C ABI -- hy_caconv on an output range, or hy_raconv_partial on a tap range -- the shards are
combined (all-gather / one int64 all-reduce + hy_raconv_finish), and every rank checks the combined ciphertexts
against its own single-rank run of the whole layer, limb for limb.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, pset, layer, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    try:
        import torch
        import torch.distributed as dist

        import paper_2302_02407_b200 as hy
        import synth
        from paper_2302_02407_b200.dist import all_gather_cts, caconv_slide_sharded, shard, tap_sharded
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        prm = synth.PARAMS[pset]
        ctx = hy.Context(**prm, device=0)
        sk, ek = synth.SEED_SK, synth.SEED_EVK
        ci, co, w, f, s, wp, g, m, d, algo, S = layer
        p = hy.ConvPlan(ctx, ci, co, w, f, s, wp, g, m, d, algo, S=S, bias=True)
        level = len(prm["q_bits"]) - 1 if pset == "toy" else (9 if algo == "CA" else 6)
        scale = 2 ** prm["log_scale"]
        cts = [ctx.encrypt(sk, 77, i, ctx.encode(synth.slots_uniform(700 + i, ctx.n), scale, level), level)
               for i in range(p.n_in)]
        evks = [ctx.keygen_rot(sk, ek, r) for r in p.rots]
        pts = p.encode_weights(synth.conv_weight(5, co, ci, f), level, bias=synth.conv_bias(6, co), bias_scale=scale)
        full = p.run(evks, cts, level, pts)           # this rank alone, the whole layer
        torch.cuda.synchronize()
        ok = True
        if algo == "CA" or p.n_out >= world:
            b, e = shard(p.n_out, rank, world)
            mine = p.run(evks, cts, level, pts, out_begin=b, out_end=e) if e > b else []
            got = all_gather_cts([t.cpu() for t in mine], p.n_out, full[0].cpu())
            ok &= len(got) == p.n_out
            ok &= all(np.array_equal(a.numpy(), x.cpu().numpy()) for a, x in zip(got, full))
        if algo == "CA" and p.n_in >= 2:  # Slide sharded by input, slid ciphertexts all-gathered
            got = caconv_slide_sharded(p, evks, cts, level, pts)
            torch.cuda.synchronize()
            ok &= len(got) == p.n_out
            ok &= all(np.array_equal(a.cpu().numpy(), x.cpu().numpy()) for a, x in zip(got, full))
        if algo == "RA":
            scratch = p.scratch(level)
            for j in range(p.n_out):
                state = p.partial_state(level)

                def partial(tb, te):
                    return p.raconv_partial(evks, cts, level, pts, j, tb, te, state, scratch).cpu()

                def finish(st):
                    return p.raconv_finish(evks, level, pts, st.to(state.device), j, scratch=scratch)

                out = tap_sharded(partial, finish, f * f)
                torch.cuda.synchronize()
                ok &= np.array_equal(out.cpu().numpy(), full[j].cpu().numpy())
        q.put((rank, bool(ok), ""))
        dist.destroy_process_group()
    except Exception as ex:  # noqa: BLE001 -- reported to the parent
        import traceback
        q.put((rank, False, traceback.format_exc()[-2000:]))


LAYERS = {
    # toy (N = 2^12): CAConv with 4 output groups over 2 ranks; BASELINE config 1 RAConv (1 output: taps sharded)
    "toy_ca": ("toy", (8, 8, 8, 3, 1, 8, 1, 1, 2, "CA", 1)),
    "toy_C1_ra": ("toy", (4, 4, 8, 3, 1, 8, 1, 1, 1, "RA", 1)),
    # toy PRCR CAConv with 2 input ciphertexts: output sharding and Slide sharding by input
    "toy_prcr_ca": ("toy", (64, 8, 6, 3, 1, 8, 1, 1, 1, "CA", 2)),
    # ResNet-18 stage-4 CAConv (8 inputs, 64 outputs, PRCR |S| = 8) at N = 2^16: both shardings
    "r18_L4_ca": ("hyp", (512, 512, 7, 3, 1, 64, 8, 8, 8, "CA", 8)),
    # Set_hyp (N = 2^16): ResNet-20 stage-3 CAConv (8 outputs) and RAConv (1 output, taps sharded), both with bias
    "r20_L3_ca": ("hyp", (64, 64, 8, 3, 1, 32, 4, 4, 8, "CA", 1)),
    "r20_L3_ra": ("hyp", (64, 64, 8, 3, 1, 32, 4, 8, 4, "RA", 1)),
}


@pytest.mark.parametrize("name", list(LAYERS))
def test_two_ranks_bit_identical(name):
    import torch.multiprocessing as mp
    pset, layer = LAYERS[name]
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, pset, layer, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=120)
    for rank, ok, err in res:
        assert ok, f"rank {rank}: {err}"
