"""Multi-GPU policy for HyPHEN conv layers.

Output ciphertexts of a conv layer are independent given its inputs, so a layer
is sharded by contiguous output ranges [begin, end) (hy_caconv / hy_raconv
`out_begin` / `out_end`) and the shards are all-gathered over the process group
(NCCL over NVLink on B200, gloo in the CPU tests).  Modular arithmetic is exact,
so the gathered result equals the single-GPU result bit for bit.
"""
from __future__ import annotations


def shard(n: int, rank: int, world: int) -> tuple[int, int]:
    """Balanced contiguous range of n items owned by `rank` (the first n % world ranks get one extra)."""
    base, extra = divmod(n, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def all_gather_cts(local: list, n_total: int, like, group=None) -> list:
    """All-gather per-rank lists of equally shaped ciphertext tensors into the full ordered list.

    local: this rank's outputs, in order; n_total: outputs over all ranks; like: a tensor with the
    ciphertext shape/dtype/device (used for padding).  Ranks own shard(n_total, r, world) each.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    sizes = [shard(n_total, r, world) for r in range(world)]
    cap = max(e - b for b, e in sizes)
    assert len(local) == sizes[rank][1] - sizes[rank][0]
    send = torch.zeros((cap,) + tuple(like.shape), dtype=like.dtype, device=like.device)
    for i, t in enumerate(local):
        send[i].copy_(t)
    recv = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(recv, send, group=group)
    out = []
    for r, (b, e) in enumerate(sizes):
        out.extend(recv[r][i] for i in range(e - b))
    return out


def tap_sharded(partial, finish, n_taps: int, group=None):
    """The exchange step of a tap-sharded RAConv output: this rank computes the lazy-sum
    state of its contiguous tap range, `partial(tap_begin, tap_end) -> int64 tensor`, the states are summed with
    one all-reduce, and `finish(state)` turns the sum into the output on every rank (modular sums are exact and
    order-free, so the result is bit-identical to the single-GPU one)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    b, e = shard(n_taps, rank, world)
    state = partial(b, e)
    dist.all_reduce(state, op=dist.ReduceOp.SUM, group=group)
    return finish(state)


def raconv_tap_sharded(plan, evks, cts, level, pts, out_index: int, scratch=None, group=None):
    """One output of an RAConv layer with its f^2 taps sharded over the ranks (include/hyphen.h
    hy_raconv_partial / hy_raconv_finish): for layers with fewer output ciphertexts than GPUs (ResNet-20
    RAConv: one output)."""
    scratch = plan.scratch(level) if scratch is None else scratch
    state = plan.partial_state(level)

    def partial(b, e):
        return plan.raconv_partial(evks, cts, level, pts, out_index, b, e, state, scratch)

    def finish(st):
        return plan.raconv_finish(evks, level, pts, st, out_index, scratch=scratch)

    return tap_sharded(partial, finish, plan.f * plan.f, group)


def caconv_slide_sharded(plan, evks, cts, level, pts, scratch=None, group=None):
    """A CAConv layer with its Slide_f sharded by input (include/hyphen.h hy_caconv_slide / hy_caconv_slid): each
    rank slides its contiguous input range, the slid ciphertexts are all-gathered (every output needs all of
    them), each rank computes its contiguous output range from the full slid set, and the outputs are
    all-gathered.  Modular arithmetic is exact and order-free, so the result is bit-identical to one GPU
    (Slide is no longer repeated on every rank)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    f2 = plan.f * plan.f
    ib, ie = shard(plan.n_in, rank, world)
    like = cts[0]
    mine = plan.slide(evks, cts, level, ib, ie)
    # all-gather of variable input ranges: pad every rank's block to the largest
    cap = max(e - b for b, e in (shard(plan.n_in, r, world) for r in range(world))) * f2
    send = torch.zeros((cap,) + tuple(like.shape), dtype=like.dtype, device=like.device)
    if mine.shape[0]:
        send[: mine.shape[0]].copy_(mine)
    recv = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(recv, send, group=group)
    slid = torch.cat([recv[r][: (e - b) * f2] for r, (b, e) in
                      enumerate(shard(plan.n_in, r, world) for r in range(world))], 0)
    ob, oe = shard(plan.n_out, rank, world)
    local = plan.run_slid(evks, slid, level, pts, scratch, ob, oe) if oe > ob else []
    lo = plan.out_level(level)
    return all_gather_cts(local, plan.n_out, plan.ctx.empty(*plan.ctx.ct_shape(lo)), group)
