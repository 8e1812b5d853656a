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
