"""Multi-process (world_size 2, gloo, CPU) checks of the conv sharding policy:
shards partition the outputs, and the all-gather reassembles every rank's
ciphertexts in global order, bit for bit."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2302_02407_b200.dist import all_gather_cts, shard, tap_sharded


def test_shard_partitions():
    for n in [0, 1, 3, 8, 9, 64]:
        for world in [1, 2, 3, 4, 8]:
            ranges = [shard(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (b0, e0), (b1, e1) in zip(ranges, ranges[1:]):
                assert e0 == b1 and e0 >= b0
            sizes = [e - b for b, e in ranges]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shape = (2, 3, 16)

    def ct(i):  # the "ciphertext" output i as a deterministic function of i (uint64 residues as int64)
        g = torch.Generator().manual_seed(1000 + i)
        return torch.randint(0, 2**47, shape, generator=g, dtype=torch.int64)

    b, e = shard(n_total, rank, world)
    local = [ct(i) for i in range(b, e)]
    full = all_gather_cts(local, n_total, torch.zeros(shape, dtype=torch.int64))
    ok = len(full) == n_total and all(torch.equal(full[i], ct(i)) for i in range(n_total))
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_total", [1, 3, 8])
def test_all_gather_world2(n_total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_total, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = dict(q.get() for _ in range(2))
    assert res == {0: True, 1: True}


Q = 281474976710597  # a 48-bit prime (residues < 2^48, as in the product's chain)


def _tap_value(t):  # the lazy-sum state contributed by tap t alone (deterministic residues)
    g = torch.Generator().manual_seed(500 + t)
    return torch.randint(0, Q, (2, 3, 16), generator=g, dtype=torch.int64)


def _partial(b, e):  # the state of taps [b, e): canonical sum mod Q (what hy_raconv_partial returns)
    st = torch.zeros((2, 3, 16), dtype=torch.int64)
    for t in range(b, e):
        st = (st + _tap_value(t)) % Q
    return st


def _tap_worker(rank, world, port, n_taps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    got = tap_sharded(_partial, lambda st: st % Q, n_taps)  # finish: reduce the integer sum mod Q
    q.put((rank, bool(torch.equal(got, _partial(0, n_taps)))))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n_taps", [(2, 9), (2, 1), (3, 9)])
def test_tap_sharded_allreduce(world, n_taps):
    """RAConv tap sharding: per-rank partial states summed by one all-reduce and reduced mod q equal the
    single-rank state for every rank (including a rank with an empty tap range)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tap_worker, args=(r, world, port, n_taps, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = dict(q.get() for _ in range(world))
    assert res == {r: True for r in range(world)}
