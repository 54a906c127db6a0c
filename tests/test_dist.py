"""Multi-process (world_size 2, gloo, CPU) coverage of the sharded trainer's
host-side plumbing: contiguous minibatch shards, the wrapping int64
all-reduce + mod-q contract, and rank-owned refresh broadcast."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2210_02574_b200 import shard
        from paper_2210_02574_b200.ckks import params as P

        assert shard.world() == (rank, world)
        primes = P.get_preset("p16").ring.moduli_chain[:2]
        n_cts = 16
        lo, hi = shard.shard_range(n_cts, rank, world)
        rng = np.random.default_rng(123)
        # every "ciphertext gradient" (2 limbs x 32 coeffs), identical on all ranks
        grads = [np.stack([rng.integers(0, q, 32, dtype=np.uint64) for q in primes])
                 for _ in range(n_cts)]
        local = np.zeros_like(grads[0])
        for i in range(lo, hi):  # local fixed-order modular sum of this rank's shard
            local = np.stack([(local[j].astype(object) + grads[i][j]) % q
                              for j, q in enumerate(primes)]).astype(np.uint64)
        t = torch.from_numpy(local.view(np.int64).copy())
        dist.all_reduce(t, op=dist.ReduceOp.SUM)  # wraps mod 2^64
        reduced = t.numpy().view(np.uint64) % np.array(primes, dtype=np.uint64)[:, None]
        want = np.stack([sum(g[j].astype(object) for g in grads) % q
                         for j, q in enumerate(primes)]).astype(np.uint64)
        ok_sum = bool(np.array_equal(reduced, want))
        # refresh ownership + broadcast of the refreshed state
        owner_w, owner_u = shard.refresh_owner(0, world), shard.refresh_owner(1, world)
        w = torch.full((4,), 7 if rank == owner_w else -1, dtype=torch.int64)
        u = torch.full((4,), 9 if rank == owner_u else -1, dtype=torch.int64)
        dist.broadcast(w, src=owner_w)
        dist.broadcast(u, src=owner_u)
        out[rank] = (ok_sum, (lo, hi), int(w[0]), int(u[0]), owner_w != owner_u)
    finally:
        dist.destroy_process_group()


def test_two_rank_gradient_allreduce():
    world = 2
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert out[0][0] and out[1][0]
    assert out[0][1] == (0, 8) and out[1][1] == (8, 16)
    assert out[0][2] == out[1][2] == 7 and out[0][3] == out[1][3] == 9
    assert out[0][4]  # w and u refresh on different ranks


def test_class_groups_layout():
    """2-D (class x minibatch) layout of One-vs-Rest training over ranks."""
    from paper_2210_02574_b200 import shard

    assert shard.class_groups(4, 1) == [[0]] * 4
    assert shard.class_groups(4, 2) == [[0], [1], [0], [1]]
    assert shard.class_groups(4, 4) == [[0], [1], [2], [3]]
    assert shard.class_groups(4, 8) == [[0, 4], [1, 5], [2, 6], [3, 7]]
    assert shard.class_groups(3, 5) == [list(range(5))] * 3  # 1-D fallback
    for world in (1, 2, 4, 8):  # every rank trains something, every class has ranks
        g = shard.class_groups(4, world)
        assert sorted({r for m in g for r in m}) == list(range(world))
