"""Minibatch sharding across GPUs for encrypted training.

One process per GPU.  Each minibatch's ciphertexts are split contiguously
across ranks; every rank computes and locally sums its gradients, then the
level-1 gradient ciphertext is combined with one modular all-reduce: an NCCL
(or gloo) int64 SUM of residues followed by one `mod q` pass.  It is exact
when world_size * (q-1) < 2^64 for every prime q of the chain (checked;
true for 8 ranks and primes < 2^61): integer addition wraps modulo 2^64, so
the reduced value equals the reference's fixed-order modular sum
(logreg.py:382-384) bit for bit.
The two refreshes per minibatch (w and u) run on different ranks and are
broadcast back, so they overlap when world_size > 1.
"""

import numpy as np

from . import _dev
from . import _lib


def world(group=None):
    """(rank, size) in `group` (default: the world), (0, 1) without a process group."""
    try:
        import torch.distributed as dist
    except Exception:
        return 0, 1
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(group), dist.get_world_size(group)
    return 0, 1


def global_rank(group, rank):
    """Global rank of group-local `rank` (collectives take global source ranks)."""
    if group is None:
        return rank
    import torch.distributed as dist

    return dist.get_global_rank(group, rank)


def class_groups(n_models, world_size):
    """2-D (class x minibatch) layout of One-vs-Rest training over ranks
    (logreg.py:393-398: classes are independent): returns, per class, the
    ranks that train it.  world <= classes: classes dealt round-robin, one
    rank each; world a multiple of classes: world/classes ranks per class,
    sharding that class's minibatches; otherwise every rank trains every
    class (1-D minibatch sharding)."""
    if world_size <= 1:
        return [[0] for _ in range(n_models)]
    if world_size <= n_models:
        return [[c % world_size] for c in range(n_models)]
    if world_size % n_models == 0:
        return [[r for r in range(world_size) if r % n_models == c] for c in range(n_models)]
    return [list(range(world_size)) for _ in range(n_models)]


def shard_range(n_items, rank, world_size):
    """Contiguous [lo, hi) share of n_items for `rank` (balanced, order-preserving)."""
    base, extra = divmod(n_items, world_size)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def refresh_owner(role, world_size):
    """Rank that refreshes the weight (role 0) or momentum (role 1) ciphertext."""
    return 0 if world_size == 1 else role % world_size


def check_allreduce_exact(primes, world_size):
    """The wrapping int64 sum is exact iff world_size*(q-1) < 2^64 for all q."""
    return all(world_size * (int(q) - 1) < (1 << 64) for q in primes)


def modular_sum_host(residue_arrays, primes):
    """Host statement of the all-reduce contract (used by the CPU tests):
    wrapping uint64 sum over ranks, then mod q per limb."""
    acc = np.zeros_like(residue_arrays[0], dtype=np.uint64)
    for a in residue_arrays:
        acc = acc + np.asarray(a, dtype=np.uint64)  # wraps mod 2^64
    q = np.asarray(primes, dtype=np.uint64).reshape((-1,) + (1,) * (acc.ndim - 1))
    return acc % q


def allreduce_ciphertext(ct, group=None):
    """In-place modular all-reduce of an (unbatched) ciphertext over `group`."""
    import torch.distributed as dist

    rank, ws = world(group)
    if ws == 1:
        return ct
    params = ct.params
    k = ct.level + 1
    if not check_allreduce_exact(params.ring.moduli_chain[:k], ws):
        raise ValueError("world size too large for an exact wrapping all-reduce")
    from .ckks import ops

    grp = ops._pair_group(ct)
    if grp is None:
        ct = ct.copy()
        grp = ops._pair_group(ct)
    base = ct.c0.data
    n = params.ring_degree
    flat = base.as_strided((2, k, n), (k * n, n, 1))
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    p, cnt, s = grp
    _lib.call(
        "hegpu_elementwise", params.ring.device(), _lib.OP_REDUCE, p, s, None, 0, p, s, cnt, k,
        _dev.chain_primes(k).ctypes.data, None, _dev.stream(),
    )
    return ct


def broadcast_ciphertext(ct, src, template, group=None):
    """Broadcast a ciphertext from (group-local) rank `src`; other ranks pass a
    same-shaped template."""
    import torch.distributed as dist

    rank, ws = world(group)
    if ws == 1:
        return ct
    from .ckks import ops

    holder = ct if rank == src else template.copy()
    grp = ops._pair_group(holder)
    if grp is None:
        holder = holder.copy()
    k = holder.level + 1
    n = holder.params.ring_degree
    flat = holder.c0.data.as_strided((2, k, n), (k * n, n, 1))
    gsrc = global_rank(group, src)
    dist.broadcast(flat, src=gsrc, group=group)
    meta = [holder.scale, int(holder.insecure_provenance)]
    obj = [meta]
    dist.broadcast_object_list(obj, src=gsrc, group=group)
    holder.scale = float(obj[0][0])
    holder.insecure_provenance = bool(obj[0][1])
    return holder


def allreduce_residues(t, primes_idx, params, group=None):
    """In-place modular all-reduce of a residue tensor (..., k, N) whose row i
    lives modulo prime index primes_idx[i] (chain and special rows mixed):
    wrapping int64 SUM, then one mod-q pass.  Exact for world*(q-1) < 2^64."""
    import torch.distributed as dist

    ws = dist.get_world_size(group) if group is not None else world()[1]
    if ws == 1:
        return t
    primes_idx = np.ascontiguousarray(primes_idx, dtype=np.int32)
    all_primes = list(params.ring.moduli_chain) + list(params.ring.special_moduli)
    if not check_allreduce_exact([all_primes[i] for i in primes_idx], ws):
        raise ValueError("world size too large for an exact wrapping all-reduce")
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    k, n = int(t.shape[-2]), int(t.shape[-1])
    p, cnt, s = _dev.group(t, k, n)
    _lib.call(
        "hegpu_elementwise", params.ring.device(), _lib.OP_REDUCE, p, s, None, 0, p, s, cnt, k,
        primes_idx.ctypes.data, None, _dev.stream(),
    )
    return t


def reduce_scatter_residues(t, out, primes_idx, params, group=None):
    """Modular reduce-scatter along dim 0: `out` (t.shape[0] // world rows of
    t's layout) receives this rank's contiguous block of the sum over ranks,
    reduced mod q.  NCCL reduce_scatter_tensor when available (half the
    traffic of an all-reduce), else an all-reduce and a copy of the block."""
    import torch.distributed as dist

    rank, ws = world(group)
    if ws == 1:
        out.copy_(t)
        return out
    n = int(t.shape[0])
    if dist.get_backend(group) == "nccl" and n % ws == 0:
        primes_idx = np.ascontiguousarray(primes_idx, dtype=np.int32)
        all_primes = list(params.ring.moduli_chain) + list(params.ring.special_moduli)
        if not check_allreduce_exact([all_primes[i] for i in primes_idx], ws):
            raise ValueError("world size too large for an exact wrapping reduction")
        dist.reduce_scatter_tensor(out, t, op=dist.ReduceOp.SUM, group=group)
        k, nn = int(out.shape[-2]), int(out.shape[-1])
        p, cnt, s = _dev.group(out, k, nn)
        _lib.call(
            "hegpu_elementwise", params.ring.device(), _lib.OP_REDUCE, p, s, None, 0, p, s, cnt,
            k, primes_idx.ctypes.data, None, _dev.stream(),
        )
        return out
    allreduce_residues(t, primes_idx, params, group)
    lo, hi = shard_range(n, rank, ws)
    out.copy_(t[lo:hi])
    return out
