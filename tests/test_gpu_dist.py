"""The sharded trainer on ONE GPU with two gloo ranks (host-side
collectives only; no kernel waits on another rank): the minibatch is split
across ranks, gradients meet in the wrapping all-reduce + mod-q kernel, w and
u are refreshed on different ranks and broadcast.  The decrypted weights must
equal a single-process run of the same minibatch."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _setup():
    from paper_2210_02574_b200 import bootstrap as bs, ckks, logreg, minimax

    params = ckks.get_preset("desk")
    keys = ckks.keygen(params, rng_seed=7)
    sig = minimax.load_approximant("sigmoid_deg15")
    layout = logreg.make_layout(params, 16)
    rng = np.random.default_rng(0)
    X = rng.uniform(-1, 1, (512, 16))
    y = (X @ rng.normal(size=16) > 0).astype(np.float64)
    pairs = logreg.pack_batch(X, y, layout, params, keys, target_level=params.max_level,
                              rng_seed=100)
    cfg = logreg.TrainConfig(1.0, 0.9, 512, 1)
    ref = bs.DebugRefresher(keys, enabled=True)
    w0 = logreg._zeros_ct(params, keys, params.max_level)
    u0 = logreg._zeros_ct(params, keys, params.max_level)
    return params, keys, sig, layout, pairs, cfg, ref, w0, u0


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2210_02574_b200 import ckks, logreg

        params, keys, sig, layout, pairs, cfg, ref, w0, u0 = _setup()
        xs = [d for d, _ in pairs]
        ys = [l for _, l in pairs]
        w, u = logreg.train_minibatch(w0, u0, xs, ys, 512, cfg, keys, sig, layout, ref)
        out[rank] = (ckks.decrypt_vector(w, keys)[:32].tolist(),
                     ckks.decrypt_vector(u, keys)[:32].tolist())
    finally:
        dist.destroy_process_group()


def test_two_rank_minibatch_matches_single_process():
    from paper_2210_02574_b200 import ckks, logreg

    params, keys, sig, layout, pairs, cfg, ref, w0, u0 = _setup()
    w, u = logreg.train_minibatch(w0, u0, [d for d, _ in pairs], [l for _, l in pairs], 512,
                                  cfg, keys, sig, layout, ref)
    want_w = ckks.decrypt_vector(w, keys)[:32]
    want_u = ckks.decrypt_vector(u, keys)[:32]
    ctx = mp.get_context("spawn")
    manager = ctx.Manager()
    out = manager.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
    for r in range(2):
        got_w, got_u = map(np.array, out[r])
        assert np.max(np.abs(got_w - want_w)) < 1e-5
        assert np.max(np.abs(got_u - want_u)) < 1e-5


def _boot_setup():
    from paper_2210_02574_b200 import bootstrap as bs, ckks, logreg, minimax
    from paper_2210_02574_b200.ckks import ops

    params = ckks.get_preset("desk-boot")
    layout = logreg.make_layout(params, 16)
    ctx = bs.build_context(params, n_slots=layout.padded_dim, input_periodic=True)
    steps = sorted(set(bs.refresh_rotation_steps(ctx)) | logreg.rotation_steps(layout))
    keys = ckks.keygen(params, rotation_steps=steps, rng_seed=7)
    sig = minimax.load_approximant("sigmoid_deg15")
    cfg = logreg.TrainConfig(1.0, 0.9, 4 * layout.rows_per_ct, 1)
    rng = np.random.default_rng(12)
    X = rng.uniform(-1, 1, (cfg.batch_size, 16))
    y = (X @ rng.normal(size=16) > 0).astype(np.float64)
    top = bs.BootstrapRefresher(ctx, keys).output_level
    xs, ys = [], []
    for c in range(4):
        r0 = c * layout.rows_per_ct
        xr, yr = X[r0: r0 + layout.rows_per_ct], y[r0: r0 + layout.rows_per_ct]
        xs.append(ckks.encrypt(ckks.encode(params, logreg._pack_slots(xr, layout), top), keys,
                               rng_seed=100 + c))
        ys.append(ckks.encrypt(ckks.encode(params, logreg._pack_label_slots(yr, layout), 3), keys,
                               rng_seed=200 + c))
    w0, u0 = logreg._zeros_ct(params, keys, top), logreg._zeros_ct(params, keys, top)
    return params, keys, sig, layout, ctx, cfg, xs, ys, w0, u0, ops


def _captured_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2210_02574_b200 import bootstrap as bs, ckks, logreg, shard

        params, keys, sig, layout, ctx, cfg, xs, ys, w0, u0, ops = _boot_setup()
        lo, hi = shard.shard_range(len(xs), rank, world)
        xb, yb = ops.stack(xs[lo:hi]), ops.stack(ys[lo:hi])
        ref = bs.BootstrapRefresher(ctx, keys)
        cs = logreg.CapturedShardedMinibatch(w0, u0, xb, yb, cfg.batch_size, cfg, keys, sig,
                                             layout, ref)
        cs.load(xb, yb)
        w, u = cs.step()
        out[rank] = (w.c0.limbs.tobytes(), ckks.decrypt_vector(w, keys).tolist(),
                     ckks.decrypt_vector(u, keys).tolist())
    finally:
        dist.destroy_process_group()


def test_two_rank_captured_sharded_minibatch():
    """CapturedShardedMinibatch over two (gloo) ranks: each rank's gradient
    graph, the eager modular all-reduce, w refreshed by rank 0's and u by rank
    1's captured bootstrap, broadcast: both ranks end with the same limbs,
    decrypting like the single-process eager update (up to bootstrap error)."""
    from paper_2210_02574_b200 import bootstrap as bs, ckks, logreg

    params, keys, sig, layout, ctx, cfg, xs, ys, w0, u0, ops = _boot_setup()
    ref = bs.BootstrapRefresher(ctx, keys)
    w, u = logreg.train_minibatch(w0, u0, ops.stack(xs), ops.stack(ys), cfg.batch_size, cfg,
                                  keys, sig, layout, ref)
    want_w, want_u = ckks.decrypt_vector(w, keys), ckks.decrypt_vector(u, keys)
    ctx_mp = mp.get_context("spawn")
    out = ctx_mp.Manager().dict()
    mp.start_processes(_captured_worker, args=(2, _free_port(), out), nprocs=2, join=True,
                       start_method="spawn")
    assert out[0][0] == out[1][0]  # broadcast: identical state on every rank
    for r in range(2):
        assert np.max(np.abs(np.array(out[r][1]) - want_w)) < 5e-3
        assert np.max(np.abs(np.array(out[r][2]) - want_u)) < 5e-3
