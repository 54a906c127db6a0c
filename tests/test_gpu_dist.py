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
        w0 = shard.broadcast_ciphertext(w0, 0, w0)  # identical state on every rank
        u0 = shard.broadcast_ciphertext(u0, 0, u0)
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
    graph, the eager modular all-reduce, then the segment-captured packed
    refresh with the transforms' giants split across the ranks (eager modular
    all-reduces between the segments): both ranks end with the same limbs,
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


def _split_boot_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2210_02574_b200 import bootstrap as bs, ckks

        params = ckks.get_preset("desk-boot")
        ctx = bs.build_context(params, n_slots=256, input_periodic=True)
        keys = ckks.keygen(params, rotation_steps=ctx.required_rotation_steps(), rng_seed=7)
        rng = np.random.default_rng(77)
        vs = [np.tile(rng.uniform(-1, 1, 256), params.slot_count // 256) for _ in range(2)]
        cts = [ckks.encrypt_vector(params, v, keys, level=0, rng_seed=300 + i)
               for i, v in enumerate(vs)]
        single = bs.bootstrap_many(cts, ctx, keys)  # this rank alone
        with bs.distributed():
            split = bs.bootstrap_many(cts, ctx, keys)
        same = all(np.array_equal(a.c0.limbs, b.c0.limbs) and np.array_equal(a.c1.limbs, b.c1.limbs)
                   for a, b in zip(single, split))
        err = max(float(np.max(np.abs(ckks.decrypt_vector(o, keys) - v))) for o, v in zip(split, vs))
        out[rank] = (same, err, split[0].c0.limbs.tobytes()[:4096])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_split_transform_bootstrap_bit_exact(world):
    """The bootstrap with CoeffToSlot / SlotToCoeff giant steps split across
    `world` gloo ranks (bootstrap.distributed: each rank its giants' diagonal
    products and key switches, one modular all-reduce of the extended-basis
    sums per transform) gives limbs identical to the single-process bootstrap
    on every rank."""
    ctx_mp = mp.get_context("spawn")
    out = ctx_mp.Manager().dict()
    mp.start_processes(_split_boot_worker, args=(world, _free_port(), out), nprocs=world,
                       join=True, start_method="spawn")
    for r in range(world):
        same, err, head = out[r]
        assert same, f"rank {r}: split bootstrap limbs differ from the single-process ones"
        assert err < 1e-2
        assert head == out[0][2]


def _eager_split_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2210_02574_b200 import bootstrap as bs, ckks, logreg

        from paper_2210_02574_b200 import shard

        params, keys, sig, layout, ctx, cfg, xs, ys, w0, u0, ops = _boot_setup()
        # the split refresh needs identical (w, u) limbs on every rank (train()
        # broadcasts its initial state the same way); zeros are encrypted unseeded
        w0 = shard.broadcast_ciphertext(w0, 0, w0)
        u0 = shard.broadcast_ciphertext(u0, 0, u0)
        w, u = logreg.train_minibatch(w0, u0, xs, ys, cfg.batch_size, cfg, keys, sig, layout,
                                      bs.BootstrapRefresher(ctx, keys))
        out[rank] = (w.c0.limbs.tobytes(), u.c1.limbs.tobytes(),
                     ckks.decrypt_vector(w, keys).tolist())
    finally:
        dist.destroy_process_group()


def test_two_rank_eager_minibatch_split_refresh():
    """train_minibatch over two gloo ranks with a bootstrap refresher: sharded
    gradients, modular all-reduce, then the packed (w, u) refresh run by both
    ranks with the transforms' giants split (no broadcast): identical limbs on
    both ranks, decrypting like the single-process update."""
    from paper_2210_02574_b200 import bootstrap as bs, ckks, logreg

    params, keys, sig, layout, ctx, cfg, xs, ys, w0, u0, ops = _boot_setup()
    w, _ = logreg.train_minibatch(w0, u0, ops.stack(xs), ops.stack(ys), cfg.batch_size, cfg,
                                  keys, sig, layout, bs.BootstrapRefresher(ctx, keys))
    want_w = ckks.decrypt_vector(w, keys)
    ctx_mp = mp.get_context("spawn")
    out = ctx_mp.Manager().dict()
    mp.start_processes(_eager_split_worker, args=(2, _free_port(), out), nprocs=2, join=True,
                       start_method="spawn")
    assert out[0][0] == out[1][0] and out[0][1] == out[1][1]
    assert np.max(np.abs(np.array(out[0][2]) - want_w)) < 5e-3


def _ovr_setup():
    from paper_2210_02574_b200 import bootstrap as bs, ckks, logreg, minimax
    from paper_2210_02574_b200.synth import make_blob_embeddings

    params = ckks.get_preset("desk")
    keys = ckks.keygen(params, rng_seed=7)
    sig = minimax.load_approximant("sigmoid_deg15")
    layout = logreg.make_layout(params, 16)
    X, y = make_blob_embeddings(np.random.default_rng(5), 64, 4, dim=16)
    X = X * 0.25
    pairs = logreg.pack_batch(X, y.astype(np.float64), layout, params, keys,
                              target_level=params.max_level, rng_seed=500)
    ovr = logreg.pack_labels_ovr(y, 4, layout, params, keys)
    cfg = logreg.TrainConfig(0.5, 0.9, 2 * layout.rows_per_ct, 1)
    return params, keys, sig, layout, X, y, pairs, ovr, cfg, bs.DebugRefresher(keys, enabled=True)


def _ovr_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2210_02574_b200 import logreg

        params, keys, sig, layout, X, y, pairs, ovr, cfg, ref = _ovr_setup()
        model, _ = logreg.train(pairs, len(y), cfg, params, keys, sig, ref, class_count=4,
                                ovr_labels=ovr, layout=layout, refreshed_data=[d for d, _ in pairs])
        out[rank] = logreg.decrypted_weights(model, keys).tolist()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [4, 8])
def test_ovr_class_by_minibatch_sharding(world):
    """One-vs-Rest over `world` gloo ranks on one GPU: 4 ranks = one class per
    rank; 8 ranks = the 2-D layout, each class's minibatches sharded over a
    2-rank subgroup (shard.class_groups).  Every rank returns the whole
    model, decrypting like the single-process training."""
    from paper_2210_02574_b200 import logreg

    params, keys, sig, layout, X, y, pairs, ovr, cfg, ref = _ovr_setup()
    model, _ = logreg.train(pairs, len(y), cfg, params, keys, sig, ref, class_count=4,
                            ovr_labels=ovr, layout=layout, refreshed_data=[d for d, _ in pairs])
    want = logreg.decrypted_weights(model, keys)
    ctx_mp = mp.get_context("spawn")
    out = ctx_mp.Manager().dict()
    mp.start_processes(_ovr_worker, args=(world, _free_port(), out), nprocs=world, join=True,
                       start_method="spawn")
    for r in range(world):
        assert np.max(np.abs(np.array(out[r]) - want)) < 1e-4
