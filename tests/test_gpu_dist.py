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
