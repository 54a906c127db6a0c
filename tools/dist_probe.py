"""Debug: packed-pair refresh with split giants (gloo, world 2, one GPU)."""
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def worker(rank, world, port):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2210_02574_b200 import bootstrap as bs, ckks, logreg

    params = ckks.get_preset("desk-boot")
    layout = logreg.make_layout(params, 16)
    ctx = bs.build_context(params, n_slots=layout.padded_dim, input_periodic=True)
    keys = ckks.keygen(params, rotation_steps=sorted(bs.refresh_rotation_steps(ctx)), rng_seed=7)
    rng = np.random.default_rng(3)
    n = layout.padded_dim
    vs = [np.tile(rng.uniform(-1, 1, n), params.slot_count // n) for _ in range(2)]
    cts = [ckks.encrypt_vector(params, v, keys, level=2, rng_seed=9 + i) for i, v in enumerate(vs)]
    ref = bs.BootstrapRefresher(ctx, keys)
    a = ref.refresh_many(cts)
    with bs.distributed():
        b = ref.refresh_many(cts)
        c = bs.bootstrap_many(cts, ctx, keys)
    d = bs.bootstrap_many(cts, ctx, keys)
    for name, o in (("packed", a), ("packed-split", b), ("many-split", c), ("many", d)):
        e = max(float(np.max(np.abs(ckks.decrypt_vector(x, keys) - v))) for x, v in zip(o, vs))
        print(rank, name, "err %.3e" % e, "levels", [x.level for x in o], flush=True)
    print(rank, "packed limbs equal:", all(np.array_equal(x.c0.limbs, y.c0.limbs) for x, y in zip(a, b)))
    # the eager sharded minibatch, split refresh vs owner refresh
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "tests"))
    import test_gpu_dist as T

    params, keys, sig, layout, ctx, cfg, xs, ys, w0, u0, ops = T._boot_setup()
    ref = bs.BootstrapRefresher(ctx, keys)
    # the same pre-refresh (w, u) both ways
    g = logreg._gradient_phase(w0, u0, ops.stack(xs), ops.stack(ys), cfg.batch_size, cfg, keys,
                               sig, layout)
    gu, G = g
    u1 = ops.add(gu, G) if gu is not None else G
    w1 = ops.sub(w0, u1)
    print(rank, "pre levels", w1.level, u1.level, w1.scale, u1.scale, flush=True)
    a = ref.refresh_many([w1, u1])
    with bs.distributed():
        b = ref.refresh_many([w1, u1])
    print(rank, "pre-refresh pair equal:", [np.array_equal(x.c0.limbs, y.c0.limbs) for x, y in zip(a, b)],
          np.round(ckks.decrypt_vector(a[0], keys)[:4], 5), np.round(ckks.decrypt_vector(b[0], keys)[:4], 5),
          flush=True)
    for split in (False, True):
        logreg.DISTRIBUTED_REFRESH = split
        w, u = logreg.train_minibatch(w0, u0, xs, ys, cfg.batch_size, cfg, keys, sig, layout, ref)
        dw = ckks.decrypt_vector(w, keys)[:8]
        print(rank, "split" if split else "owner", "w", np.round(dw, 5), w.level, w.scale, flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.start_processes(worker, args=(2, port), nprocs=2, join=True, start_method="spawn")
