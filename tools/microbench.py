"""Kernel microbenchmarks through the C ABI (device-resident inputs, CUDA
events on the launching stream).  Not part of the product or the tests; used
to iterate on single kernels:  python tools/microbench.py [ntt] [bsgs] [ip]."""

import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_02574_b200 import _dev, _lib, ckks  # noqa: E402


def timeit(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(iters):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3  # us


def rand_limbs(params, shape, k):
    qs = torch.tensor([int(q) for q in params.ring.moduli_chain[:k]], dtype=torch.int64,
                      device="cuda")
    x = torch.randint(0, 2 ** 62, shape, dtype=torch.int64, device="cuda")
    return torch.remainder(x, qs.view(*([1] * (len(shape) - 2)), k, 1))


def bench_ntt(params):
    n = params.ring_degree
    ring = params.ring.device()
    k = params.max_level + 1
    for polys in (1, 2, 10):
        x = rand_limbs(params, (polys, k, n), k)
        sel = np.arange(k, dtype=np.int32)
        for inv in (0, 1):
            f = lambda: _lib.call("hegpu_ntt", ring, inv, x.data_ptr(), k * n, x.data_ptr(),
                                  k * n, polys, k, sel.ctypes.data, _dev.stream())
            us = timeit(f)
            r = polys * k
            bfly = r * n // 2 * int(np.log2(n))
            print(f"ntt inv={inv} rows={r:4d}: {us:8.1f} us  {us / r:6.2f} us/row  "
                  f"{bfly / us / 1e6:6.3f} T bfly/s")


def bench_bsgs(params):
    n = params.ring_degree
    ring = params.ring.device()
    k = 22 if params.max_level >= 21 else params.max_level + 1
    n_terms, n_giants = 64, 32
    for nb in (1, 2):
        babies = rand_limbs(params, (n_terms, nb * 2, k, n), k)
        ptrs = (ctypes.c_void_p * n_terms)(*[babies[t].data_ptr() for t in range(n_terms)])
        idx = torch.arange(n_giants * n_terms, dtype=torch.int32, device="cuda") % 2048
        out = torch.empty((n_giants, nb, 2, k, n), dtype=torch.int64, device="cuda")
        for lr in (0, 3, 4):
            pts = rand_limbs(params, (2048, k, n >> lr), k)
            f = lambda: _lib.call("hegpu_bsgs", ring, ptrs, n_terms, k * n, 2 * k * n, nb,
                                  pts.data_ptr(), k * (n >> lr), lr, idx.data_ptr(), n_giants,
                                  out.data_ptr(), nb * 2 * k * n, k, 0, _dev.stream())
            us = timeit(f, iters=5, warm=1)
            macs = n_giants * n_terms * nb * 2 * k * n
            print(f"bsgs nb={nb} lr={lr} k={k}: {us:9.1f} us  {macs / us / 1e6:6.3f} T mac/s")
            del pts


def bench_ip(params):
    """Key-switch inner products (ks_ip class) of a relinearising mult and a
    15-rotation hoisted rotate-and-sum, batched, at two levels."""
    from paper_2210_02574_b200.ckks import ops

    steps = list(range(1, 16))
    keys = ckks.keygen(params, rotation_steps=steps, rng_seed=7)
    rng = np.random.default_rng(3)
    only = os.environ.get("IP_ONLY")  # e.g. "rotsum15:21:16"
    for lvl in (21, 11):
        for B in (1, 4, 16):
            if only and not any(o.endswith(f":{lvl}:{B}") for o in only.split(",")):
                continue
            cts = [ckks.encrypt_vector(params, rng.uniform(-1, 1, params.slot_count), keys,
                                       level=lvl, rng_seed=i) for i in range(B)]
            ct = cts[0] if B == 1 else ops.stack(cts)
            for name, fn in (("mult", lambda: ops.mult(ct, ct, keys, rescale_after=False)),
                             ("rotsum15", lambda: ops.rotate_sum(ct, steps, keys))):
                if only and f"{name}:{lvl}:{B}" not in only.split(","):
                    continue
                fn()
                torch.cuda.synchronize()
                _lib.profile_enable(True)
                for _ in range(5):
                    fn()
                prof = _lib.profile_read()
                _lib.profile_enable(False)
                p = prof["ks_ip"]
                print(f"ip {name:8s} level {lvl:2d} B={B:2d}: ks_ip {p['ms'] / 5 * 1e3:8.1f} us/op "
                      f"{p['bytes'] / p['ms'] / 1e6:7.1f} GB/s alg  launches {p['launches'] // 5}",
                      flush=True)


def main():
    params = ckks.get_preset("p16")
    which = sys.argv[1:] or ["ntt", "bsgs"]
    if "ntt" in which:
        bench_ntt(params)
    if "bsgs" in which:
        bench_bsgs(params)
    if "ip" in which:
        bench_ip(params)


if __name__ == "__main__":
    main()
