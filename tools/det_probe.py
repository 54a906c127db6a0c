"""Determinism check (single process): gradient phase and packed refresh
repeated on identical inputs must give identical limbs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import test_gpu_dist as T  # noqa: E402
from paper_2210_02574_b200 import bootstrap as bs, ckks, logreg  # noqa: E402

params, keys, sig, layout, ctx, cfg, xs, ys, w0, u0, ops = T._boot_setup()
ref = bs.BootstrapRefresher(ctx, keys)
res = []
for it in range(3):
    gu, G = logreg._gradient_phase(w0, u0, ops.stack(xs), ops.stack(ys), cfg.batch_size, cfg,
                                   keys, sig, layout)
    u1 = ops.add(gu, G) if gu is not None else G
    w1 = ops.sub(w0, u1)
    a = ref.refresh_many([w1, u1])
    res.append((w1.c0.limbs.copy(), u1.c0.limbs.copy(), a[0].c0.limbs.copy(), a[1].c0.limbs.copy()))
    print(it, "w1 dec", np.round(ckks.decrypt_vector(w1, keys)[:3], 6), "ref", np.round(ckks.decrypt_vector(a[0], keys)[:3], 6), flush=True)
for it in range(1, 3):
    print("iter", it, "same as 0:", [bool(np.array_equal(x, y)) for x, y in zip(res[0], res[it])])
# refresh of one fixed input repeated
a0 = ref.refresh_many([w1, u1])
a1 = ref.refresh_many([w1, u1])
print("refresh repeat equal:", np.array_equal(a0[0].c0.limbs, a1[0].c0.limbs))
c0 = bs.bootstrap(w1, ctx, keys)
c1 = bs.bootstrap(w1, ctx, keys)
print("bootstrap repeat equal:", np.array_equal(c0.c0.limbs, c1.c0.limbs))
import hashlib  # noqa: E402
print("digest", hashlib.sha256(b"".join(x.tobytes() for x in res[0])).hexdigest()[:16],
      hashlib.sha256(a0[0].c0.limbs.tobytes()).hexdigest()[:16], flush=True)
