"""Attribute hegpu_rescale calls of one bootstrap to their Python call sites."""
import collections
import os
import sys
import traceback

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2210_02574_b200 import bootstrap as bs, ckks  # noqa: E402
from paper_2210_02574_b200.ckks import ops  # noqa: E402

params = ckks.CkksParams.from_config_text(
    open(os.path.join(os.path.dirname(__file__), "..", "paper_2210_02574_b200", "presets",
                      "p16.preset")).read())
ctx = bs.build_context(params, n_slots=1024, input_periodic=True)
keys = ckks.keygen(params, rotation_steps=ctx.required_rotation_steps(), rng_seed=7)
v = np.tile(np.random.default_rng(1).uniform(-1, 1, 1024), 32)
ct = ckks.encrypt_vector(params, v, keys, level=0, rng_seed=5)
bs.bootstrap(ct, ctx, keys)  # warm
sites = collections.Counter()
orig = ops._rescale_polys


def spy(*a, **k):
    st = traceback.extract_stack()[-6:-1]
    sites[" <- ".join(f"{f.name}:{f.lineno}" for f in reversed(st))] += 1
    return orig(*a, **k)


ops._rescale_polys = spy
bs.bootstrap(ct, ctx, keys)
for s, n in sites.most_common(20):
    print(n, s)
print("total", sum(sites.values()))
