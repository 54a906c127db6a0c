"""Error budget of the P16 bootstrap (full-slot and sparse): runs the real
bootstrap, then variants with one stage replaced by its exact (decrypt ->
float64 math -> re-encrypt) counterpart, and variants of the EvalMod
polynomial.  Prints max |dec(out) - v| for each.  Diagnostic only."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2210_02574_b200 import bootstrap as bs, ckks, minimax  # noqa: E402
from paper_2210_02574_b200.ckks import ops  # noqa: E402

MODE = sys.argv[1] if len(sys.argv) > 1 else "full"
DEGS = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["119", "127"])]

params = ckks.get_preset("p16")
slots = params.slot_count
n = slots if MODE == "full" else 1024
ctxs = {d: bs.build_context(params, n_slots=n, evalmod_degree=d, input_periodic=(MODE != "full"))
        for d in DEGS}
ctx0 = ctxs[DEGS[0]]
steps = sorted(set(ctx0.required_rotation_steps()) | set(bs.refresh_rotation_steps(ctx0)))
t0 = time.time()
keys = ckks.keygen(params, rotation_steps=steps, rng_seed=7)
print(f"keygen {len(steps)} steps {time.time() - t0:.1f}s", flush=True)

rng = np.random.default_rng(1002)
if MODE == "full":
    v = rng.uniform(-1, 1, slots)
else:
    v = np.tile(rng.uniform(-1, 1, n), slots // n)
ct = ckks.encrypt_vector(params, v, keys, level=0, rng_seed=5)


def err(out):
    return float(np.max(np.abs(ckks.decrypt_vector(out, keys) - v)))


real_eval = ops.eval_poly_bsgs


def exact_eval(ct_in, poly, keyset, input_prescaled=False):
    out = real_eval(ct_in, poly, keyset, input_prescaled=input_prescaled)
    D = poly.domain[1]
    parts_in = ops.unstack(ct_in) if ct_in.batch is not None else [ct_in]
    parts_out = ops.unstack(out) if out.batch is not None else [out]
    res = []
    for a, o in zip(parts_in, parts_out):
        y = ckks.decrypt_vector(a, keys)
        f = np.sin(2 * np.pi * D * y) / (2 * np.pi)
        res.append(ckks.encrypt_vector(params, f, keys, level=o.level, scale=o.scale, rng_seed=9))
    return ops.stack(res) if out.batch is not None else res[0]


for d in DEGS:
    ctx = ctxs[d]
    for rep in range(2):
        out = bs.bootstrap(ct, ctx, keys)
        print(f"deg {d} rep {rep}: err {err(out):.3e} level {out.level}", flush=True)
    ops.eval_poly_bsgs = exact_eval
    bs.ops.eval_poly_bsgs = exact_eval
    try:
        out = bs.bootstrap(ct, ctx, keys)
        print(f"deg {d} EXACT EvalMod: err {err(out):.3e}", flush=True)
    finally:
        ops.eval_poly_bsgs = real_eval
        bs.ops.eval_poly_bsgs = real_eval
    # EvalMod-only error: decrypt in / out of the real EvalMod
    cap = {}

    def cap_eval(ct_in, poly, keyset, input_prescaled=False):
        out = real_eval(ct_in, poly, keyset, input_prescaled=input_prescaled)
        cap["in"], cap["out"], cap["D"] = ct_in, out, poly.domain[1]
        return out

    ops.eval_poly_bsgs = cap_eval
    bs.ops.eval_poly_bsgs = cap_eval
    try:
        bs.bootstrap(ct, ctx, keys)
    finally:
        ops.eval_poly_bsgs = real_eval
        bs.ops.eval_poly_bsgs = real_eval
    ins = ops.unstack(cap["in"]) if cap["in"].batch is not None else [cap["in"]]
    outs = ops.unstack(cap["out"]) if cap["out"].batch is not None else [cap["out"]]
    D = cap["D"]
    q0 = params.ring.moduli_chain[0]
    for a, o in zip(ins, outs):
        y = ckks.decrypt_vector(a, keys)
        z = ckks.decrypt_vector(o, keys)
        f = np.sin(2 * np.pi * D * y) / (2 * np.pi)
        frac = D * y - np.round(D * y)
        print(f"   evalmod in: |y|max {np.max(np.abs(y)):.4f} |I|max {np.max(np.abs(np.round(D*y))):.0f}"
              f" frac rms {np.sqrt(np.mean(frac**2)):.3e} max {np.max(np.abs(frac)):.3e};"
              f" out-f max {np.max(np.abs(z - f)):.3e} rms {np.sqrt(np.mean((z - f)**2)):.3e}"
              f" (x q0/scale = msg units {np.max(np.abs(z - f)) * q0 / params.default_scale:.3e})",
              flush=True)
