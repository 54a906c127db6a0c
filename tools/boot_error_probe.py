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
SPECS = sys.argv[2].split(",") if len(sys.argv) > 2 else ["119", "da"]
import torch  # noqa: E402

params = ckks.get_preset(os.environ.get("PROBE_PRESET", "p16"))
slots = params.slot_count
n = slots if MODE == "full" else 1024


def make_ctx(spec):
    kw = dict(n_slots=n, input_periodic=(MODE != "full"))
    if spec.startswith("da"):  # "daR" or "daR:D" (R squarings, degree-D cos base)
        r_s, _, d_s = spec[2:].partition(":")
        return bs.build_context(params, evalmod="double_angle", double_angle=int(r_s or 3),
                                evalmod_degree=int(d_s) if d_s else None, **kw)
    return bs.build_context(params, evalmod="sine", evalmod_degree=int(spec), **kw)


ctxs = {sp: make_ctx(sp) for sp in SPECS}
steps = set()
for c in ctxs.values():
    steps |= set(c.required_rotation_steps()) | set(bs.refresh_rotation_steps(c))
steps = sorted(steps)
t0 = time.time()
keys = ckks.keygen(params, rotation_steps=steps, rng_seed=7)
print(f"keygen {len(steps)} steps {time.time() - t0:.1f}s", flush=True)
rng = np.random.default_rng(1002)
vs = []
for i in range(2):
    vs.append(rng.uniform(-1, 1, slots) if MODE == "full" else np.tile(rng.uniform(-1, 1, n), slots // n))
cts = [ckks.encrypt_vector(params, v, keys, level=0, rng_seed=5 + i) for i, v in enumerate(vs)]
_real_evalmod = bs._evalmod


def _spy_evalmod(w, ctx, keyset):
    out = _real_evalmod(w, ctx, keyset)
    parts_in = ops.unstack(w) if w.batch is not None else [w]
    parts_out = ops.unstack(out) if out.batch is not None else [out]
    D = ctx.range_k + 0.5
    q0 = params.ring.moduli_chain[0]
    for a, o in zip(parts_in[:1], parts_out[:1]):
        y = ckks.decrypt_vector(a, keys)
        z = ckks.decrypt_vector(o, keys)
        f = np.sin(2 * np.pi * D * y) / (2 * np.pi)
        frac = D * y - np.round(D * y)
        print(f"   evalmod in: level {a.level} scale {a.scale:.4g} |y|max {np.max(np.abs(y)):.4f} "
              f"|I|max {np.max(np.abs(np.round(D * y))):.0f} frac max {np.max(np.abs(frac)):.3e}; "
              f"out level {o.level} scale {o.scale:.4g} |out - f| max {np.max(np.abs(z - f)):.3e}"
              f" (x q0/scale {np.max(np.abs(z - f)) * q0 / params.default_scale:.3e})", flush=True)
    return out


bs._evalmod = _spy_evalmod
for sp, ctx in ctxs.items():
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        outs = bs.bootstrap_many(cts, ctx, keys) if MODE != "full" else [bs.bootstrap(cts[0], ctx, keys)]
        e1.record()
        torch.cuda.synchronize()
        errs = [float(np.max(np.abs(ckks.decrypt_vector(o, keys) - v))) for o, v in zip(outs, vs)]
        print(f"{MODE} {sp}: err {max(errs):.3e} level {outs[0].level} time {e0.elapsed_time(e1):.1f} ms"
              f" (B={len(outs)})", flush=True)
    if MODE != "full":
        refr = bs.BootstrapRefresher(ctx, keys)
        for rep in range(2):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            outs = refr.refresh_many(cts)
            e1.record()
            torch.cuda.synchronize()
            errs = [float(np.max(np.abs(ckks.decrypt_vector(o, keys) - v))) for o, v in zip(outs, vs)]
            print(f"{MODE} {sp} packed pair: err {max(errs):.3e} time {e0.elapsed_time(e1):.1f} ms",
                  flush=True)
