"""Device time of the phases of the training step's packed pair refresh
(ModRaise, CoeffToSlot, EvalMod, SlotToCoeff, masks) with CUDA events around
wrapped bootstrap functions (eager, not captured)."""
import os
import sys

os.environ["BENCH_GRAPH"] = "0"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2210_02574_b200 import bootstrap as bs  # noqa: E402
from paper_2210_02574_b200.ckks import ops  # noqa: E402

times = {}


def wrap(mod, name, label):
    fn = getattr(mod, name)

    def w(*a, **k):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        r = fn(*a, **k)
        e1.record()
        times.setdefault(label, []).append((e0, e1))
        return r

    setattr(mod, name, w)


wrap(bs, "_mod_raise", "mod_raise")
wrap(bs, "_apply_diag_transform", "diag_transform (CtS / StC)")
wrap(ops, "eval_poly_bsgs", "eval_poly (EvalMod)")
wrap(bs, "_bootstrap_core", "bootstrap_core (all)")
wl = bench.TrainWorkload()
wl.setup(0, 1)
w, u = ops.mod_down(wl.w, 1), ops.mod_down(wl.u, 1)
for it in range(3):
    times.clear()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    wl.refresher.refresh_many([w, u])
    e1.record()
    torch.cuda.synchronize()
    print(f"iter {it}: refresh {e0.elapsed_time(e1):.1f} ms")
    for k, v in times.items():
        print(f"   {k}: " + ", ".join(f"{a.elapsed_time(b):.2f}" for a, b in v))
