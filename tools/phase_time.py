"""Split one cfg4 training minibatch into its phases (gradient, sum, update,
bootstrap refresh) with CUDA-event timing and per-class kernel profiles."""
import os
import sys

os.environ["BENCH_GRAPH"] = "0"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2210_02574_b200 import _lib, logreg  # noqa: E402
from paper_2210_02574_b200.ckks import ops  # noqa: E402

wl = bench.TrainWorkload()
wl.setup(0, 1)
xb, yb = wl.pool_dev[0]
cfg, keys, sig, layout = wl.cfg, wl.keys, wl.sig, wl.layout


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


for it in range(3):
    w, u = wl.w, wl.u
    t0 = ev()
    gu = ops.mult_plain(u, cfg.momentum_gamma)
    wl_ = ops.sub(w, gu)
    t1 = ev()
    g = logreg._batched_gradient(xb, yb, wl_, layout, keys, sig, cfg.learning_rate, wl.batch_rows)
    t2 = ev()
    G = logreg._sum_gradient(g, layout, keys)
    t3 = ev()
    u2 = ops.add(gu, G)
    w2 = ops.sub(w, u2)
    t4 = ev()
    w3, u3 = wl.refresher.refresh_many([w2, u2])
    t5 = ev()
    torch.cuda.synchronize()
    print(f"iter {it}: lookahead {t0.elapsed_time(t1):.1f} gradient {t1.elapsed_time(t2):.1f} "
          f"sum+rotsum {t2.elapsed_time(t3):.1f} update {t3.elapsed_time(t4):.1f} "
          f"refresh {t4.elapsed_time(t5):.1f} ms")
for name, fn in (("gradient", lambda: logreg._batched_gradient(xb, yb, wl.w, layout, keys, sig,
                                                                cfg.learning_rate, wl.batch_rows)),
                 ("refresh", lambda: wl.refresher.refresh_many([w2, u2]))):
    _lib.profile_enable(True)
    fn()
    prof = _lib.profile_read()
    _lib.profile_enable(False)
    print(name, {c: round(p["ms"], 1) for c, p in prof.items() if p["launches"]},
          {c: p["launches"] for c, p in prof.items() if p["launches"]})

# captured (graph-replayed) device time of the two phases, as in the bench
from paper_2210_02574_b200 import bootstrap as bs  # noqa: E402


def captured_ms(fn, reps=5):
    seg = bs.SegmentedCapture()
    fn()  # warm caches
    seg.capture(fn)
    seg.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        seg.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


grad_ms = captured_ms(lambda: logreg._gradient_phase(wl.w, wl.u, xb, yb, wl.batch_rows, cfg, keys,
                                                     sig, layout))
ref_ms = captured_ms(lambda: wl.refresher.refresh_many([w2, u2]))
print(f"captured: gradient phase (lookahead + 16 gradients + sum) {grad_ms:.2f} ms, "
      f"packed refresh {ref_ms:.2f} ms")

# per-rank device time at G ranks, simulated on this GPU: the rank's shard of
# the gradient (16/G ciphertexts) and the split refresh with rank 0's share of
# the giant steps (the modular all-reduces are skipped: the numbers are
# garbage, the timing is the rank's compute).  Collective cost is added in
# DESIGN.md from the message sizes.
from paper_2210_02574_b200 import shard  # noqa: E402

_real_ar = shard.allreduce_residues
_real_rs = shard.reduce_scatter_residues
for G in (2, 4, 8):
    shard.allreduce_residues = lambda *a, **k: None
    shard.reduce_scatter_residues = lambda t, out, *a, **k: out.copy_(t[: out.shape[0]])
    xs, ys = ops.unstack(xb), ops.unstack(yb)
    lo, hi = shard.shard_range(len(xs), 0, G)
    xg, yg = ops.stack(xs[lo:hi]), ops.stack(ys[lo:hi])
    g_ms = captured_ms(lambda: logreg._gradient_phase(wl.w, wl.u, xg, yg, wl.batch_rows, cfg,
                                                      keys, sig, layout))
    shares = {}
    for babies in (False, True):
        bs._DIST = (0, G, None)
        bs.SPLIT_BABIES = babies
        try:
            shares[babies] = captured_ms(lambda: wl.refresher.refresh_many([w2, u2]))
        finally:
            bs._DIST = None
    shard.allreduce_residues = _real_ar
    shard.reduce_scatter_residues = _real_rs
    print(f"G={G}: rank-0 gradient shard ({hi - lo} cts) {g_ms:.2f} ms, split refresh share: "
          f"giants only {shares[False]:.2f} ms, giants + babies {shares[True]:.2f} ms",
          flush=True)
