"""cfg4 end to end through the PUBLIC API: one full encrypted-LR training epoch
on SST-2-sized synthetic 768-d embeddings at P16 (N = 2^16), as
test_acceptance.py:98-131 runs it at desk scale:

  pack_batch (level-3 transport ciphertexts) -> logreg.train(...) with the
  batched full-slot ingest bootstrap (data_refresher) and the sparse-1024
  bootstrap refresh of w / u -> decrypted_weights -> held-out accuracy,
  next to the float64 shadow trainer (logreg.py:495-576).

Reports epoch samples/s (reference semantics: ingest excluded,
logreg.py:337-339), ingest ciphertexts/s, the weight gap to the shadow and
the held-out accuracies.  Usage (GPU box):

    PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True python tools/epoch_run.py [n_rows] [n_test]

(default 67349 2000; expandable segments keep the ingest outputs from pinning
large cached blocks, so the memory libhegpu's stream-ordered scratch needs is
not stranded in torch's cache)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2210_02574_b200 import bootstrap as bs, ckks, logreg, minimax  # noqa: E402
from paper_2210_02574_b200.synth import make_separable  # noqa: E402


def main():
    n_rows = int(sys.argv[1]) if len(sys.argv) > 1 else 67349
    n_test = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    preset = os.environ.get("EPOCH_PRESET", "p16")  # "p16s": the 128-bit-secure preset
    params = ckks.get_preset(preset)
    sig = minimax.load_approximant("sigmoid_deg15")
    layout = logreg.make_layout(params, 768)
    ctx = bs.build_context(params, n_slots=layout.padded_dim, input_periodic=True,
                           evalmod=os.environ.get("SPARSE_EVALMOD", "double_angle"))
    ctx_full = bs.build_context(params, n_slots=params.slot_count)
    steps = sorted(set(bs.refresh_rotation_steps(ctx)) | set(logreg.rotation_steps(layout))
                   | set(ctx_full.required_rotation_steps()))
    t0 = time.time()
    keys = ckks.keygen(params, rotation_steps=steps, rng_seed=7)
    t_keygen = time.time() - t0
    X, y = make_separable(np.random.default_rng(100), n_rows + n_test, dim=768, margin=0.5)
    Xtr, ytr, Xte, yte = X[:n_rows], y[:n_rows], X[n_rows:], y[n_rows:]
    t0 = time.time()
    pairs = logreg.pack_batch(Xtr, ytr, layout, params, keys, rng_seed=1_000_000)
    torch.cuda.synchronize()
    t_pack = time.time() - t0
    # lr 0.02: the acceptance test's lr 1.0 (T/test_acceptance.py:107-110, 2 minibatches)
    # diverges over a 132-minibatch epoch -- the float64 shadow trainer itself leaves the
    # sigmoid's domain; 0.02 trains it to 100% held-out accuracy with no domain breach
    lr = float(os.environ.get("EPOCH_LR", "0.02"))
    cfg = logreg.TrainConfig(lr, 0.9, 512, 1)

    class TimedRefresher(bs.BootstrapRefresher):
        seconds = 0.0
        count = 0

        def refresh_many(self, cts):
            torch.cuda.synchronize()
            t = time.time()
            out = super().refresh_many(cts)
            torch.cuda.synchronize()
            TimedRefresher.seconds += time.time() - t
            TimedRefresher.count += len(cts)
            if TimedRefresher.count % 200 < len(cts):
                free, total = torch.cuda.mem_get_info()
                print(f"ingest {TimedRefresher.count} cts {TimedRefresher.seconds:.0f}s "
                      f"free {free / 2**30:.1f}/{total / 2**30:.0f} GiB", flush=True)
            return out

    t0 = time.time()
    model, timing = logreg.train(pairs, n_rows, cfg, params, keys, sig,
                                 bs.BootstrapRefresher(ctx, keys), layout=layout,
                                 data_refresher=TimedRefresher(ctx_full, keys))
    torch.cuda.synchronize()
    t_train = time.time() - t0
    got = logreg.decrypted_weights(model, keys)
    shadow = logreg.shadow_train(Xtr, ytr, cfg, sig, layout=layout)

    def acc(w):
        s = np.asarray(logreg.shadow_scores(Xte, w, sig, layout)).ravel()
        return float(np.mean((s > 0.5).astype(int) == yte))

    epoch_s = timing[0]["seconds"]
    rec = {
        "workload": f"cfg4 one epoch, public logreg.train(), {preset}, SST-2-sized synthetic 768-d",
        "rows": n_rows, "test_rows": n_test, "data_cts": len(pairs),
        "minibatches": -(-n_rows // cfg.batch_size),
        "epoch_seconds": round(epoch_s, 3),
        "epoch_samples_per_s": round(n_rows / epoch_s, 1),
        "ingest_cts": TimedRefresher.count, "ingest_seconds": round(TimedRefresher.seconds, 2),
        "ingest_cts_per_s": round(TimedRefresher.count / TimedRefresher.seconds, 3),
        "ingest_batch": logreg.INGEST_BATCH,
        "train_call_seconds": round(t_train, 2), "pack_seconds": round(t_pack, 2),
        "keygen_seconds": round(t_keygen, 2), "rotation_keys": len(steps),
        "w_gap_vs_shadow": float(np.max(np.abs(got - shadow.weights))),
        "shadow_domain_breaches": int(shadow.domain_breaches),
        "test_acc_encrypted": acc(got), "test_acc_shadow": acc(shadow.weights),
        "level_refreshes": timing[0]["level_refreshes"],
        "train_config": {"learning_rate": cfg.learning_rate, "momentum_gamma": cfg.momentum_gamma,
                         "batch_size": cfg.batch_size, "epochs": cfg.epochs},
    }
    rec["acc_delta"] = round(rec["test_acc_encrypted"] - rec["test_acc_shadow"], 6)
    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
