"""Time ONE cfg4 training minibatch of the REFERENCE itself (numba, all host
cores) end to end, next to the oracle cost model on the same machine: the
calibration of bench.py's reference arm.

Run in the build container (needs /root/reference):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tools/ref_minibatch_time.py > profiles/r02_ref_minibatch_time.log

Workload = bench.py --config train: P16, 512 rows of 768-d separable data =
16 ciphertexts at the refresh level (the reference's epoch timing excludes
ingest, logreg.py:337-339), TrainConfig(1.0, 0.9, 512, 1), sparse-1024
periodic BootstrapRefresher for w and u (two bootstraps per minibatch).
"""
import json
import os
import platform
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from hebert import bootstrap as bs, ckks, logreg, minimax  # noqa: E402


class _Identity:
    """Data refresher for ciphertexts already at the training level."""

    output_level = None

    def refresh(self, ct):
        return ct


def main():
    with open(os.path.join(REPO, "paper_2210_02574_b200", "presets", "p16.preset")) as fh:
        params = ckks.CkksParams.from_config_text(fh.read())
    ctx = bs.build_context(params, n_slots=1024, input_periodic=True)
    steps = sorted(set(ctx.required_rotation_steps()) | set(ckks.default_rotation_steps(params)))
    t0 = time.time()
    keys = ckks.keygen(params, rotation_steps=steps, rng_seed=7)
    t_keygen = time.time() - t0
    sig = minimax.import_text(open(os.path.join(
        REPO, "paper_2210_02574_b200", "approximants", "sigmoid_deg15.txt")).read())
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "ref_conftest", "/root/reference/pkg/tests/conftest.py")
    rc = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(rc)
    X, y = rc.make_separable(np.random.default_rng(100), 512, dim=768, margin=0.5)
    layout = logreg.make_layout(params, 768)
    refresher = bs.BootstrapRefresher(ctx, keys)
    lvl = refresher.output_level
    pairs = []
    for i in range(0, 512, layout.rows_per_ct):
        xs = logreg._pack_slots(X[i:i + layout.rows_per_ct], layout)
        ys = logreg._pack_label_slots(y[i:i + layout.rows_per_ct].astype(np.float64), layout)
        pairs.append((ckks.encrypt_vector(params, xs, keys, level=lvl, rng_seed=100 + i),
                      ckks.encrypt_vector(params, ys, keys, level=lvl, rng_seed=200 + i)))
    cfg = logreg.TrainConfig(1.0, 0.9, 512, 1)
    t0 = time.time()
    model, timing = logreg.train(pairs, 512, cfg, params, keys, sig, refresher, layout=layout,
                                 data_refresher=_Identity())
    total = time.time() - t0
    rec = {"what": "reference hebert, one cfg4 minibatch (16 cts, 2 sparse-1024 refreshes), P16",
           "minibatch_seconds": timing[0]["seconds"], "train_call_seconds": total,
           "keygen_seconds": t_keygen, "rotation_keys": len(steps),
           "cpu": platform.processor() or open("/proc/cpuinfo").read().split("model name")[1]
           .split("\n")[0].strip(": "),
           "cores": os.cpu_count(), "numba_threads": os.environ.get("NUMBA_NUM_THREADS")}
    print(json.dumps(rec), flush=True)
    # the oracle cost model of the same workload on the same machine (what
    # bench.py's reference arm runs on the GPU box's host cores)
    from oracle import kernels as OK
    from oracle.costmodel import OracleCostModel, histogram_levels, load_histogram

    if OK.clib() is None:
        OK.build_c()
        OK._clib = None
    hist = load_histogram("train")
    t0 = time.time()
    cm = OracleCostModel(params.to_config_text())
    ks_levels, other = histogram_levels(hist)
    cm.sample(ks_levels, other)
    model_s = cm.seconds(hist)
    rec2 = {"what": "oracle cost model (C/OpenMP), same machine", "model_minibatch_seconds": model_s,
            "model_eval_seconds": time.time() - t0,
            "measured_over_model": rec["minibatch_seconds"] / model_s}
    print(json.dumps(rec2), flush=True)

if __name__ == "__main__":
    main()
