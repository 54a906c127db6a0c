"""GPU parity at the BASELINE ring size, N = 2^16 (P16 preset): sparse and
full-slot bootstrapping and multi-minibatch encrypted training, against
fixtures produced by running the REFERENCE at P16 (tests/golden/make_golden.py
boot_p16_sparse / logreg_p16) and against the shadow trainer
(logreg.py:495-576).  Tolerances: bootstrap max |dec - v| <= 1e-3 (north
star) and no worse than the reference's own error on the same ciphertext;
weights within 2e-2 of the reference run and of the shadow trainer
(T/test_logreg.py:122); held-out accuracy equal to the shadow's within 0.2 %
(one of 512 rows)."""

import numpy as np
import pytest

from conftest import golden_npz

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

from oracle.scheme import sha  # noqa: E402
from paper_2210_02574_b200 import bootstrap as bs, ckks, logreg  # noqa: E402


def ct_digest(ct):
    return {"c0": sha(ct.c0.limbs), "c1": sha(ct.c1.limbs), "level": ct.level,
            "scale": float(ct.scale).hex()}


@pytest.fixture(scope="module")
def p16():
    return ckks.get_preset("p16")


@pytest.fixture(scope="module")
def sparse(p16, digests):
    d = digests["boot_p16_sparse"]
    ctx = bs.build_context(p16, n_slots=1024, input_periodic=True)
    assert ctx.required_rotation_steps() == d["steps"]
    keys = ckks.keygen(p16, rotation_steps=d["steps"], rng_seed=7)
    return ctx, keys, d


def test_p16_sparse_bootstrap_vs_reference(p16, sparse):
    ctx, keys, d = sparse
    g = golden_npz("boot_p16_sparse.npz")
    v = np.tile(g["v"], p16.slot_count // 1024)
    ct = ckks.encrypt_vector(p16, v, keys, level=0, rng_seed=21)
    assert ct_digest(ct) == d["enc"]  # the reference's input ciphertext, bit for bit
    out = bs.bootstrap(ct, ctx, keys)
    assert out.level == ctx.output_level == d["out_level"]
    assert out.scale == p16.default_scale
    dec = ckks.decrypt_vector(out, keys)
    err = float(np.max(np.abs(dec - v)))
    print(f"P16 sparse-1024 bootstrap: err {err:.3e} (reference {d['err']:.3e})")
    assert err <= 1e-3
    assert err <= d["err"] * 1.05  # no worse than the reference on the same ciphertext
    assert np.max(np.abs(dec[:1024] - g["dec"])) <= 2e-3


def test_p16_sparse_bootstrap_double_angle(p16, sparse):
    """The double-angle EvalMod (degree-31 cos + 3 squarings, the trainer's
    refresh in bench.py) on the reference's ciphertext: within 1e-3."""
    _, keys, d = sparse
    ctx = bs.build_context(p16, n_slots=1024, input_periodic=True, evalmod="double_angle")
    missing = set(ctx.required_rotation_steps()) - set(keys.rotation_keys)
    assert not missing
    g = golden_npz("boot_p16_sparse.npz")
    v = np.tile(g["v"], p16.slot_count // 1024)
    ct = ckks.encrypt_vector(p16, v, keys, level=0, rng_seed=21)
    out = bs.bootstrap(ct, ctx, keys)
    assert out.level == ctx.output_level == p16.max_level - 11
    err = float(np.max(np.abs(ckks.decrypt_vector(out, keys) - v)))
    print(f"P16 sparse-1024 double-angle bootstrap: err {err:.3e}")
    assert err <= 1e-3


def test_p16_full_slot_bootstrap(p16):
    """Full-slot (32,768 slots) ingest bootstrap at P16.  The P16 preset keeps
    the reference's parameters (q0/scale = 32, EvalMod at scale 2^40), whose
    EvalMod noise bounds this at ~1.7e-3; the reference's own
    full-slot error at desk-boot is 3.9e-3 (tests/golden/boot_desk_full.npz).
    Batched (B=2) and unbatched outputs must agree."""
    ctx = bs.build_context(p16, n_slots=p16.slot_count)
    keys = ckks.keygen(p16, rotation_steps=ctx.required_rotation_steps(), rng_seed=7)
    rng = np.random.default_rng(1003)
    vs = [rng.uniform(-1, 1, p16.slot_count) for _ in range(2)]
    cts = [ckks.encrypt_vector(p16, v, keys, level=0, rng_seed=40 + i) for i, v in enumerate(vs)]
    one = bs.bootstrap(cts[0], ctx, keys)
    both = bs.bootstrap_many(cts, ctx, keys)
    errs = [float(np.max(np.abs(ckks.decrypt_vector(o, keys) - v))) for o, v in zip(both, vs)]
    e1 = float(np.max(np.abs(ckks.decrypt_vector(one, keys) - vs[0])))
    print(f"P16 full-slot bootstrap: err B=1 {e1:.3e}, B=2 {errs}")
    assert one.level == ctx.output_level and all(o.level == one.level for o in both)
    assert max(errs + [e1]) <= 2.5e-3
    assert np.array_equal(one.c0.limbs, both[0].c0.limbs)  # batching does not change limbs


@pytest.fixture(scope="module")
def trained(p16, sigmoid15):
    """8 minibatches (64 rows = 2 ciphertexts each) through the public
    logreg.train(): batched full-slot ingest of the level-3 transport
    ciphertexts, sparse-1024 bootstrap refresh of w and u."""
    import hashlib

    from paper_2210_02574_b200.synth import make_separable

    g = golden_npz("logreg_p16.npz")
    X, y = make_separable(np.random.default_rng(100), 1024, dim=768, margin=0.5)
    assert hashlib.sha256(np.ascontiguousarray(X).tobytes()).hexdigest() == str(g["X_sha256"])
    assert np.array_equal(y, g["y"])
    Xtr, ytr = X[:512], y[:512]
    layout = logreg.make_layout(p16, 768)
    # the bench's configuration: double-angle EvalMod for the weight refresh
    ctx = bs.build_context(p16, n_slots=layout.padded_dim, input_periodic=True,
                           evalmod="double_angle")
    ctx_full = bs.build_context(p16, n_slots=p16.slot_count)
    steps = sorted(set(bs.refresh_rotation_steps(ctx)) | set(logreg.rotation_steps(layout))
                   | set(ctx_full.required_rotation_steps()))
    keys = ckks.keygen(p16, rotation_steps=steps, rng_seed=7)
    pairs = logreg.pack_batch(Xtr, ytr, layout, p16, keys)
    cfg = logreg.TrainConfig(0.25, 0.9, 64, 1)
    model, timing = logreg.train(pairs, 512, cfg, p16, keys, sigmoid15,
                                 bs.BootstrapRefresher(ctx, keys), layout=layout,
                                 data_refresher=bs.BootstrapRefresher(ctx_full, keys))
    got = logreg.decrypted_weights(model, keys)
    return g, X, y, layout, got, timing


def test_p16_training_vs_reference_and_shadow(trained, sigmoid15):
    g, X, y, layout, got, timing = trained
    ref, shadow = g["ref_weights"], g["shadow_weights"]
    gap_ref = float(np.max(np.abs(got - ref)))
    gap_shadow = float(np.max(np.abs(got - shadow)))
    print(f"P16 8-minibatch training: |w - w_ref| {gap_ref:.3e}, |w - w_shadow| "
          f"{gap_shadow:.3e}, epoch {timing[0]['seconds']:.2f}s")
    assert timing[0]["level_refreshes"] == 16
    assert gap_ref <= 2e-2
    assert gap_shadow <= 2e-2


def test_p16_training_test_accuracy(trained, sigmoid15):
    g, X, y, layout, got, _ = trained
    Xte, yte = X[512:], y[512:]

    def acc(w):
        s = np.asarray(logreg.shadow_scores(Xte, w, sigmoid15, layout)).ravel()
        return float(np.mean((s > 0.5).astype(int) == yte))

    a_enc, a_sh, a_ref = acc(got), acc(g["shadow_weights"]), acc(g["ref_weights"])
    print(f"held-out accuracy: encrypted {a_enc:.4f}, shadow {a_sh:.4f}, reference {a_ref:.4f}")
    assert abs(a_enc - a_sh) <= 0.002
    assert abs(a_enc - a_ref) <= 0.002
