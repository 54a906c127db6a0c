"""GPU encrypted logistic regression vs the reference's trained weights and
the plaintext shadow oracle (T/test_logreg.py, T/test_acceptance.py)."""

import numpy as np
import pytest

from conftest import golden_npz, make_separable

pytestmark = pytest.mark.gpu

from paper_2210_02574_b200 import bootstrap as bs, ckks, logreg  # noqa: E402


@pytest.fixture(scope="module")
def desk():
    params = ckks.get_preset("desk")
    return params, ckks.keygen(params, rng_seed=7)


def test_training_matches_reference_and_shadow(desk, sigmoid15):
    params, keys = desk
    g = golden_npz("logreg_desk.npz")
    X, y = g["X"], g["y"]
    layout = logreg.make_layout(params, 16)
    pairs = logreg.pack_batch(X, y, layout, params, keys)
    cfg = logreg.TrainConfig(1.0, 0.9, 128, 2)
    model, timing = logreg.train(pairs, 256, cfg, params, keys, sigmoid15,
                                 bs.DebugRefresher(keys, enabled=True), layout=layout)
    got = logreg.decrypted_weights(model, keys)
    shadow = logreg.shadow_train(X, y, cfg, sigmoid15, layout=layout)
    assert np.array_equal(shadow.weights, g["shadow_weights"])  # host mirror is exact
    assert np.max(np.abs(got - shadow.weights)) <= 2e-2
    assert np.max(np.abs(got - g["ref_weights"])) <= 2e-2
    assert model.provenance == "insecure_debug_refresh"
    assert timing[0]["level_refreshes"] == 4


def test_training_hoisted_rotsum_radix4(sigmoid15):
    """With the radix-4 rotation keys (logreg.rotation_steps) every
    rotate-and-sum round runs 3 rotations through one hoisted key switch;
    the trained weights still track the shadow trainer and the reference."""
    params = ckks.get_preset("desk")
    g = golden_npz("logreg_desk.npz")
    X, y = g["X"], g["y"]
    layout = logreg.make_layout(params, 16)
    keys = ckks.keygen(params, rotation_steps=sorted(logreg.rotation_steps(layout)), rng_seed=7)
    assert all(s in keys.rotation_keys for s in (3, -3, 12, -12))
    pairs = logreg.pack_batch(X, y, layout, params, keys)
    cfg = logreg.TrainConfig(1.0, 0.9, 128, 2)
    model, _ = logreg.train(pairs, 256, cfg, params, keys, sigmoid15,
                            bs.DebugRefresher(keys, enabled=True), layout=layout)
    got = logreg.decrypted_weights(model, keys)
    assert np.max(np.abs(got - g["shadow_weights"])) <= 2e-2
    assert np.max(np.abs(got - g["ref_weights"])) <= 2e-2


def test_encrypted_vs_shadow_acceptance(desk, sigmoid15):
    """Acceptance criterion (T/test_acceptance.py:98-131), 1000 rows x 768."""
    params, keys = desk
    rng = np.random.default_rng(100)
    X, y = make_separable(rng, 1200, dim=768, margin=0.5)
    Xtr, ytr, Xte, yte = X[:1000], y[:1000], X[1000:], y[1000:]
    layout = logreg.make_layout(params, 768)
    pairs = logreg.pack_batch(Xtr, ytr, layout, params, keys)
    cfg = logreg.TrainConfig(1.0, 0.9, 512, 1)
    model, _ = logreg.train(pairs, 1000, cfg, params, keys, sigmoid15,
                            bs.DebugRefresher(keys, enabled=True), layout=layout)
    shadow = logreg.shadow_train(Xtr, ytr, cfg, sigmoid15, layout=layout)
    got = logreg.decrypted_weights(model, keys)
    assert np.max(np.abs(got - shadow.weights)) <= 2e-2
    enc_acc = np.mean((logreg.shadow_scores(Xte, got, sigmoid15, layout) > 0.5) == yte)
    sh_acc = np.mean((logreg.shadow_scores(Xte, shadow.weights, sigmoid15, layout) > 0.5) == yte)
    assert abs(enc_acc - sh_acc) <= 0.02 and sh_acc >= 0.95


def test_predict_scores(desk, sigmoid15):
    params, keys = desk
    rng = np.random.default_rng(6)
    layout = logreg.make_layout(params, 16)
    X = rng.uniform(-1, 1, (32, 16))
    w = np.zeros(layout.padded_dim)
    w[:16] = rng.normal(0, 0.3, 16)
    wslots = np.tile(w, layout.rows_per_ct)
    model = logreg.EncryptedModel(2, layout, [ckks.encrypt_vector(params, wslots, keys)],
                                  [ckks.encrypt_vector(params, 0 * wslots, keys)])
    pairs = logreg.pack_batch(X, np.zeros(32), layout, params, keys)
    scores = logreg.predict(model, [pairs[0][0]], keys, sigmoid15,
                            refresher=bs.DebugRefresher(keys, enabled=True))
    got = logreg.decrypt_scores(scores, keys, layout, 32)
    want = logreg.shadow_scores(X, w[None, :], sigmoid15, layout)
    assert np.max(np.abs(got - want)) < 1e-2


def test_packing_roundtrip(desk):
    params, keys = desk
    layout = logreg.make_layout(params, 768)
    assert layout.padded_dim == 1024 and layout.rows_per_ct == 4
    rng = np.random.default_rng(1)
    X = rng.uniform(-1, 1, (8, 768))
    pairs = logreg.pack_batch(X, np.zeros(8), layout, params, keys)
    assert len(pairs) == 2 and pairs[0][0].level == logreg.DEFAULT_TRANSPORT_LEVEL
    slots = ckks.decrypt_vector(pairs[0][0], keys)
    assert np.max(np.abs(logreg.unpack_rows(slots, layout, 4) - X[:4])) < 1e-4


def test_predict_p14_cfg1_matches_reference(digests, sigmoid15):
    """BASELINE cfg1: P14 (N=2^14) encrypt -> 768-d
    inference on one ciphertext of 8 rows -> decrypt.  The seeded data and
    weight ciphertexts are bit-exact with the reference's; the decrypted
    scores match the reference's run and the plaintext shadow."""
    d = digests["predict_p14"]
    g = golden_npz("predict_p14.npz")
    params = ckks.get_preset("p14")
    keys = ckks.keygen(params, rng_seed=7)
    layout = logreg.make_layout(params, 768)
    X, w = g["X"], g["w"]
    data = ckks.encrypt_vector(params, logreg._pack_slots(X, layout), keys, rng_seed=1)
    wv = np.zeros(layout.slot_count)
    for b in range(layout.rows_per_ct):
        wv[b * layout.padded_dim: b * layout.padded_dim + 768] = w
    wct = ckks.encrypt_vector(params, wv, keys, rng_seed=2)
    from oracle.scheme import sha

    for ct, want in ((data, d["data"]), (wct, d["weights"])):
        assert {"c0": sha(ct.c0.limbs), "c1": sha(ct.c1.limbs), "level": ct.level,
                "scale": float(ct.scale).hex()} == want
    model = logreg.EncryptedModel(2, layout, [wct], [wct])
    scores = logreg.predict(model, [data], keys, sigmoid15)
    assert scores[0][0].level == d["scores"]["level"]
    got = logreg.decrypt_scores(scores, keys, layout, 8)
    assert np.max(np.abs(got - g["dec"])) < 1e-4  # the reference's decrypted scores
    assert np.max(np.abs(got - g["shadow"])) < 1e-2  # T/test_logreg.py:259


def test_ovr_multiclass_1024d_matches_reference(sigmoid15):
    """BASELINE cfg5 semantics (One-vs-Rest, logreg.py:325-331) at desk
    scale: 4 classes of 1024-d embeddings (2 rows per ciphertext); weights
    against the reference's trained weights and the shadow trainer, argmax
    agreement with the shadow (T/test_acceptance.py:171)."""
    g = golden_npz("ovr_desk.npz")
    X, y = g["X"], g["y"]
    params = ckks.get_preset("desk")
    keys = ckks.keygen(params, rotation_steps=sorted(set(ckks.default_rotation_steps(params))),
                       rng_seed=7)
    layout = logreg.make_layout(params, 1024)
    assert layout.padded_dim == 2048 and layout.rows_per_ct == 2
    pairs = logreg.pack_batch(X, y.astype(np.float64), layout, params, keys)
    ovr = logreg.pack_labels_ovr(y, 4, layout, params, keys)
    cfg = logreg.TrainConfig(0.5, 0.9, 16, 1)
    model, _ = logreg.train(pairs, len(y), cfg, params, keys, sigmoid15,
                            bs.DebugRefresher(keys, enabled=True), class_count=4, ovr_labels=ovr,
                            layout=layout)
    assert len(model.weights) == 4
    got = logreg.decrypted_weights(model, keys)
    shadow = logreg.shadow_train(X, y, cfg, sigmoid15, class_count=4, layout=layout)
    assert np.array_equal(np.asarray(shadow.weights), g["shadow_weights"])
    assert np.max(np.abs(got - shadow.weights)) <= 2e-2
    assert np.max(np.abs(got - g["ref_weights"])) <= 2e-2
    enc = logreg.shadow_scores(X, got, sigmoid15, layout)
    sh = logreg.shadow_scores(X, np.asarray(shadow.weights), sigmoid15, layout)
    assert np.mean(np.argmax(enc, axis=1) == np.argmax(sh, axis=1)) >= 0.98


def test_captured_minibatch_graphs_match_eager(sigmoid15):
    """The bench's graph-replayed trainer steps (desk-boot, true bootstrap
    refresh): CapturedMinibatch reproduces the eager train_minibatch limb for
    limb; CapturedShardedMinibatch (the multi-GPU form: gradient graph, eager
    collectives, per-owner refresh graphs), run at world size 1, decrypts like
    it (w and u are bootstrapped separately there instead of packed)."""
    from paper_2210_02574_b200.ckks import ops

    params = ckks.get_preset("desk-boot")
    layout = logreg.make_layout(params, 16)
    ctx = bs.build_context(params, n_slots=layout.padded_dim, input_periodic=True)
    steps = sorted(set(bs.refresh_rotation_steps(ctx)) | logreg.rotation_steps(layout))
    keys = ckks.keygen(params, rotation_steps=steps, rng_seed=7)
    ref = bs.BootstrapRefresher(ctx, keys)
    cfg = logreg.TrainConfig(1.0, 0.9, 4 * layout.rows_per_ct, 1)
    rng = np.random.default_rng(12)
    X = rng.uniform(-1, 1, (cfg.batch_size, 16))
    y = (X @ rng.normal(size=16) > 0).astype(np.float64)
    top = ctx.output_level
    xs, ys = [], []
    for c in range(4):
        r0 = c * layout.rows_per_ct
        xr, yr = X[r0: r0 + layout.rows_per_ct], y[r0: r0 + layout.rows_per_ct]
        xs.append(ckks.encrypt(ckks.encode(params, logreg._pack_slots(xr, layout), top), keys,
                               rng_seed=100 + c))
        ys.append(ckks.encrypt(ckks.encode(params, logreg._pack_label_slots(yr, layout), 3), keys,
                               rng_seed=200 + c))
    xb, yb = ops.stack(xs), ops.stack(ys)
    w0, u0 = logreg._zeros_ct(params, keys, top), logreg._zeros_ct(params, keys, top)
    args = (cfg.batch_size, cfg, keys, sigmoid15, layout, ref)
    we, ue = logreg.train_minibatch(w0, u0, xb, yb, *args, local_shard=True)
    cm = logreg.CapturedMinibatch(w0, u0, xb, yb, *args)
    cm.load(xb, yb)
    wg, ug = cm.step()
    assert np.array_equal(wg.c0.limbs, we.c0.limbs) and np.array_equal(ug.c1.limbs, ue.c1.limbs)
    # the OvR bench form: a second class's graph shares the first one's pool
    # (replayed in capture order); each stays bit-exact with its eager update
    yb2 = ops.stack([ckks.encrypt(ckks.encode(params, logreg._pack_label_slots(
        1.0 - y[c * layout.rows_per_ct: (c + 1) * layout.rows_per_ct], layout), 3), keys,
        rng_seed=300 + c) for c in range(4)])
    we2, ue2 = logreg.train_minibatch(w0, u0, xb, yb2, *args, local_shard=True)
    cm2 = logreg.CapturedMinibatch(w0, u0, xb, yb2, *args, pool=cm.pool)
    for _ in range(2):  # the second round replays over the first round's intermediates
        for g in (cm, cm2):
            for dst, src in ((g.w, w0), (g.u, u0)):
                dst.c0.data.copy_(src.c0.data)
                dst.c1.data.copy_(src.c1.data)
        cm.load(xb, yb)
        wg, ug = cm.step()
        cm2.load(cm.x, yb2)
        wg2, ug2 = cm2.step()
        assert np.array_equal(wg.c0.limbs, we.c0.limbs) and np.array_equal(ug.c1.limbs, ue.c1.limbs)
        assert np.array_equal(wg2.c0.limbs, we2.c0.limbs)
        assert np.array_equal(ug2.c1.limbs, ue2.c1.limbs)
    cs = logreg.CapturedShardedMinibatch(w0, u0, xb, yb, *args)
    cs.load(xb, yb)
    ws, us = cs.step()
    for a, b in ((ws, we), (us, ue)):
        assert a.level == b.level and a.scale == b.scale
        # two independent bootstraps' errors (desk-boot: ~1e-3 each; the
        # reference's bootstrap tolerance is 1e-2, T/test_bootstrap.py:23)
        assert np.max(np.abs(ckks.decrypt_vector(a, keys) - ckks.decrypt_vector(b, keys))) < 5e-3
