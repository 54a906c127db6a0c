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
