"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Outputs (committed): tests/golden/*.npz and tests/golden/digests.json.  Small
cases store full arrays; large ones store SHA-256 digests of the little-endian
limb bytes plus the seeds that recreate their inputs.  Nothing in the GPU tests
or the bench reads /root/reference; they read these files.
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))

from hebert import _kernels, bootstrap as bs, ckks, logreg, minimax, ring  # noqa: E402
from hebert.ckks import keys as K, ops  # noqa: E402


def sha(arr):
    return hashlib.sha256(np.ascontiguousarray(arr, dtype="<u8").tobytes()).hexdigest()


def ct_digest(ct):
    return {"c0": sha(ct.c0.limbs), "c1": sha(ct.c1.limbs), "level": ct.level,
            "scale": float(ct.scale).hex()}


def load_preset(name):
    path = os.path.join(REPO, "paper_2210_02574_b200", "presets", f"{name}.preset")
    with open(path) as fh:
        return ckks.CkksParams.from_config_text(fh.read())


def kernels_fixture():
    rng = np.random.default_rng(11)
    n = 64
    primes = ring.generate_ntt_primes(61, 2, n)
    q = np.array(primes, dtype=np.uint64)
    qinv = np.array([(-pow(int(p), -1, 1 << 64)) % (1 << 64) for p in primes], dtype=np.uint64)
    r2 = np.array([(1 << 128) % int(p) for p in primes], dtype=np.uint64)
    a = np.stack([rng.integers(0, p, n, dtype=np.uint64) for p in primes])
    b = np.stack([rng.integers(0, p, n, dtype=np.uint64) for p in primes])
    a[:, 0] = 0
    b[:, 1] = 0
    a[:, 2] = q - 1
    b[:, 2] = q - 1
    c = np.array([rng.integers(0, p) for p in primes], dtype=np.uint64)
    p3 = ring.RingParams("k64", n, tuple(primes))
    st = p3.stacked(tuple(primes))
    hat = np.stack([rng.integers(0, p, n, dtype=np.uint64) for p in primes])
    # convert hat (rows under prime 0/1) into the 2 target primes
    punc = np.array([[rng.integers(0, p) for p in primes] for _ in range(2)], dtype=np.uint64)
    key = np.stack([rng.integers(0, primes[i % 2], n, dtype=np.uint64) for i in range(5)])
    rows = np.array([3, 0], dtype=np.int64)
    key[3] %= q[0]
    key[0] %= q[1]
    out = dict(q=q, qinv=qinv, r2=r2, a=a, b=b, c=c, hat=hat, punc=punc, key=key, rows=rows,
               psi_rev=st.psi_rev, ipsi_rev=st.ipsi_rev, ninv=st.ninv1)
    out["mulmod"] = _kernels.elementwise_mulmod(a, b, q, qinv, r2)
    out["mont"] = _kernels.elementwise_mont(a, b, q, qinv)
    out["rowwise"] = _kernels.rowwise_mont(a, c, q, qinv)
    out["add"] = _kernels.addmod_rows(a, b, q)
    out["sub"] = _kernels.submod_rows(a, b, q)
    out["bconv"] = _kernels.base_convert(hat, punc, q, qinv)
    acc = a.copy()
    out["fma"] = _kernels.fma_inplace(acc, b, a, q, qinv, r2).copy()
    acc = b.copy()
    out["fma_gather"] = _kernels.fma_gather_inplace(acc, a, key, rows, q, qinv, r2).copy()
    f = a.copy()
    out["ntt_fwd"] = _kernels.ntt_forward_inplace(f, st.psi_rev, q, qinv).copy()
    g = a.copy()
    out["ntt_inv"] = _kernels.ntt_inverse_inplace(g, st.ipsi_rev, st.ninv1, q, qinv).copy()
    np.savez_compressed(os.path.join(HERE, "kernels_n64.npz"), **out)


def ring_fixture():
    n = 64
    primes = tuple(ring.generate_ntt_primes(40, 3, n))
    p = ring.RingParams("r64", n, primes)
    rng = np.random.default_rng(2)
    x = ring.sample_poly(p, "uniform", 2, rng)
    y = ring.sample_poly(p, "uniform", 2, rng)
    xe, ye = ring.to_eval(x), ring.to_eval(y)
    out = dict(primes=np.array(primes, dtype=np.uint64), x=x.limbs, y=y.limbs, x_eval=xe.limbs,
               y_eval=ye.limbs, prod=ring.poly_mul(xe, ye).limbs,
               prod_coeff=ring.to_coeff(ring.poly_mul(xe, ye)).limbs)
    exps, pos = ring._eval_exponent_map(p)
    out["exps"] = exps
    for g in (3, 5, 127, 2 * n - 1):
        out[f"auto_eval_{g}"] = ring.poly_automorphism_eval(xe, g).limbs
        out[f"auto_coeff_{g}"] = ring.poly_automorphism(x, g).limbs
    signed = np.random.default_rng(3).integers(-(1 << 61), 1 << 61, size=n)
    out["signed"] = signed
    out["lifted"] = ring.limbs_from_signed(signed, primes)
    np.savez_compressed(os.path.join(HERE, "ring_n64.npz"), **out)


def scheme_digests(params, name, steps, seed=7, conj=True, full=True):
    t0 = time.time()
    keys = ckks.keygen(params, rotation_steps=steps, rng_seed=seed, include_conjugation=conj)
    d = {"keygen_seconds": time.time() - t0, "rotation_steps": list(keys.rotation_steps)}
    d["secret_ext"] = sha(keys.secret_ext)
    d["pk_b"] = sha(keys.public_key[0].limbs)
    d["pk_a"] = sha(keys.public_key[1].limbs)
    d["relin_b"] = [sha(x) for x in keys.relin_key.digits_b]
    d["relin_a"] = [sha(x) for x in keys.relin_key.digits_a]
    d["rot"] = {str(s): [sha(x) for x in keys.rotation_keys[s].digits_b]
                + [sha(x) for x in keys.rotation_keys[s].digits_a] for s in keys.rotation_steps}
    if conj:
        d["conj"] = [sha(x) for x in keys.conj_key.digits_b] + [sha(x) for x in keys.conj_key.digits_a]
    L = params.max_level
    # NTT of a seeded uniform poly at the top level
    up = ring.sample_poly(params.ring, "uniform", L, np.random.default_rng(1000))
    d["ntt_fwd"] = sha(ring.to_eval(up).limbs)
    d["ntt_inv"] = sha(ring.ntt_transform(ring.RnsPoly(params.ring, up.limbs.copy(), ring.EVAL, L),
                                          "inverse").limbs)
    # key switch of a seeded uniform eval-form d at several levels
    d["ks"] = {}
    for lvl in sorted({L, max(1, L // 2), 1}):
        dp = ring.sample_poly(params.ring, "uniform", lvl, np.random.default_rng(2000 + lvl))
        dp = ring.RnsPoly(params.ring, dp.limbs, ring.EVAL, lvl)
        kb, ka = K.ks_apply(keys, keys.relin_key, dp)
        d["ks"][str(lvl)] = [sha(kb.limbs), sha(ka.limbs)]
    rng = np.random.default_rng(5)
    slots = params.slot_count
    u = rng.uniform(-1, 1, slots)
    v = rng.uniform(-1, 1, slots)
    cu = ckks.encrypt_vector(params, u, keys, rng_seed=1)
    cv = ckks.encrypt_vector(params, v, keys, rng_seed=2)
    d["enc_u"] = ct_digest(cu)
    d["enc_v"] = ct_digest(cv)
    c3 = ckks.encrypt(ckks.encode(params, u[:768], 3), keys, rng_seed=3)
    d["enc_l3"] = ct_digest(c3)
    prod = ckks.mult(cu, cv, keys)
    d["mult"] = ct_digest(prod)
    d["mult_dec"] = ckks.decrypt_vector(prod, keys)[:64].tolist()
    d["add"] = ct_digest(ckks.add(cu, cv))
    d["sub"] = ct_digest(ckks.sub(cu, cv))
    d["rescale"] = ct_digest(ckks.rescale(ops.mult_plain(cu, 0.5, rescale_after=False)))
    d["mult_plain_vec"] = ct_digest(ckks.mult_plain(cu, v))
    d["add_plain_const"] = ct_digest(ckks.add_plain(cu, 0.25))
    d["mod_down"] = ct_digest(ckks.mod_down(cu, max(1, L // 2)))
    d["add_aligned"] = ct_digest(ckks.add(prod, ckks.mod_down(cv, prod.level - 1)))
    if full:
        for s in steps:
            d[f"rot_{s}"] = ct_digest(ckks.rotate(cu, s, keys))
        d["rot_3"] = ct_digest(ckks.rotate(cu, 3, keys))
        if conj:
            d["conj_ct"] = ct_digest(ckks.conjugate(cu, keys))
        d["dec_u"] = ckks.decrypt_vector(cu, keys)[:64].tolist()
    return d, keys


def desk_extra(params, keys, d):
    path = os.path.join(REPO, "paper_2210_02574_b200", "approximants", "sigmoid_deg15.txt")
    sig = minimax.import_text(open(path).read())
    pts = np.linspace(-12, 12, params.slot_count)
    ct = ckks.encrypt_vector(params, pts, keys, rng_seed=9)
    out = ckks.eval_poly_bsgs(ct, sig, keys)
    d["sigmoid_bsgs"] = ct_digest(out)
    d["sigmoid_dec"] = ckks.decrypt_vector(out, keys)[:64].tolist()


def boot_fixture():
    params = ckks.get_preset("desk-boot")
    ctx = bs.build_context(params, n_slots=64)
    steps = sorted(set(list(ckks.default_rotation_steps(params)) + ctx.required_rotation_steps()))
    t0 = time.time()
    keys = ckks.keygen(params, rotation_steps=steps, rng_seed=11)
    tk = time.time() - t0
    v = np.random.default_rng(1002).uniform(-1, 1, 64)
    ct = ckks.encrypt_vector(params, v, keys, level=0, rng_seed=21)
    raised = bs._mod_raise(ct)
    t0 = time.time()
    out = bs.bootstrap(ct, ctx, keys)
    tb = time.time() - t0
    dec = ckks.decrypt_vector(out, keys)
    res = {"steps": steps, "keygen_seconds": tk, "bootstrap_seconds": tb,
           "enc": ct_digest(ct), "mod_raise": ct_digest(raised), "out_level": out.level,
           "out_scale": float(out.scale).hex(), "err": float(np.max(np.abs(dec[:64] - v))),
           "sine_coeffs": [float(c).hex() for c in ctx.evalmod_poly.cheb_coeffs]}
    np.savez_compressed(os.path.join(HERE, "boot_desk64.npz"), v=v, dec=dec)
    return res


def boot_full_fixture():
    """Full-slot (4,096 slots) bootstrap at desk-boot, N = 2^13: the
    reference's error on one seeded ciphertext (its diagonals are the ones
    the GPU encoder generates, bootstrap.py:319-335)."""
    params = ckks.get_preset("desk-boot")
    ctx = bs.build_context(params, n_slots=params.slot_count)
    steps = sorted(set(ctx.required_rotation_steps()))
    keys = ckks.keygen(params, rotation_steps=steps, rng_seed=11)
    v = np.random.default_rng(1003).uniform(-1, 1, params.slot_count)
    ct = ckks.encrypt_vector(params, v, keys, level=0, rng_seed=22)
    t0 = time.time()
    out = bs.bootstrap(ct, ctx, keys)
    tb = time.time() - t0
    dec = ckks.decrypt_vector(out, keys)
    np.savez_compressed(os.path.join(HERE, "boot_desk_full.npz"), v=v, dec=dec)
    return {"steps": steps, "enc": ct_digest(ct), "out_level": out.level,
            "bootstrap_seconds": tb, "err": float(np.max(np.abs(dec - v)))}


def _sigmoid15():
    path = os.path.join(REPO, "paper_2210_02574_b200", "approximants", "sigmoid_deg15.txt")
    return minimax.import_text(open(path).read())


def predict_p14_fixture():
    """BASELINE cfg1: N=2^14 (P14) encrypt -> 768-d logistic-regression
    inference on one ciphertext of 8 rows -> decrypt."""
    params = load_preset("p14")
    keys = ckks.keygen(params, rng_seed=7)
    layout = logreg.make_layout(params, 768)
    X = np.random.default_rng(0).uniform(-1, 1, (8, 768))
    w = np.random.default_rng(0).normal(0, 0.05, 768)
    data = ckks.encrypt_vector(params, logreg._pack_slots(X, layout), keys, rng_seed=1)
    wv = np.zeros(layout.slot_count)
    for b in range(layout.rows_per_ct):
        wv[b * layout.padded_dim: b * layout.padded_dim + 768] = w
    wct = ckks.encrypt_vector(params, wv, keys, rng_seed=2)
    model = logreg.EncryptedModel(2, layout, [wct], [wct])
    sig = _sigmoid15()
    t0 = time.time()
    scores = logreg.predict(model, [data], keys, sig)
    tp = time.time() - t0
    dec = logreg.decrypt_scores(scores, keys, layout, 8)
    shadow = logreg.shadow_scores(X, np.concatenate([w, np.zeros(layout.padded_dim - 768)])[None, :],
                                  sig, layout)
    np.savez_compressed(os.path.join(HERE, "predict_p14.npz"), X=X, w=w, dec=dec,
                        shadow=np.asarray(shadow))
    return {"data": ct_digest(data), "weights": ct_digest(wct), "scores": ct_digest(scores[0][0]),
            "predict_seconds": tp}


def ovr_fixture():
    """BASELINE cfg5 semantics at desk scale: One-vs-Rest (logreg.py:325-331)
    over 4 classes of 1024-d blob embeddings, debug refresh, 1 epoch."""
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "ref_conftest", "/root/reference/pkg/tests/conftest.py")
    rc = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(rc)
    params = ckks.get_preset("desk")
    X, y = rc.make_blob_embeddings(np.random.default_rng(200), 8, 4, dim=1024)
    X = X * 0.25  # keeps every logit inside the sigmoid's fitted domain (|z| <= 12)
    layout = logreg.make_layout(params, 1024)
    keys = ckks.keygen(params, rotation_steps=sorted(set(ckks.default_rotation_steps(params))),
                       rng_seed=7)
    pairs = logreg.pack_batch(X, y.astype(np.float64), layout, params, keys)
    ovr = logreg.pack_labels_ovr(y, 4, layout, params, keys)
    cfg = logreg.TrainConfig(0.5, 0.9, 16, 1)
    sig = _sigmoid15()
    t0 = time.time()
    model, _ = logreg.train(pairs, len(y), cfg, params, keys, sig,
                            bs.DebugRefresher(keys, enabled=True), class_count=4, ovr_labels=ovr,
                            layout=layout)
    tt = time.time() - t0
    got = logreg.decrypted_weights(model, keys)
    shadow = logreg.shadow_train(X, y, cfg, sig, class_count=4, layout=layout)
    np.savez_compressed(os.path.join(HERE, "ovr_desk.npz"), X=X, y=y, ref_weights=got,
                        shadow_weights=np.asarray(shadow.weights))
    return {"train_seconds": tt}


def boot_p16_sparse_fixture():
    """P16 (N=2^16) sparse-1024 periodic bootstrap of one seeded ciphertext: the
    reference's own decrypted output and error (
    bootstrap.py:278-349).  The GPU test bootstraps the same (bit-exact)
    ciphertext and must be within 1e-3 and no worse than 2x this error."""
    params = load_preset("p16")
    ctx = bs.build_context(params, n_slots=1024, input_periodic=True)
    steps = sorted(set(ctx.required_rotation_steps()))
    t0 = time.time()
    keys = ckks.keygen(params, rotation_steps=steps, rng_seed=7)
    tk = time.time() - t0
    v = np.tile(np.random.default_rng(1002).uniform(-1, 1, 1024), params.slot_count // 1024)
    ct = ckks.encrypt_vector(params, v, keys, level=0, rng_seed=21)
    t0 = time.time()
    out = bs.bootstrap(ct, ctx, keys)
    tb = time.time() - t0
    dec = ckks.decrypt_vector(out, keys)
    np.savez_compressed(os.path.join(HERE, "boot_p16_sparse.npz"), v=v[:1024], dec=dec[:1024])
    return {"steps": steps, "keygen_seconds": tk, "bootstrap_seconds": tb, "enc": ct_digest(ct),
            "out_level": out.level, "out_scale": float(out.scale).hex(),
            "err": float(np.max(np.abs(dec - v)))}


def logreg_p16_fixture():
    """cfg4 shape at P16 (768-d rows, 32 rows per ciphertext): 8 minibatches of
    64 rows trained by the reference with its debug refresher, plus the shadow
    trainer's weights and held-out accuracies (logreg.py:290-417;
    test_acceptance.py:98-131 pattern)."""
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "ref_conftest", "/root/reference/pkg/tests/conftest.py")
    rc = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(rc)
    params = load_preset("p16")
    X, y = rc.make_separable(np.random.default_rng(100), 1024, dim=768, margin=0.5)
    Xtr, ytr, Xte, yte = X[:512], y[:512], X[512:], y[512:]
    layout = logreg.make_layout(params, 768)
    keys = ckks.keygen(params, rotation_steps=sorted(set(ckks.default_rotation_steps(params))),
                       rng_seed=7)
    pairs = logreg.pack_batch(Xtr, ytr, layout, params, keys)
    cfg = logreg.TrainConfig(0.25, 0.9, 64, 1)  # lr/B as in test_acceptance; 1.0 diverges
    sig = _sigmoid15()

    class LevelDebugRefresher:
        """bootstrap.debug_refresh (bootstrap.py:352-369) re-encrypting at the
        sparse bootstrap's output level L-10 instead of the top: at P16 the
        top prime is 60 bits and the reference's own level alignment of
        top-level ciphertexts overflows encode_const (ops.py:55-61)."""

        insecure = True
        output_level = params.max_level - 10

        def refresh(self, ct):
            from hebert.ckks.encoding import decode_real, encode

            vals = decode_real(ops.decrypt(ct, keys))
            out = ops.encrypt(encode(params, vals, self.output_level, params.default_scale), keys)
            out.insecure_provenance = True
            return out

    t0 = time.time()
    model, timing = logreg.train(pairs, len(ytr), cfg, params, keys, sig, LevelDebugRefresher(),
                                 layout=layout)
    tt = time.time() - t0
    got = logreg.decrypted_weights(model, keys)
    shadow = logreg.shadow_train(Xtr, ytr, cfg, sig, layout=layout)

    def acc(w):
        s = logreg.shadow_scores(Xte, w, sig, layout)
        return float(np.mean((np.asarray(s) > 0.5).astype(int).ravel() == yte))

    # X is regenerated by the tests from its seed (synth.make_separable mirrors
    # T/conftest.py:68-82); its digest pins it
    np.savez_compressed(os.path.join(HERE, "logreg_p16.npz"), y=y,
                        X_sha256=hashlib.sha256(np.ascontiguousarray(X).tobytes()).hexdigest(),
                        ref_weights=got, shadow_weights=np.asarray(shadow.weights))
    return {"train_seconds": tt, "epoch_seconds": timing[0]["seconds"],
            "ref_acc": acc(got), "shadow_acc": acc(shadow.weights),
            "w_gap": float(np.max(np.abs(got - shadow.weights))),
            "domain_breaches": int(shadow.domain_breaches)}


def sine_artifact():
    """The EvalMod sine the reference fits at runtime for h = 64 (K = 14,
    bootstrap.py:98-107), shipped as paper_2210_02574_b200/approximants/
    sine2pi_k14_deg119.txt so the engine evaluates the reference's exact
    polynomial."""
    poly = minimax.remez_fit("sine2pi", (-14.5, 14.5), 119)
    path = os.path.join(REPO, "paper_2210_02574_b200", "approximants", "sine2pi_k14_deg119.txt")
    with open(path, "w") as fh:
        fh.write(minimax.export_text(poly))
    return [float(c).hex() for c in poly.cheb_coeffs]


def logreg_fixture():
    params = ckks.get_preset("desk")
    keys = ckks.keygen(params, rng_seed=7)
    path = os.path.join(REPO, "paper_2210_02574_b200", "approximants", "sigmoid_deg15.txt")
    sig = minimax.import_text(open(path).read())
    rng = np.random.default_rng(0)
    X = rng.uniform(-1, 1, (256, 16))
    w = rng.normal(size=16)
    y = (X @ w > 0).astype(np.int64)
    layout = logreg.make_layout(params, 16)
    pairs = logreg.pack_batch(X, y, layout, params, keys)
    cfg = logreg.TrainConfig(1.0, 0.9, 128, 2)
    model, _ = logreg.train(pairs, 256, cfg, params, keys, sig,
                            bs.DebugRefresher(keys, enabled=True), layout=layout)
    got = logreg.decrypted_weights(model, keys)
    shadow = logreg.shadow_train(X, y, cfg, sig, layout=layout)
    np.savez_compressed(os.path.join(HERE, "logreg_desk.npz"), X=X, y=y, ref_weights=got,
                        shadow_weights=shadow.weights)


def wire_fixture():
    """CKT1 / CKK1 / HLR1 bytes of the reference (serial.py:61-209, logreg.py:583-633)
    for seeded desk material: SHA-256 of each blob and its length."""
    import hashlib as _h

    from hebert.ckks import serial as S

    params = ckks.get_preset("desk")
    keys = ckks.keygen(params, rotation_steps=[1, -1, 2, 4], rng_seed=7, include_conjugation=True)
    rng = np.random.default_rng(5)
    u = rng.uniform(-1, 1, params.slot_count)
    cts = [ckks.encrypt_vector(params, u * (i + 1) / 4, keys, rng_seed=20 + i) for i in range(4)]
    layout = logreg.make_layout(params, 100)
    model = logreg.EncryptedModel(3, layout, cts[:3], [cts[3]] * 3, "secure")
    blobs = {"ckt1": S.serialize_ciphertext(cts[0]),
             "ckk1_eval": S.serialize_keyset(keys, include_secret=False),
             "ckk1_secret": S.serialize_keyset(keys, include_secret=True),
             "hlr1": logreg.serialize_model(model)}
    return {k: {"sha256": _h.sha256(b).hexdigest(), "bytes": len(b)} for k, b in blobs.items()}


def main():
    t0 = time.time()
    only = {"boot_full": ("boot_desk_full", boot_full_fixture),
            "predict_p14": ("predict_p14", predict_p14_fixture),
            "ovr": ("ovr_desk", ovr_fixture),
            "boot_p16_sparse": ("boot_p16_sparse", boot_p16_sparse_fixture),
            "logreg_p16": ("logreg_p16", logreg_p16_fixture),
            "sine_artifact": ("sine_artifact", sine_artifact),
            "wire": ("wire_desk", wire_fixture),
            "p16s": ("p16s", lambda: scheme_digests(load_preset("p16s"), "p16s", [1], conj=False,
                                                    full=False)[0])}
    if sys.argv[1:] and sys.argv[1] in only:  # add / refresh only these entries
        path = os.path.join(HERE, "digests.json")
        digests = json.load(open(path))
        for name in sys.argv[1:]:
            key, fn = only[name]
            digests[key] = fn()
            with open(path, "w") as fh:  # after each: a later failure keeps this one
                json.dump(digests, fh, indent=1, sort_keys=True)
        print("%s written in %.1fs" % (sys.argv[1:], time.time() - t0), file=sys.stderr)
        return
    kernels_fixture()
    ring_fixture()
    digests = {}
    desk = ckks.get_preset("desk")
    d, keys = scheme_digests(desk, "desk", [1, -1, 2, 4])
    desk_extra(desk, keys, d)
    digests["desk"] = d
    for name in ("p14", "p16"):
        params = load_preset(name)
        digests[name], _ = scheme_digests(params, name, [1], conj=False, full=(name == "p14"))
        print(name, "done", time.time() - t0, file=sys.stderr)
    digests["boot_desk64"] = boot_fixture()
    digests["boot_desk_full"] = boot_full_fixture()
    digests["predict_p14"] = predict_p14_fixture()
    digests["ovr_desk"] = ovr_fixture()
    ref_sig = os.path.join(os.path.dirname(minimax.__file__), "approximants", "sigmoid_deg15.txt")
    digests["sigmoid_ref"] = [float(c).hex() for c in
                              minimax.import_text(open(ref_sig).read()).cheb_coeffs]
    logreg_fixture()
    with open(os.path.join(HERE, "digests.json"), "w") as fh:
        json.dump(digests, fh, indent=1, sort_keys=True)
    print("golden fixtures written in %.1fs" % (time.time() - t0), file=sys.stderr)


if __name__ == "__main__":
    main()
