"""GPU parity for the CKKS layer: keygen, seeded encryption, key switching,
products, rotations, rescale -- limbs bit-exact against digests of the
reference's own outputs -- plus the reference's tolerance tests
(T/test_ckks.py)."""

import numpy as np
import pytest

from conftest import preset_text

pytestmark = pytest.mark.gpu

from oracle.scheme import sha  # noqa: E402  (digest helper only)
from paper_2210_02574_b200 import ckks, minimax, ring  # noqa: E402
from paper_2210_02574_b200.ckks import keys as K, ops  # noqa: E402
from paper_2210_02574_b200.errors import (  # noqa: E402
    CryptoError,
    MissingRotationKeyError,
    OutOfLevelsError,
    ScaleMismatchError,
)


def params_for(name):
    if name == "desk":
        return ckks.get_preset("desk")
    return ckks.CkksParams.from_config_text(preset_text(name))


def ct_digest(ct):
    return {"c0": sha(ct.c0.limbs), "c1": sha(ct.c1.limbs), "level": ct.level,
            "scale": float(ct.scale).hex()}


_KEYS = {}


def keyset(name, d):
    if name not in _KEYS:
        params = params_for(name)
        _KEYS[name] = (params, ckks.keygen(params, rotation_steps=d["rotation_steps"], rng_seed=7,
                                           include_conjugation="conj" in d))
    return _KEYS[name]


@pytest.mark.parametrize("name", ["desk", "p14", "p16", "p16s"])
def test_keygen_bit_exact(name, digests):
    d = digests[name]
    params, keys = keyset(name, d)
    assert sha(keys.secret_ext) == d["secret_ext"]
    assert sha(keys.public_key[0].limbs) == d["pk_b"]
    assert sha(keys.public_key[1].limbs) == d["pk_a"]
    assert [sha(x) for x in keys.relin_key.digits_b] == d["relin_b"]
    assert [sha(x) for x in keys.relin_key.digits_a] == d["relin_a"]
    for s, hs in d["rot"].items():
        k = keys.rotation_keys[int(s)]
        assert [sha(x) for x in k.digits_b] + [sha(x) for x in k.digits_a] == hs
    if "conj" in d:
        c = keys.conj_key
        assert [sha(x) for x in c.digits_b] + [sha(x) for x in c.digits_a] == d["conj"]


@pytest.mark.parametrize("name", ["desk", "p14", "p16", "p16s"])
def test_key_switch_bit_exact(name, digests):
    d = digests[name]
    params, keys = keyset(name, d)
    for lvl, want in d["ks"].items():
        lvl = int(lvl)
        dp = ring.sample_poly(params.ring, "uniform", lvl, np.random.default_rng(2000 + lvl))
        dp = ring.RnsPoly(params.ring, dp.limbs, ring.EVAL, lvl)
        kb, ka = K.ks_apply(keys, keys.relin_key, dp)
        assert [sha(kb.limbs), sha(ka.limbs)] == want, f"level {lvl}"


@pytest.mark.parametrize("name", ["desk", "p14", "p16", "p16s"])
def test_ciphertext_ops_bit_exact(name, digests):
    d = digests[name]
    params, keys = keyset(name, d)
    L = params.max_level
    rng = np.random.default_rng(5)
    u = rng.uniform(-1, 1, params.slot_count)
    v = rng.uniform(-1, 1, params.slot_count)
    cu = ckks.encrypt_vector(params, u, keys, rng_seed=1)
    cv = ckks.encrypt_vector(params, v, keys, rng_seed=2)
    assert ct_digest(cu) == d["enc_u"]
    assert ct_digest(cv) == d["enc_v"]
    c3 = ckks.encrypt(ckks.encode(params, u[:768], 3), keys, rng_seed=3)
    assert ct_digest(c3) == d["enc_l3"]
    prod = ckks.mult(cu, cv, keys)
    assert ct_digest(prod) == d["mult"]
    assert np.array_equal(ckks.decrypt_vector(prod, keys)[:64], np.array(d["mult_dec"]))
    assert ct_digest(ckks.add(cu, cv)) == d["add"]
    assert ct_digest(ckks.sub(cu, cv)) == d["sub"]
    assert ct_digest(ckks.rescale(ops.mult_plain(cu, 0.5, rescale_after=False))) == d["rescale"]
    assert ct_digest(ckks.mult_plain(cu, v)) == d["mult_plain_vec"]
    assert ct_digest(ckks.add_plain(cu, 0.25)) == d["add_plain_const"]
    assert ct_digest(ckks.mod_down(cu, max(1, L // 2))) == d["mod_down"]
    assert ct_digest(ckks.add(prod, ckks.mod_down(cv, prod.level - 1))) == d["add_aligned"]
    if "rot_3" in d:
        for s in d["rotation_steps"]:
            assert ct_digest(ckks.rotate(cu, s, keys)) == d[f"rot_{s}"]
        assert ct_digest(ckks.rotate(cu, 3, keys)) == d["rot_3"]
        assert np.array_equal(ckks.decrypt_vector(cu, keys)[:64], np.array(d["dec_u"]))
    if "conj_ct" in d:
        assert ct_digest(ckks.conjugate(cu, keys)) == d["conj_ct"]


@pytest.mark.parametrize("name", ["desk", "p14"])
def test_fused_relin_rescale_decrypts_like_reference(name, digests):
    """ops.fused_rescale(): one ModDown from {q_l} + P replaces ModDown then
    rescale (desk: N < 2^12 takes the unfused fallback).  Same level/scale,
    the decryption agrees with the reference-exact product to noise level,
    and batched operands work."""
    d = digests[name]
    params, keys = keyset(name, d)
    rng = np.random.default_rng(9)
    u = rng.uniform(-1, 1, params.slot_count)
    v = rng.uniform(-1, 1, params.slot_count)
    cu = ckks.encrypt_vector(params, u, keys, rng_seed=1)
    cv = ckks.encrypt_vector(params, v, keys, rng_seed=2)
    exact = ckks.mult(cu, cv, keys)
    with ops.fused_rescale():
        fused = ckks.mult(cu, cv, keys)
        sq = ckks.mult(fused, fused, keys)
        batch = ckks.mult(ops.stack([cu, cv]), cv, keys)
    assert (fused.level, fused.scale) == (exact.level, exact.scale)
    de, df = ckks.decrypt_vector(exact, keys), ckks.decrypt_vector(fused, keys)
    assert np.max(np.abs(df - de)) < 1e-6
    assert np.max(np.abs(df - u * v)) < 1e-4
    assert np.max(np.abs(ckks.decrypt_vector(sq, keys) - (u * v) ** 2)) < 1e-4
    b0, b1 = ops.unstack(batch)
    assert np.max(np.abs(ckks.decrypt_vector(b0, keys) - u * v)) < 1e-4
    assert np.max(np.abs(ckks.decrypt_vector(b1, keys) - v * v)) < 1e-4
    assert not ops.fused_rescale_enabled()


def test_rotate_sum_matches_sequential(desk_keys):
    """ops.rotate_sum (one hoisted key switch for several rotations) decrypts
    like the reference's sequential rotate-and-add, batched too."""
    params, keys = desk_keys
    steps = [s for s in (1, 2, 3) if s in keys.rotation_keys]
    if len(steps) < 2:
        keys = ckks.keygen(params, rotation_steps=[1, 2, 3], rng_seed=7)
        steps = [1, 2, 3]
    rng = np.random.default_rng(12)
    v = rng.uniform(-1, 1, params.slot_count)
    ct = ckks.encrypt_vector(params, v, keys, rng_seed=4)
    want = v + sum(np.roll(v, -s) for s in steps)
    got = ops.rotate_sum(ct, steps, keys)
    assert (got.level, got.scale) == (ct.level, ct.scale)
    seq = ct
    for s in steps:
        seq = ckks.add(seq, ckks.rotate(ct, s, keys))
    assert np.max(np.abs(ckks.decrypt_vector(got, keys) - ckks.decrypt_vector(seq, keys))) < 1e-6
    assert np.max(np.abs(ckks.decrypt_vector(got, keys) - want)) < 1e-4
    batch = ops.rotate_sum(ops.stack([ct, ckks.encrypt_vector(params, -v, keys)]), steps, keys)
    assert np.max(np.abs(ckks.decrypt_vector(ops.unstack(batch)[1], keys) + want)) < 1e-4
    assert np.max(np.abs(ckks.decrypt_vector(ops.rotate_sum(ct, [0], keys), keys) - 2 * v)) < 1e-4
    many = list(range(1, 19))  # more than one 16-rotation chunk
    keys18 = ckks.keygen(params, rotation_steps=many, rng_seed=7)
    ct18 = ckks.encrypt_vector(params, v, keys18, rng_seed=4)
    want18 = v + sum(np.roll(v, -s) for s in many)
    got18 = ckks.decrypt_vector(ops.rotate_sum(ct18, many, keys18), keys18)
    assert np.max(np.abs(got18 - want18)) < 1e-3


def test_sigmoid_bsgs_bit_exact(digests, sigmoid15):
    d = digests["desk"]
    params, keys = keyset("desk", d)
    pts = np.linspace(-12, 12, params.slot_count)
    ct = ckks.encrypt_vector(params, pts, keys, rng_seed=9)
    out = ckks.eval_poly_bsgs(ct, sigmoid15, keys)
    assert ct_digest(out) == d["sigmoid_bsgs"]
    assert np.array_equal(ckks.decrypt_vector(out, keys)[:64], np.array(d["sigmoid_dec"]))


def test_batched_key_switch_equals_single(digests):
    """B ciphertext components through one key switch stream the key once and
    give the same limbs as B separate switches."""
    params, keys = keyset("desk", digests["desk"])
    lvl = params.max_level
    polys = [ring.sample_poly(params.ring, "uniform", lvl, np.random.default_rng(50 + i))
             for i in range(4)]
    batch = ring.RnsPoly(params.ring, np.stack([p.limbs for p in polys]), ring.EVAL, lvl)
    kb, ka = K.ks_apply(keys, keys.relin_key, batch)
    for i, p in enumerate(polys):
        sb, sa = K.ks_apply(keys, keys.relin_key, ring.RnsPoly(params.ring, p.limbs, ring.EVAL, lvl))
        assert np.array_equal(kb.limbs[i], sb.limbs)
        assert np.array_equal(ka.limbs[i], sa.limbs)


def test_batched_ciphertext_pipeline(digests):
    """mult / rotate / rescale on a stacked batch equal the per-ciphertext results."""
    params, keys = keyset("desk", digests["desk"])
    rng = np.random.default_rng(77)
    cts = [ckks.encrypt_vector(params, rng.uniform(-1, 1, params.slot_count), keys, rng_seed=i)
           for i in range(3)]
    w = ckks.encrypt_vector(params, rng.uniform(-1, 1, params.slot_count), keys, rng_seed=10)
    batch = ops.stack(cts)
    got = ckks.rotate(ckks.mult(batch, w, keys), 1, keys)
    for i, c in enumerate(cts):
        want = ckks.rotate(ckks.mult(c, w, keys), 1, keys)
        assert np.array_equal(got[i].c0.limbs, want.c0.limbs)
        assert np.array_equal(got[i].c1.limbs, want.c1.limbs)
        assert got.scale == want.scale


# ---- reference tolerance tests (T/test_ckks.py) ----------------------------


@pytest.fixture(scope="module")
def desk_keys(digests):
    return keyset("desk", digests["desk"])


def test_encode_decode(desk_keys):
    params, _ = desk_keys
    rng = np.random.default_rng(12)
    v = rng.uniform(-1, 1, 768)
    pt = ckks.encode(params, v, 3)
    out = ckks.decode_real(pt)
    assert np.max(np.abs(out[:768] - v)) < 1e-4
    assert np.max(np.abs(out[768:])) < 1e-4
    with pytest.raises(CryptoError):
        ckks.encode(params, v[:16], 0, scale=2.0 ** 80)


def test_add_mult_rotate_tolerances(desk_keys):
    params, keys = desk_keys
    rng = np.random.default_rng(12)
    for _ in range(5):
        u = rng.uniform(-1, 1, params.slot_count)
        v = rng.uniform(-1, 1, params.slot_count)
        cu = ckks.encrypt_vector(params, u, keys)
        cv = ckks.encrypt_vector(params, v, keys)
        assert np.max(np.abs(ckks.decrypt_vector(ckks.add(cu, cv), keys) - (u + v))) < 1e-3
        prod = ckks.mult(cu, cv, keys)
        assert np.max(np.abs(ckks.decrypt_vector(prod, keys) - u * v)) < 1e-2
        assert prod.level == cu.level - 1
    u = rng.uniform(-1, 1, params.slot_count)
    ct = ckks.encrypt_vector(params, u, keys)
    back = ckks.rotate(ckks.rotate(ct, 1, keys), -1, keys)
    assert np.max(np.abs(ckks.decrypt_vector(back, keys) - u)) < 1e-3
    five = ckks.decrypt_vector(ckks.rotate(ct, 5, keys), keys)
    assert np.max(np.abs(five - np.roll(u, -5))) < 1e-3
    conj = ckks.decrypt_vector(ckks.conjugate(ct, keys), keys)
    assert np.max(np.abs(conj - u)) < 1e-3


def test_squaring_chain_and_levels(desk_keys):
    params, keys = desk_keys
    ct = ckks.encrypt_vector(params, np.full(params.slot_count, 0.9), keys)
    for _ in range(params.max_level - 1):
        ct = ckks.square(ct, keys)
    want = 0.9 ** (2 ** (params.max_level - 1))
    assert np.max(np.abs(ckks.decrypt_vector(ct, keys) - want)) < 1e-2
    low = ckks.mod_down(ckks.encrypt_vector(params, np.ones(8), keys), 0)
    with pytest.raises(OutOfLevelsError, match="bootstrap"):
        ckks.mult(low, low, keys)
    with pytest.raises(OutOfLevelsError):
        ckks.rescale(low)


def test_scale_mismatch_and_missing_key(desk_keys):
    params, keys = desk_keys
    rng = np.random.default_rng(3)
    v = rng.uniform(-1, 1, 16)
    a = ckks.encrypt(ckks.encode(params, v, 2, scale=2.0 ** 40), keys)
    b = ckks.encrypt(ckks.encode(params, v, 2, scale=2.0 ** 41), keys)
    with pytest.raises(ScaleMismatchError):
        ckks.add(a, b)
    limited = ckks.keygen(params, rotation_steps=[], rng_seed=1, include_conjugation=False)
    ct = ckks.encrypt_vector(params, v, limited)
    with pytest.raises(MissingRotationKeyError):
        ckks.rotate(ct, 3, limited)


def test_poly_eval_depth(desk_keys, sigmoid15):
    params, keys = desk_keys
    pts = np.array([-12.0, -6.0, 0.0, 6.0, 12.0])
    ct = ckks.encrypt_vector(params, pts, keys)
    out = ckks.eval_poly_bsgs(ct, sigmoid15, keys)
    got = ckks.decrypt_vector(out, keys, 5)
    assert np.max(np.abs(got - minimax.eval_cheb(sigmoid15, pts))) < 1e-2
    assert ct.level - out.level == ckks.bsgs_depth(15)
    lin = minimax.remez_fit("linear", (-1, 1), 1)
    v = np.random.default_rng(4).uniform(-1, 1, params.slot_count)
    got = ckks.decrypt_vector(ckks.eval_poly_bsgs(ckks.encrypt_vector(params, v, keys), lin, keys),
                              keys)
    assert np.max(np.abs(got - v)) < 1e-3


def test_serialization_roundtrip(desk_keys):
    params, keys = desk_keys
    ct = ckks.encrypt_vector(params, np.random.default_rng(1).uniform(-1, 1, 32), keys)
    blob = ckks.serialize_ciphertext(ct)
    assert ckks.serialize_ciphertext(ckks.deserialize_ciphertext(blob, params)) == blob
    assert len(blob) == ckks.size_report(params, ct.level)


def test_batched_ciphertext_ingest(desk_keys):
    """deserialize_ciphertexts: several CKT1 buffers -> one batched device
    ciphertext through one pinned H2D copy; each element re-serializes to its
    own bytes, and mismatched buffers are refused like the single path."""
    from paper_2210_02574_b200.errors import SerializationError

    params, keys = desk_keys
    rng = np.random.default_rng(4)
    cts = [ckks.encrypt_vector(params, rng.uniform(-1, 1, 32), keys, level=3, rng_seed=i)
           for i in range(3)]
    blobs = [ckks.serialize_ciphertext(c) for c in cts]
    batch = ckks.deserialize_ciphertexts(blobs, params)
    assert batch.batch == 3 and batch.level == 3
    for i, blob in enumerate(blobs):
        assert ckks.serialize_ciphertext(batch[i]) == blob
    other = ckks.serialize_ciphertext(ckks.encrypt_vector(params, np.zeros(4), keys, level=2))
    with pytest.raises(SerializationError):
        ckks.deserialize_ciphertexts(blobs + [other], params)
    with pytest.raises(SerializationError):
        ckks.deserialize_ciphertexts([blobs[0][:-8]], params)


def test_tma_and_register_inner_products_agree(digests):
    """The TMA-staged key-switch inner product (default) and the
    register-staged one (HEGPU_NO_TMA=1, a separate process: the switch is read
    once) give the same limbs -- both equal the reference's digests."""
    import json
    import os
    import subprocess
    import sys

    code = (
        "import json, numpy as np\n"
        "from oracle.scheme import sha\n"
        "from paper_2210_02574_b200 import ckks, ring\n"
        "from paper_2210_02574_b200.ckks import keys as K\n"
        "from conftest import preset_text\n"
        "p = ckks.CkksParams.from_config_text(preset_text('p16'))\n"
        "keys = ckks.keygen(p, rotation_steps=[1], rng_seed=7, include_conjugation=False)\n"
        "out = {}\n"
        "for lvl in (21, 10):\n"
        "    dp = ring.sample_poly(p.ring, 'uniform', lvl, np.random.default_rng(2000 + lvl))\n"
        "    dp = ring.RnsPoly(p.ring, dp.limbs, ring.EVAL, lvl)\n"
        "    kb, ka = K.ks_apply(keys, keys.relin_key, dp)\n"
        "    out[str(lvl)] = [sha(kb.limbs), sha(ka.limbs)]\n"
        "print(json.dumps(out))\n"
    )
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, HEGPU_NO_TMA="1",
               PYTHONPATH=os.pathsep.join([os.path.dirname(here), here]))
    res = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         timeout=600, cwd=os.path.dirname(here))
    assert res.returncode == 0, res.stderr[-2000:]
    got = json.loads(res.stdout.strip().splitlines()[-1])
    for lvl in ("21", "10"):
        if lvl in digests["p16"]["ks"]:
            assert got[lvl] == digests["p16"]["ks"][lvl]


@pytest.mark.gpu
def test_fused_inverse_ntt_bit_identical():
    """The cluster/DSMEM fused inverse NTT (HEGPU_INTT_FUSED=1, read once per
    process) gives the same limbs as the default two-kernel inverse."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for flag in ("0", "1"):
        env = dict(os.environ, HEGPU_INTT_FUSED=flag, PROBE_POLYS="3", PROBE_LIMBS="22")
        res = subprocess.run([sys.executable, os.path.join(root, "tools", "intt_fused_probe.py")],
                             env=env, capture_output=True, text=True, timeout=600, cwd=root)
        assert res.returncode == 0, res.stderr[-2000:]
        out[flag] = json.loads(res.stdout.strip().splitlines()[-1])["digest"]
    assert out["0"] == out["1"]


def test_wire_formats_match_reference_bytes(desk_keys, digests):
    """CKT1, CKK1 (evaluation and secret roles) and HLR1 blobs written from
    the device tensors are byte-identical to the reference's for the same
    seeds (tests/golden/make_golden.py wire_fixture), and parse straight back
    into device tensors that re-serialize to the same bytes and decrypt."""
    import hashlib

    from paper_2210_02574_b200 import logreg

    params, keys = desk_keys  # keygen(desk, [1, -1, 2, 4], seed 7, conjugation)
    want = digests["wire_desk"]
    rng = np.random.default_rng(5)
    u = rng.uniform(-1, 1, params.slot_count)
    cts = [ckks.encrypt_vector(params, u * (i + 1) / 4, keys, rng_seed=20 + i) for i in range(4)]
    layout = logreg.make_layout(params, 100)
    model = logreg.EncryptedModel(3, layout, cts[:3], [cts[3]] * 3, "secure")
    blobs = {"ckt1": ckks.serialize_ciphertext(cts[0]),
             "ckk1_eval": ckks.serialize_keyset(keys, include_secret=False),
             "ckk1_secret": ckks.serialize_keyset(keys, include_secret=True),
             "hlr1": logreg.serialize_model(model)}
    for name, blob in blobs.items():
        assert len(blob) == want[name]["bytes"], name
        assert hashlib.sha256(blob).hexdigest() == want[name]["sha256"], name
    k2 = ckks.deserialize_keyset(blobs["ckk1_secret"], params)
    assert k2.relin_key.b.is_cuda and k2.public_key[0].data.is_cuda
    assert ckks.serialize_keyset(k2, include_secret=True) == blobs["ckk1_secret"]
    assert ckks.serialize_keyset(ckks.deserialize_keyset(blobs["ckk1_eval"], params)) == \
        blobs["ckk1_eval"]
    m2 = logreg.deserialize_model(blobs["hlr1"], params)
    assert logreg.serialize_model(m2) == blobs["hlr1"]
    got = ckks.decrypt_vector(m2.weights[1], k2)[:64]
    assert np.max(np.abs(got - u[:64] * 2 / 4)) < 1e-3


def test_unseeded_encrypt_uses_device_randomness(desk_keys):
    """Unseeded encryptions (OS entropy in the reference, ops.py:87) expand
    their v, e0, e1 on the device (hegpu_sample_encrypt): ternary on {-1,0,1}
    and rint(N(0, sigma^2)) like ring.py:499-509, fresh per call, and the
    ciphertexts decrypt; seeded encryptions keep the reference's host stream
    (their digests are checked in test_scheme_digests)."""
    from paper_2210_02574_b200.ckks import ops

    params, keys = desk_keys
    big = type("P", (), {"ring_degree": 1 << 20, "error_sigma": params.error_sigma})()
    s = ops.device_samples(big, seed=12345).cpu().numpy()
    v, e = s[0], s[1:].ravel()
    counts = np.bincount(v + 1, minlength=3) / v.size
    assert set(np.unique(v)) <= {-1, 0, 1} and np.all(np.abs(counts - 1 / 3) < 3e-3)
    assert abs(e.mean()) < 0.02 and abs(e.std() - np.sqrt(params.error_sigma ** 2 + 1 / 12)) < 0.02
    assert np.max(np.abs(e)) < 12 * params.error_sigma
    assert np.array_equal(ops.device_samples(big, seed=12345).cpu().numpy(), s)  # counter-based
    rng = np.random.default_rng(3)
    u = rng.uniform(-1, 1, params.slot_count)
    c1 = ckks.encrypt_vector(params, u, keys)
    c2 = ckks.encrypt_vector(params, u, keys)
    assert not np.array_equal(c1.c1.limbs, c2.c1.limbs)
    for c in (c1, c2):
        assert np.max(np.abs(ckks.decrypt_vector(c, keys) - u)) < 1e-4
