"""GPU bootstrapping vs the reference (tolerance; T/test_bootstrap.py) and
ModRaise / seeded input limbs (bit-exact vs reference digests)."""

import numpy as np
import pytest

from conftest import golden_npz

pytestmark = pytest.mark.gpu

from oracle.scheme import sha  # noqa: E402
from paper_2210_02574_b200 import bootstrap as bs, ckks  # noqa: E402
from paper_2210_02574_b200.errors import InsecureDebugError  # noqa: E402


def ct_digest(ct):
    return {"c0": sha(ct.c0.limbs), "c1": sha(ct.c1.limbs), "level": ct.level,
            "scale": float(ct.scale).hex()}


@pytest.fixture(scope="module")
def boot(digests):
    params = ckks.get_preset("desk-boot")
    ctx = bs.build_context(params, n_slots=64)
    d = digests["boot_desk64"]
    assert ctx.required_rotation_steps() == [s for s in d["steps"] if s in set(
        ctx.required_rotation_steps())]
    keys = ckks.keygen(params, rotation_steps=d["steps"], rng_seed=11)
    return params, ctx, keys, d


def test_sine_fit_matches_reference(boot):
    params, ctx, keys, d = boot
    ref = np.array([float.fromhex(c) for c in d["sine_coeffs"]])
    assert np.max(np.abs(ctx.evalmod_poly.cheb_coeffs - ref)) < 1e-12


def test_mod_raise_bit_exact(boot):
    params, ctx, keys, d = boot
    v = golden_npz("boot_desk64.npz")["v"]
    ct = ckks.encrypt_vector(params, v, keys, level=0, rng_seed=21)
    assert ct_digest(ct) == d["enc"]
    assert ct_digest(bs._mod_raise(ct)) == d["mod_raise"]


def test_bootstrap_matches_reference(boot):
    params, ctx, keys, d = boot
    g = golden_npz("boot_desk64.npz")
    v = g["v"]
    ct = ckks.encrypt_vector(params, v, keys, level=0, rng_seed=21)
    out = bs.bootstrap(ct, ctx, keys)
    assert out.level == ctx.output_level == d["out_level"]
    assert out.scale == params.default_scale
    dec = ckks.decrypt_vector(out, keys)
    err = np.max(np.abs(dec[:64] - v))
    assert err < 1e-2  # reference tolerance (T/test_bootstrap.py:23)
    assert np.max(np.abs(dec[64:])) < 1e-2  # padding restored
    # same quality as the reference implementation on the same ciphertext
    assert err <= max(2 * d["err"], 5e-3)
    assert np.max(np.abs(dec - g["dec"])) < 1e-2


def test_bootstrap_random_and_compose(boot):
    params, ctx, keys, _ = boot
    rng = np.random.default_rng(31)
    for _ in range(2):
        v = rng.uniform(-1, 1, 64)
        ct = ckks.encrypt_vector(params, v, keys, level=0)
        out = bs.bootstrap(ct, ctx, keys)
        assert np.max(np.abs(ckks.decrypt_vector(out, keys)[:64] - v)) < 1e-2
    v = rng.uniform(-1, 1, 64)
    ct = ckks.encrypt_vector(params, v, keys, level=0)
    twice = bs.bootstrap(bs.bootstrap(ct, ctx, keys), ctx, keys)
    assert np.max(np.abs(ckks.decrypt_vector(twice, keys)[:64] - v)) < 2e-2
    hi = ckks.encrypt_vector(params, np.linspace(-1, 1, 64), keys, level=4)
    out = bs.bootstrap(hi, ctx, keys)
    assert np.max(np.abs(ckks.decrypt_vector(out, keys)[:64] - np.linspace(-1, 1, 64))) < 1e-2


def test_bootstrap_off_default_scale(boot):
    """Input scale != default (the w/u refresh case): the scale-independent
    diagonals plus the mask correction keep the message."""
    params, ctx, keys, _ = boot
    v = np.random.default_rng(5).uniform(-1, 1, 64)
    ct = ckks.encrypt(ckks.encode(params, v, 0, scale=params.default_scale * 1.03), keys)
    out = bs.bootstrap(ct, ctx, keys)
    assert np.max(np.abs(ckks.decrypt_vector(out, keys)[:64] - v)) < 1e-2
    assert out.scale == params.default_scale


def test_context_invariants(boot):
    params, ctx, _, _ = boot
    assert ctx.consumed_levels + ctx.output_level == params.max_level
    assert ctx.evalmod_poly.degree >= 2 * ctx.range_k
    with pytest.raises(Exception, match="sparse"):
        bs.build_context(ckks.get_preset("desk"), n_slots=64)


def test_debug_refresh_flags():
    params = ckks.get_preset("desk")
    keys = ckks.keygen(params, rotation_steps=[1], rng_seed=7)
    v = np.random.default_rng(33).uniform(-1, 1, params.slot_count)
    ct = ckks.mod_down(ckks.encrypt_vector(params, v, keys), 1)
    out = bs.debug_refresh(ct, keys, enabled=True)
    assert out.level == params.max_level and out.insecure_provenance
    assert np.max(np.abs(ckks.decrypt_vector(out, keys) - v)) < 1e-4
    assert ckks.rotate(out, 1, keys).insecure_provenance
    with pytest.raises(InsecureDebugError):
        bs.debug_refresh(ct, keys, enabled=1)
    with pytest.raises(InsecureDebugError):
        bs.debug_refresh(ct, keys.public_only(), enabled=True)
    with pytest.raises(InsecureDebugError):
        bs.DebugRefresher(keys)


def test_hoisted_rotations_decrypt_like_rotate(boot):
    """Hoisted baby-step rotations (one shared ModUp) decrypt to the same
    slots as the reference's per-rotation key switch."""
    from paper_2210_02574_b200.ckks import ops

    params, ctx, keys, _ = boot
    v = np.random.default_rng(8).uniform(-1, 1, params.slot_count)
    ct = ckks.encrypt_vector(params, v, keys, rng_seed=3)
    steps = [0, 1, 2, 3, 5]
    hoisted = ops.rotate_hoisted(ct, steps, keys)
    for s, h in zip(steps, hoisted):
        want = ckks.decrypt_vector(ckks.rotate(ct, s, keys), keys)
        got = ckks.decrypt_vector(h, keys)
        assert np.max(np.abs(got - want)) < 1e-6
        assert np.max(np.abs(got - np.roll(v, -s))) < 1e-3
    batch = ops.stack([ct, ckks.encrypt_vector(params, -v, keys, rng_seed=4)])
    hb = ops.rotate_hoisted(batch, [1, 2], keys)
    assert np.max(np.abs(ckks.decrypt_vector(hb[1][1], keys) - np.roll(-v, -2))) < 1e-3


def test_packed_pair_refresh(boot):
    """Two periodic ciphertexts refreshed by ONE bootstrap of twice the period
    (BootstrapRefresher.refresh_many): each output decrypts like its own
    bootstrap, at the same level and the default scale."""
    params, ctx0, _, _ = boot
    ctx = bs.build_context(params, n_slots=64, input_periodic=True)
    keys = ckks.keygen(params, rotation_steps=bs.refresh_rotation_steps(ctx), rng_seed=11)
    rng = np.random.default_rng(17)
    va, vb = rng.uniform(-1, 1, 64), rng.uniform(-1, 1, 64)
    reps = params.slot_count // 64
    a = ckks.encrypt(ckks.encode(params, np.tile(va, reps), 2, scale=params.default_scale * 1.02),
                     keys)
    b = ckks.encrypt(ckks.encode(params, np.tile(vb, reps), 2), keys)
    ref = bs.BootstrapRefresher(ctx, keys)
    assert bs._pair_packable([a, b], ctx, keys)
    ra, rb = ref.refresh_many([a, b])
    for r, v in ((ra, va), (rb, vb)):
        assert r.level == ctx.output_level and r.scale == params.default_scale
        assert np.max(np.abs(ckks.decrypt_vector(r, keys) - np.tile(v, reps))) < 1e-2


def test_captured_bootstrap_replays(boot):
    """CapturedBootstrap (CUDA graph of one bootstrap) gives the same output
    as the eager call on the same input and accepts new inputs of the same
    shape (ciphertext or packed host tensor)."""
    params, ctx, keys, _ = boot
    rng = np.random.default_rng(23)
    v1, v2 = rng.uniform(-1, 1, 64), rng.uniform(-1, 1, 64)
    c1 = ckks.encrypt_vector(params, v1, keys, level=0, rng_seed=31)
    c2 = ckks.encrypt_vector(params, v2, keys, level=0, rng_seed=32)
    cap = bs.CapturedBootstrap(c1, ctx, keys)
    out = cap.run(c1)
    eager = bs.bootstrap(c1, ctx, keys)
    assert np.array_equal(out.c0.limbs, eager.c0.limbs)
    assert np.array_equal(out.c1.limbs, eager.c1.limbs)
    import torch

    host = torch.stack([c2.c0.data, c2.c1.data]).cpu()
    out2 = cap.run(host.to("cuda"))
    assert np.max(np.abs(ckks.decrypt_vector(out2, keys)[:64] - v2)) < 1e-2


# ---------------------------------------------------------------------------
# full-slot contexts: diagonals generated + encoded on the device
# ---------------------------------------------------------------------------


def test_gpu_diag_encode_matches_host_encode():
    """hegpu_encode_diags reproduces the host encode (numpy FFT + rint,
    encoding.py:62-97) of the closed-form diagonals (bootstrap.py:174-197),
    rolled and conjugated as in the BSGS loop (bootstrap.py:219-236), up to
    float rounding of the last bits."""
    import ctypes

    import torch

    from paper_2210_02574_b200 import _dev, _lib

    params = ckks.get_preset("desk-boot")
    ctx = bs.build_context(params, n_slots=params.slot_count)
    n, s = params.ring_degree, params.slot_count
    s_in = params.default_scale
    cases = [(bs.DIAG_KIND_CTS, 0, 0, 0, 0), (bs.DIAG_KIND_CTS, 1, 65, 64, 1),
             (bs.DIAG_KIND_CTS, 0, s - 1, s - 64, 1), (bs.DIAG_KIND_STC, 0, 3, 0, 0),
             (bs.DIAG_KIND_STC, 1, 130, 128, 0)]
    for kind, half, d, g0, conj in cases:
        if kind == bs.DIAG_KIND_CTS:
            vals, fold, scale = bs._cts_diag_full(ctx, d, half, s_in), bs._cts_fold(ctx, s_in), \
                float(params.ring.moduli_chain[params.max_level])
        else:
            vals, fold, scale = bs._stc_diag_full(ctx, d, half, s_in), \
                params.ring.moduli_chain[0] / s_in, params.default_scale
        if conj:
            vals = np.conj(vals)
        want = bs._coeffs_from_rows(n, np.roll(vals, g0)[None, :], scale)[0]
        coeffs = _dev.empty(1, n)
        scratch = torch.empty((1, n, 2), dtype=torch.float64, device="cuda")
        dd, gg, cc = (np.array([x], dtype=t) for x, t in ((d, np.int32), (g0, np.int32),
                                                           (conj, np.uint8)))
        _lib.call("hegpu_encode_diags", params.ring.device(), kind, half, ctypes.c_double(fold),
                  ctypes.c_double(scale), 1, dd.ctypes.data, gg.ctypes.data, cc.ctypes.data,
                  scratch.data_ptr(), coeffs.data_ptr(), _dev.stream())
        got = coeffs.cpu().numpy()[0].astype(np.float64)
        tol = max(2.0, 1e-12 * np.max(np.abs(want)))
        assert np.max(np.abs(got - want)) <= tol, (kind, half, d, g0, conj)


@pytest.fixture(scope="module")
def boot_full(digests):
    params = ckks.get_preset("desk-boot")
    ctx = bs.build_context(params, n_slots=params.slot_count)
    d = digests["boot_desk_full"]
    assert sorted(set(ctx.required_rotation_steps())) == d["steps"]
    keys = ckks.keygen(params, rotation_steps=d["steps"], rng_seed=11)
    return params, ctx, keys, d


def test_full_slot_bootstrap_matches_reference(boot_full):
    """Full-slot bootstrap (4,096 slots, bootstrap.py:319-335) with the
    device-generated diagonals: reference tolerance, same quality as the
    reference's own run on the same seeded ciphertext (golden fixture)."""
    params, ctx, keys, d = boot_full
    g = golden_npz("boot_desk_full.npz")
    v = g["v"]
    ct = ckks.encrypt_vector(params, v, keys, level=0, rng_seed=22)
    assert ct_digest(ct) == d["enc"]
    out = bs.bootstrap(ct, ctx, keys)
    assert out.level == ctx.output_level == d["out_level"]
    assert out.scale == params.default_scale
    dec = ckks.decrypt_vector(out, keys)
    err = np.max(np.abs(dec - v))
    assert err < 1e-2  # T/test_bootstrap.py:23
    assert err <= max(2 * d["err"], 5e-3)
    assert np.max(np.abs(dec - g["dec"])) < 1e-2


def test_full_slot_bootstrap_batched(boot_full):
    """Two ciphertexts refreshed by one batched full-slot bootstrap (the
    ingest path): every diagonal is generated once for the batch."""
    params, ctx, keys, _ = boot_full
    rng = np.random.default_rng(41)
    vs = [rng.uniform(-1, 1, params.slot_count) for _ in range(2)]
    cts = [ckks.encrypt_vector(params, v, keys, level=0) for v in vs]
    outs = bs.bootstrap_many(cts, ctx, keys)
    for o, v in zip(outs, vs):
        assert np.max(np.abs(ckks.decrypt_vector(o, keys) - v)) < 1e-2


def test_segmented_capture_replays_bootstrap(boot):
    """bootstrap.SegmentedCapture (the capture the sharded trainer uses around
    its split refresh) replays a bootstrap with the eager result's limbs."""
    import torch

    params, ctx, keys, _ = boot
    v = np.random.default_rng(41).uniform(-1, 1, 64)
    ct = ckks.encrypt_vector(params, v, keys, level=0, rng_seed=42)
    want = bs.bootstrap(ct, ctx, keys)
    inp = ct.copy()
    seg = bs.SegmentedCapture()
    out = seg.capture(lambda: bs.bootstrap(inp, ctx, keys))
    assert len(seg.graphs) == 1 and not seg.points  # one process: no collective cut
    inp.c0.data.copy_(ct.c0.data)
    inp.c1.data.copy_(ct.c1.data)
    seg.replay()
    torch.cuda.synchronize()
    assert np.array_equal(out.c0.limbs, want.c0.limbs)
    assert np.array_equal(out.c1.limbs, want.c1.limbs)
