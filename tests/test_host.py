"""Host-side logic of the engine (no GPU): presets and params hash, digit
groups, minimax fits vs the reference's coefficients, packing layouts, the
plaintext shadow trainer vs the reference's, sharding arithmetic."""

import numpy as np
import pytest

from conftest import golden_npz, preset_text
from paper_2210_02574_b200 import logreg, minimax, ring, shard
from paper_2210_02574_b200.ckks import params as P
from paper_2210_02574_b200.errors import ApproximationError, CryptoError, DataError


def test_preset_hashes_match_survey():
    assert P.get_preset("p14").params_hash().hex()[:16] == "19ccb5aaa2a93e75"
    assert P.get_preset("p16").params_hash().hex()[:16] == "6d2a5cc54b140f43"
    p16 = P.get_preset("p16")
    assert p16.max_level == 21 and p16.digit_size == 6 and len(p16.ring.special_moduli) == 5
    assert p16.digit_groups(21) == [list(range(0, 6)), list(range(6, 12)), list(range(12, 18)),
                                    list(range(18, 22))]
    assert p16.digit_groups(13)[-1] == [12, 13]


def test_builtin_presets_roundtrip(tmp_path, monkeypatch):
    for name in P.PRESET_NAMES:
        params = P.get_preset(name)
        assert params.slot_count == params.ring_degree // 2
        back = P.CkksParams.from_config_text(params.to_config_text())
        assert back == params and back.params_hash() == params.params_hash()
    desk = P.get_preset("desk")
    custom = desk.to_config_text().replace("security insecure-test-only",
                                           "security custom-flavor")
    (tmp_path / "desk.preset").write_text(custom)
    monkeypatch.setenv("HEBERT_PRESET_DIR", str(tmp_path))
    assert P.get_preset("desk").security_preset_name == "custom-flavor"
    with pytest.raises(CryptoError, match="unknown preset"):
        P.get_preset("made-up")


def test_ring_params_validation():
    with pytest.raises(CryptoError):
        ring.RingParams("bad", 24, (97,))
    with pytest.raises(CryptoError):
        ring.RingParams("bad", 16, (91,))
    with pytest.raises(CryptoError):
        ring.RingParams("bad", 16, (17,))
    with pytest.raises(CryptoError):
        ring.RingParams("bad", 16, (97, 97))
    primes = ring.generate_ntt_primes(40, 4, 1 << 13)
    assert all(q % (1 << 14) == 1 and q.bit_length() == 40 for q in primes)
    p = ring.RingParams("cfg", 32, tuple(ring.generate_ntt_primes(30, 2, 32)),
                        tuple(ring.generate_ntt_primes(31, 1, 32)))
    assert ring.RingParams.from_config_text(p.to_config_text()) == p


def test_host_tables_match_reference_formula():
    g = golden_npz("kernels_n64.npz")
    primes = [int(q) for q in g["q"]]
    p = ring.RingParams("k64", 64, tuple(primes))
    st = p.stacked(tuple(primes))
    assert np.array_equal(st.psi_rev, g["psi_rev"])
    assert np.array_equal(st.ipsi_rev, g["ipsi_rev"])
    assert np.array_equal(st.ninv1, g["ninv"])


def test_sigmoid_fit_matches_reference(digests):
    """The shipped artifact IS the reference's fit (bit for bit); this
    package's own exchange reproduces it to the reference's convergence
    tolerance (tol 1e-11 on the levelled error)."""
    ref = np.array([float.fromhex(c) for c in digests["sigmoid_ref"]])
    shipped = minimax.load_approximant("sigmoid_deg15")
    assert np.array_equal(shipped.cheb_coeffs, ref)
    assert minimax.import_text(minimax.export_text(shipped)).cheb_coeffs.tolist() == ref.tolist()
    poly = minimax.remez_fit("sigmoid", (-12, 12), 15)
    assert np.max(np.abs(poly.cheb_coeffs - ref)) < 1e-7
    assert abs(poly.certified_max_error - 0.00614) <= 0.05 * 0.00614
    assert minimax.equioscillation_check(poly, "sigmoid")


def test_sine_fit_matches_reference(digests):
    ref = np.array([float.fromhex(c) for c in digests["boot_desk64"]["sine_coeffs"]])
    shipped = minimax.evalmod_sine(14, 119)  # what build_context uses (h = 64 -> K = 14)
    assert np.array_equal(shipped.cheb_coeffs, ref)
    assert shipped.domain == (-14.5, 14.5)
    poly = minimax.remez_fit("sine2pi", (-14.5, 14.5), 119)
    assert np.max(np.abs(poly.cheb_coeffs - ref)) < 1e-12
    assert minimax.equioscillation_check(poly, "sine2pi")


def test_minimax_contract():
    assert minimax.remez_fit("linear", (-3, 5), 1).certified_max_error <= 1e-12
    with pytest.raises(ApproximationError):
        minimax.remez_fit("sigmoid", (-1, 1), 0)
    odd = minimax.remez_fit("sine2pi", (-5.5, 5.5), 47)
    assert odd.degree == 47 and minimax.equioscillation_check(odd, "sine2pi")
    a = minimax.remez_fit("sigmoid", (-6, 6), 7)
    b = minimax.remez_fit("sigmoid", (-6, 6), 7)
    assert np.array_equal(a.cheb_coeffs, b.cheb_coeffs)
    xs = np.linspace(-8, 8, 257)
    poly = minimax.remez_fit("sigmoid", (-8, 8), 15)
    mono = minimax.to_monomial(poly)
    assert np.max(np.abs(minimax.eval_cheb(poly, xs) - np.polynomial.polynomial.polyval(xs, mono))) < 1e-10


def test_layout_and_config():
    params = P.get_preset("p16")
    lay = logreg.make_layout(params, 768)
    assert (lay.padded_dim, lay.rows_per_ct, lay.bias_index) == (1024, 32, 768)
    assert logreg.make_layout(params, 1024).rows_per_ct == 16
    with pytest.raises(DataError):
        logreg.PackingLayout(768, 768, 1, 1024)
    with pytest.raises(DataError):
        logreg.TrainConfig(momentum_gamma=1.0)
    slots = logreg._pack_slots(np.ones((2, 768)), lay)
    assert slots[768] == 1.0 and slots[1024 + 768] == 1.0 and slots[769] == 0.0
    assert logreg.iteration_depth(minimax.load_approximant("sigmoid_deg15")) == 8


def test_shadow_trainer_matches_reference(sigmoid15):
    g = golden_npz("logreg_desk.npz")
    layout = logreg.make_layout(P.get_preset("desk"), 16)
    cfg = logreg.TrainConfig(1.0, 0.9, 128, 2)
    sh = logreg.shadow_train(g["X"], g["y"], cfg, sigmoid15, layout=layout)
    assert np.array_equal(sh.weights, g["shadow_weights"])


def test_batches_and_threshold():
    assert list(logreg._batches(5, 32, 150, 64)) == [([0, 1], 64), ([2, 3], 64), ([4], 22)]
    scores = np.array([0.1, 0.4, 0.6, 0.9])
    assert logreg.tune_threshold(scores, np.array([0, 0, 1, 1])) == pytest.approx(0.5)


@pytest.mark.parametrize("n,world", [(16, 1), (16, 2), (16, 8), (3, 8), (17, 4)])
def test_shard_ranges_partition(n, world):
    seen = []
    for r in range(world):
        lo, hi = shard.shard_range(n, r, world)
        seen.extend(range(lo, hi))
    assert seen == list(range(n))
    sizes = [shard.shard_range(n, r, world)[1] - shard.shard_range(n, r, world)[0]
             for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def test_wrapping_allreduce_contract():
    """NCCL int64 SUM wraps mod 2^64; one mod-q pass gives the modular sum."""
    primes = P.get_preset("p16").ring.moduli_chain[:3] + (2 ** 61 - 1,)
    assert shard.check_allreduce_exact(primes, 8)
    rng = np.random.default_rng(0)
    ranks = [np.stack([rng.integers(0, q, 64, dtype=np.uint64) for q in primes])
             for _ in range(8)]
    got = shard.modular_sum_host(ranks, primes)
    want = np.stack([sum(r[i].astype(object) for r in ranks) % q for i, q in enumerate(primes)])
    assert got.astype(object).tolist() == want.tolist()
    assert shard.refresh_owner(0, 1) == 0 and shard.refresh_owner(1, 2) == 1


def test_periodic_diagonal_run_compression():
    """Slot vectors periodic with period P encode to polynomials in X^(N/2P)
    (the small-ring embedding the diagonal cache uses), whose evaluation
    vectors are constant on runs of N/2P coefficients in the reference's
    bit-reversed NTT order -- the layout hegpu_bsgs reads (pt_log_run)."""
    from oracle import scheme as S
    from paper_2210_02574_b200 import bootstrap as bs

    p = S.Params.from_text(preset_text("p14"))
    n = p.n
    rng = np.random.default_rng(4)
    for period in (n // 8, n // 32):
        r = n // (2 * period)
        v = rng.uniform(-1, 1, period) + 1j * rng.uniform(-1, 1, period)
        dense = bs._coeffs_from_rows(n, np.tile(v, (n // 2) // period)[None], 2.0 ** 20)
        emb = np.zeros((1, n))
        emb[:, ::r] = bs._coeffs_from_rows(2 * period, v[None], 2.0 ** 20)
        assert np.max(np.abs(dense - emb)) <= 1
        assert not np.any(np.delete(dense, np.s_[::r], axis=1))
        primes = list(p.chain[:2])
        ev = S.ntt_fwd(p, S.from_signed(emb[0].astype(np.int64), primes), primes)
        runs = ev.reshape(len(primes), n // r, r)
        assert (runs == runs[..., :1]).all()
        assert bs._run_log(type("P", (), {"ring_degree": n})(), period) == min(r.bit_length() - 1, 5)


def test_pcg64_advance_matches_numpy():
    """ring.pcg64_advance_state (the host half of hegpu_pcg64_uniform) is
    numpy's PCG64 jump: the generator state after d draws."""
    import numpy as np

    from paper_2210_02574_b200 import ring as rg

    for seed, d in ((7, 1), (11, 1_769_473), (3, 12345678901)):
        g = np.random.default_rng(seed)
        st = g.bit_generator.state["state"]
        want = np.random.default_rng(seed)
        want.bit_generator.advance(d)
        assert rg.pcg64_advance_state(st["state"], st["inc"], d) == \
            want.bit_generator.state["state"]["state"]
    # one bounded uint64 draw = one 64-bit output: the stream position the
    # device fill reports for k*n draws without rejections
    g = np.random.default_rng(5)
    st = g.bit_generator.state["state"]
    g.integers(0, 0xffffe80001, size=1000, dtype=np.uint64)
    assert rg.pcg64_advance_state(st["state"], st["inc"], 1000) == \
        g.bit_generator.state["state"]["state"]


def test_pair_packing_stops_at_period_1024():
    """refresh_many packs w and u into one bootstrap of twice the period only
    up to n = 1024 slots (cfg4); at n = 2048 (cfg5 OvR) the packed transforms
    cost more than a batch of two (bootstrap.PACKED_PAIR_MAX_SLOTS)."""
    from types import SimpleNamespace

    from paper_2210_02574_b200 import bootstrap as bs

    params = SimpleNamespace(slot_count=32768)
    def ctx(n, **kw):
        return SimpleNamespace(params=params, n_slots=n, is_full=kw.get("full", False),
                               input_periodic=kw.get("periodic", True))
    assert bs._pair_packable_ctx(ctx(64)) and bs._pair_packable_ctx(ctx(1024))
    assert not bs._pair_packable_ctx(ctx(2048))
    assert not bs._pair_packable_ctx(ctx(1024, periodic=False))


def test_double_angle_evalmod_fit():
    """The double-angle EvalMod base (bootstrap._cos_quarter_target): a
    degree-31 minimax fit of cos(2 pi (x - 1/4) / 2^r) on +-(K + 1/2), whose r
    doublings reproduce sin(2 pi x) -- the function the reference's degree-119
    sine approximates -- to better than its fit."""
    from paper_2210_02574_b200 import bootstrap as bs

    for K, r in ((14, 3), (25, 4)):
        D = K + 0.5
        poly = minimax.remez_fit(bs._cos_quarter_target(D, r), (-D, D), 31)
        x = np.linspace(-D, D, 20001)
        c = minimax.eval_cheb(poly, x)
        for _ in range(r):
            c = 2 * c * c - 1
        err = np.max(np.abs(c / (2 * np.pi) - np.sin(2 * np.pi * x) / (2 * np.pi)))
        assert poly.certified_max_error < 1e-10
        assert err < 1e-9


def test_evalmod_context_levels():
    """Level budgets: the reference sine (K = 14) costs 10 levels, the double
    angle 11 (P16); p16s (h = 192 -> K = 25) picks the double angle with r = 4
    and keeps output level 9 (the trainer's 8 + the packed refresh's mask)."""
    from paper_2210_02574_b200 import bootstrap as bs

    p16 = P.get_preset("p16")
    assert bs.build_context(p16, 1024, input_periodic=True).output_level == 11
    da = bs.build_context(p16, 1024, input_periodic=True, evalmod="double_angle")
    assert (da.double_angle, da.output_level) == (3, 10)
    secure = bs.build_context(P.get_preset("p16s"), 1024, input_periodic=True)
    assert (secure.range_k, secure.double_angle, secure.output_level) == (25, 4, 9)
