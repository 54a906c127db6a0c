"""GPU parity: the kernel table and ring layer vs the reference's golden
vectors (bit-exact) and the reference ring tests (T/test_ring.py)."""

import numpy as np
import pytest

from conftest import golden_npz, preset_text

pytestmark = pytest.mark.gpu

from paper_2210_02574_b200 import _kernels, ring  # noqa: E402
from paper_2210_02574_b200.errors import CryptoError, FormMismatchError, LevelMismatchError  # noqa: E402


def test_kernel_table_bit_exact():
    g = golden_npz("kernels_n64.npz")
    q, qinv, r2 = g["q"], g["qinv"], g["r2"]
    a, b = g["a"], g["b"]
    assert np.array_equal(_kernels.elementwise_mulmod(a, b, q, qinv, r2), g["mulmod"])
    assert np.array_equal(_kernels.elementwise_mont(a, b, q, qinv), g["mont"])
    assert np.array_equal(_kernels.rowwise_mont(a, g["c"], q, qinv), g["rowwise"])
    assert np.array_equal(_kernels.addmod_rows(a, b, q), g["add"])
    assert np.array_equal(_kernels.submod_rows(a, b, q), g["sub"])
    assert np.array_equal(_kernels.base_convert(g["hat"], g["punc"], q, qinv), g["bconv"])
    acc = a.copy()
    assert np.array_equal(_kernels.fma_inplace(acc, b, a, q, qinv, r2), g["fma"])
    acc = b.copy()
    out = _kernels.fma_gather_inplace(acc, a, g["key"], g["rows"], q, qinv, r2)
    assert out is acc and np.array_equal(out, g["fma_gather"])
    f = a.copy()
    assert np.array_equal(_kernels.ntt_forward_inplace(f, g["psi_rev"], q, qinv), g["ntt_fwd"])
    assert np.array_equal(f, g["ntt_fwd"])  # in place
    f = a.copy()
    assert np.array_equal(_kernels.ntt_inverse_inplace(f, g["ipsi_rev"], g["ninv"], q, qinv),
                          g["ntt_inv"])


def test_ring_ops_bit_exact():
    g = golden_npz("ring_n64.npz")
    primes = tuple(int(x) for x in g["primes"])
    p = ring.RingParams("r64", 64, primes)
    x = ring.RnsPoly(p, g["x"], ring.COEFF, 2)
    y = ring.RnsPoly(p, g["y"], ring.COEFF, 2)
    xe, ye = ring.to_eval(x), ring.to_eval(y)
    assert np.array_equal(xe.limbs, g["x_eval"])
    assert np.array_equal(ring.poly_mul(xe, ye).limbs, g["prod"])
    assert np.array_equal(ring.to_coeff(ring.poly_mul(xe, ye)).limbs, g["prod_coeff"])
    for gg in (3, 5, 127):
        assert np.array_equal(ring.poly_automorphism_eval(xe, gg).limbs, g[f"auto_eval_{gg}"])
        assert np.array_equal(ring.poly_automorphism(x, gg).limbs, g[f"auto_coeff_{gg}"])
    assert np.array_equal(ring.poly_from_signed(p, g["signed"], 2).limbs, g["lifted"])
    assert np.array_equal(ring._eval_exponent_map(p)[0], g["exps"])


@pytest.mark.parametrize("name", ["p14", "p16"])
def test_full_chain_ntt_digest(name, digests):
    from oracle.scheme import sha
    from paper_2210_02574_b200.ckks import CkksParams

    params = CkksParams.from_config_text(preset_text(name))
    L = params.max_level
    up = ring.sample_poly(params.ring, "uniform", L, np.random.default_rng(1000))
    assert sha(ring.to_eval(up).limbs) == digests[name]["ntt_fwd"]
    inv = ring.ntt_transform(ring.RnsPoly(params.ring, up.limbs, ring.EVAL, L), "inverse")
    assert sha(inv.limbs) == digests[name]["ntt_inv"]


@pytest.mark.parametrize("n", [16, 1024, 1 << 13, 1 << 15, 1 << 17])
def test_ntt_roundtrip_and_oracle(n):
    """Every supported size vs the oracle (reference T/test_ring.py:29-42)."""
    from oracle import scheme as S

    # 60-bit: integer Shoup path; 40- and 46-bit (just below 2^46, the widest
    # lazy ranges): FP64 path (common.cuh kFpMaxBits)
    primes = tuple(ring.generate_ntt_primes(60, 1, n) + ring.generate_ntt_primes(40, 2, n)
                   + ring.generate_ntt_primes(46, 1, n))
    p = ring.RingParams("rt", n, primes)
    a = ring.sample_poly(p, "uniform", 3, np.random.default_rng(1))
    fwd = ring.ntt_transform(a, "forward")
    op = S.Params(n, primes, (), 2.0 ** 40, 1, None, 3.2)
    assert np.array_equal(fwd.limbs, S.ntt_fwd(op, a.limbs, primes))
    back = ring.ntt_transform(fwd, "inverse")
    assert np.array_equal(a.limbs, back.limbs)
    # extreme residues (every coefficient q - 1, then alternating 0 / q - 1)
    qv = np.array(primes, dtype=np.uint64)[:, None]
    for lim in (np.broadcast_to(qv - np.uint64(1), (len(primes), n)),
                (qv - np.uint64(1)) * (np.arange(n, dtype=np.uint64) % np.uint64(2))):
        x = ring.RnsPoly(p, np.ascontiguousarray(lim, dtype=np.uint64), ring.COEFF, 3)
        fx = ring.ntt_transform(x, "forward")
        assert np.array_equal(fx.limbs, S.ntt_fwd(op, x.limbs, primes))
        assert np.array_equal(ring.ntt_transform(fx, "inverse").limbs, x.limbs)


def test_constant_and_wraparound():
    p = ring.RingParams("t16", 16, (97,))
    c = ring.poly_from_signed(p, [5] + [0] * 15, 0)
    assert set(ring.to_eval(c).limbs[0].tolist()) == {5}
    half = ring.to_eval(ring.poly_from_signed(p, [0] * 8 + [1] + [0] * 7, 0))
    assert ring.to_coeff(ring.poly_mul(half, half)).limbs[0].tolist() == [96] + [0] * 15
    z = ring.zero_poly(p, 0, form=ring.COEFF)
    assert not ring.ntt_transform(z, "forward").limbs.any()


def test_errors():
    p = ring.RingParams("lm", 16, tuple(ring.generate_ntt_primes(30, 2, 16)))
    rng = np.random.default_rng(4)
    a = ring.to_eval(ring.sample_poly(p, "uniform", 1, rng))
    b = ring.to_eval(ring.sample_poly(p, "uniform", 0, rng))
    with pytest.raises(LevelMismatchError):
        ring.poly_mul(a, b)
    with pytest.raises(FormMismatchError):
        ring.ntt_transform(a, "forward")
    with pytest.raises(CryptoError):
        ring.sample_poly(p, "discrete_gaussian", 0, rng, sigma=0)


def test_sampling_statistics():
    p = ring.RingParams("s13", 1 << 13, tuple(ring.generate_ntt_primes(40, 1, 1 << 13)))
    s = ring.sample_poly(p, "ternary", 0, np.random.default_rng(6))
    q = p.moduli_chain[0]
    vals = s.limbs[0]
    assert set(np.unique(vals)) <= {0, 1, q - 1}
    g = ring.sample_poly(p, "discrete_gaussian", 0, np.random.default_rng(7), sigma=3.2)
    v = g.limbs[0].astype(np.int64)
    v = np.where(v > q // 2, v - q, v)
    assert abs(v.std() - 3.2) < 0.32
    h = ring.sample_poly(p, "ternary", 0, np.random.default_rng(8), hamming_weight=64)
    assert int(np.sum(h.limbs[0] != 0)) == 64


def test_batched_ops_equal_single():
    """A (B, k, N) batch through one launch equals B separate calls."""
    primes = tuple(ring.generate_ntt_primes(40, 3, 1024))
    p = ring.RingParams("cc", 1024, primes)
    rng = np.random.default_rng(13)
    polys = [ring.to_eval(ring.sample_poly(p, "uniform", 2, rng)) for _ in range(5)]
    batch = ring.RnsPoly(p, np.stack([x.limbs for x in polys]), ring.EVAL, 2)
    other = polys[0]
    prod = ring.poly_mul(batch, other)
    coeff = ring.to_coeff(batch)
    for i, x in enumerate(polys):
        assert np.array_equal(prod.limbs[i], ring.poly_mul(x, other).limbs)
        assert np.array_equal(coeff.limbs[i], ring.to_coeff(x).limbs)


@pytest.mark.parametrize("lr,ns,T,G", [(2, 0, 21, 5), (3, 0, 100, 5), (4, 0, 21, 5), (5, 0, 21, 5),
                                        (4, 2, 21, 5), (3, 2, 256, 37), (5, 1, 33, 17)])
def test_bsgs_run_compressed_matches_dense_and_exact(lr, ns, T, G):
    """hegpu_bsgs on run-compressed diagonals (pt_log_run, the sparse-bootstrap
    cache layout; lr >= 3 takes the tensor-core byte-plane GEMM) equals the dense
    kernel on the expanded diagonals and the exact sum mod q -- including 256
    terms on 60-bit special primes (the largest exact sum, < 2^128) and giant
    counts that are not multiples of the 16-giant tile."""
    import ctypes

    import torch

    from paper_2210_02574_b200 import _dev, _lib, ckks

    params = ckks.get_preset("desk")
    n, k, nb = params.ring_degree, 3 + ns, 2
    # ns > 0: the last ns limbs are special primes (extended-basis babies)
    qs = ([int(q) for q in params.ring.moduli_chain[:k - ns]]
          + [int(q) for q in params.ring.special_moduli[:ns]])
    rng = np.random.default_rng(lr)

    def rand(shape):
        return np.stack([rng.integers(0, q, shape[:-2] + (shape[-1],), dtype=np.uint64)
                         for q in qs], axis=-2)

    babies = _dev.to_device(rand((T, nb, 2, k, n)).view(np.int64))
    pts_c = rand((9, k, n >> lr))
    idx = rng.integers(-1, 9, (G, T)).astype(np.int32)
    idx_d = torch.from_numpy(idx).to(_dev.device())
    ptrs = (ctypes.c_void_p * T)(*[babies[t].data_ptr() for t in range(T)])
    outs = []
    for run_log, pts in ((lr, pts_c), (0, np.repeat(pts_c, 1 << lr, axis=-1))):
        pd = _dev.to_device(np.ascontiguousarray(pts).view(np.int64))
        out = _dev.empty(G, nb, 2, k, n)
        _lib.call("hegpu_bsgs", params.ring.device(), ptrs, T, k * n, 2 * k * n, nb,
                  pd.data_ptr(), k * (n >> run_log), run_log, idx_d.data_ptr(), G,
                  out.data_ptr(), nb * 2 * k * n, k, ns, _dev.stream())
        outs.append(out.cpu().numpy().view(np.uint64))
    assert np.array_equal(outs[0], outs[1])
    bab = babies.cpu().numpy().view(np.uint64)
    for (g, b, c, l, x) in [(0, 0, 0, 0, 0), (4, 1, 1, 2, n - 1), (2, 1, 0, 1, 37),
                            (G - 1, 1, 1, k - 1, n - 2)]:
        want = sum(int(pts_c[idx[g, t], l, x >> lr]) * int(bab[t, b, c, l, x])
                   for t in range(T) if idx[g, t] >= 0) % qs[l]
        assert int(outs[0][g, b, c, l, x]) == want


def test_pcg64_uniform_device_matches_numpy():
    """hegpu_pcg64_uniform reproduces numpy's Generator(PCG64).integers(0, q,
    dtype=uint64) stream (keygen's uniform `a` draws) and leaves the generator
    where numpy would: bit-exact on P16's 27 primes, and with bounds whose
    Lemire rejection rate is ~1/4 (many rejected draws re-mapped)."""
    from paper_2210_02574_b200 import _dev, ckks, ring as rg

    params = ckks.get_preset("p16")
    primes = list(params.ring.moduli_chain) + list(params.ring.special_moduli)
    n = params.ring_degree
    for bounds, m in ((primes, n), ([(1 << 62) + 1, (1 << 62) + 3, (1 << 63) - 25], 48)):
        dev_rng, host_rng = np.random.default_rng(2024), np.random.default_rng(2024)
        dev_rng.integers(-1, 2, size=17)  # leave a buffered uint32 behind, as keygen does
        host_rng.integers(-1, 2, size=17)
        out = _dev.empty(len(bounds), m)
        rg.sample_uniform_dev(dev_rng, bounds, m, out)
        want = np.stack([host_rng.integers(0, q, size=m, dtype=np.uint64) for q in bounds])
        assert np.array_equal(out.cpu().numpy().view(np.uint64), want)
        assert dev_rng.bit_generator.state == host_rng.bit_generator.state
        assert np.array_equal(dev_rng.normal(size=5), host_rng.normal(size=5))
        assert np.array_equal(dev_rng.integers(-1, 2, size=9), host_rng.integers(-1, 2, size=9))


def test_row_grid_overhang_guard():
    """n_polys * k just above 65535 rows (grid.z = 2 with a partial last slice):
    every row is computed and nothing past the output is written."""
    import torch

    g = golden_npz("ring_n64.npz")
    primes = tuple(int(x) for x in g["primes"])
    p = ring.RingParams("r64", 64, primes)
    k, n = 3, 64
    cnt = 65535 // k + 2  # 21847 polys -> 65541 rows
    rng = np.random.default_rng(9)
    q = np.array(primes, dtype=np.uint64)[None, :, None]
    a_h = (rng.integers(0, 1 << 62, (cnt, k, n), dtype=np.uint64) % q)
    b_h = (rng.integers(0, 1 << 62, (cnt, k, n), dtype=np.uint64) % q)
    a = ring.RnsPoly(p, a_h, ring.EVAL, 2)
    b = ring.RnsPoly(p, b_h, ring.EVAL, 2)
    # output with a sentinel tail: the guard must keep the overhanging slice out
    big = torch.full((cnt + 1, k, n), -1, dtype=torch.int64, device=a.data.device)
    out = big[:cnt]
    ring._binary(ring._lib.OP_ADD, a, b, out=out)
    got = out.cpu().numpy().view(np.uint64)
    want = (a_h + b_h) % q
    assert np.array_equal(got, want)
    assert bool((big[cnt] == -1).all())
    s = ring.poly_automorphism_eval(a, 5)
    assert np.array_equal(s.limbs[-1], ring.poly_automorphism_eval(
        ring.RnsPoly(p, a_h[-1], ring.EVAL, 2), 5).limbs)
