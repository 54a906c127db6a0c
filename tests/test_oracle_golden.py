"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import golden_npz, preset_text
from oracle import kernels as OK
from oracle import scheme as S


@pytest.fixture(scope="module", params=["c", "numpy"])
def kernel_path(request, monkeypatch_module=None):
    if request.param == "c":
        if OK.clib() is None:
            OK.build_c()
            OK._clib = None
        assert OK.clib() is not None
        OK._force_numpy = False
    else:
        OK._force_numpy = True
    yield request.param
    OK._force_numpy = False


def test_kernel_table_matches_reference(kernel_path):
    g = golden_npz("kernels_n64.npz")
    q, qinv, r2 = g["q"], g["qinv"], g["r2"]
    a, b = g["a"], g["b"]
    assert np.array_equal(OK.elementwise_mulmod(a, b, q, qinv, r2), g["mulmod"])
    assert np.array_equal(OK.elementwise_mont(a, b, q, qinv), g["mont"])
    assert np.array_equal(OK.rowwise_mont(a, g["c"], q, qinv), g["rowwise"])
    assert np.array_equal(OK.addmod_rows(a, b, q), g["add"])
    assert np.array_equal(OK.submod_rows(a, b, q), g["sub"])
    assert np.array_equal(OK.base_convert(g["hat"], g["punc"], q, qinv), g["bconv"])
    acc = a.copy()
    assert np.array_equal(OK.fma_inplace(acc, b, a, q, qinv, r2), g["fma"])
    acc = b.copy()
    assert np.array_equal(OK.fma_gather_inplace(acc, a, g["key"], g["rows"], q, qinv, r2),
                          g["fma_gather"])
    f = a.copy()
    assert np.array_equal(OK.ntt_forward_inplace(f, g["psi_rev"], q, qinv), g["ntt_fwd"])
    f = a.copy()
    assert np.array_equal(OK.ntt_inverse_inplace(f, g["ipsi_rev"], g["ninv"], q, qinv),
                          g["ntt_inv"])


def test_kernels_against_bigint():
    """Reference T/test_ring.py:177-203 semantics with Python ints."""
    g = golden_npz("kernels_n64.npz")
    q = g["q"]
    a, b = g["a"], g["b"]
    want = (a.astype(object) * b.astype(object)) % q.astype(object)[:, None]
    assert g["mulmod"].astype(object).tolist() == want.tolist()


def test_ring_tables_and_ntt():
    g = golden_npz("ring_n64.npz")
    primes = tuple(int(x) for x in g["primes"])
    p = S.Params(64, primes, (), 2.0 ** 40, 1, None, 3.2)
    assert np.array_equal(S.ntt_fwd(p, g["x"], primes), g["x_eval"])
    assert np.array_equal(S.ntt_inv(p, g["x_eval"], primes), g["x"])
    assert np.array_equal(S.mul(p, g["x_eval"], g["y_eval"], primes), g["prod"])
    assert np.array_equal(S.ntt_inv(p, g["prod"], primes), g["prod_coeff"])
    for gg in (3, 5, 127):
        assert np.array_equal(S.auto_eval(g["x_eval"], gg, 64), g[f"auto_eval_{gg}"])
    assert np.array_equal(2 * S.bitrev(64) + 1, g["exps"])
    assert np.array_equal(S.from_signed(g["signed"], primes), g["lifted"])


def test_negacyclic_schoolbook():
    """poly_mul == schoolbook negacyclic convolution (T/test_ring.py:14-26)."""
    g = golden_npz("ring_n64.npz")
    primes = tuple(int(x) for x in g["primes"])
    n = 64
    for i, q in enumerate(primes):
        x, y = g["x"][i].tolist(), g["y"][i].tolist()
        out = [0] * n
        for a in range(n):
            for b in range(n):
                k = a + b
                if k >= n:
                    out[k - n] -= x[a] * y[b]
                else:
                    out[k] += x[a] * y[b]
        assert [v % q for v in out] == g["prod_coeff"][i].tolist()


def _check_scheme(name, d, full):
    p = S.Params.from_text(preset_text(name) if name != "desk" else DESK_TEXT)
    keys = S.keygen(p, d["rotation_steps"], 7, conj="conj" in d)
    assert S.sha(keys.s_ext) == d["secret_ext"]
    assert S.sha(keys.pk[0]) == d["pk_b"]
    assert S.sha(keys.pk[1]) == d["pk_a"]
    assert [S.sha(x) for x in keys.relin[0]] == d["relin_b"]
    assert [S.sha(x) for x in keys.relin[1]] == d["relin_a"]
    for s, hs in d["rot"].items():
        k = keys.rot[int(s)]
        assert [S.sha(x) for x in k[0]] + [S.sha(x) for x in k[1]] == hs
    L = p.max_level
    rng = np.random.default_rng(1000)
    up = np.stack([rng.integers(0, q, size=p.n, dtype=np.uint64) for q in p.chain])
    assert S.sha(S.ntt_fwd(p, up, p.chain)) == d["ntt_fwd"]
    assert S.sha(S.ntt_inv(p, up, p.chain)) == d["ntt_inv"]
    for lvl, want in d["ks"].items():
        lvl = int(lvl)
        r = np.random.default_rng(2000 + lvl)
        dp = np.stack([r.integers(0, q, size=p.n, dtype=np.uint64) for q in p.chain[: lvl + 1]])
        kb, ka = S.ks_apply(p, keys.relin, dp, lvl)
        assert [S.sha(kb), S.sha(ka)] == want, f"ks level {lvl}"
    rng = np.random.default_rng(5)
    u = rng.uniform(-1, 1, p.slots)
    v = rng.uniform(-1, 1, p.slots)
    cu = S.encrypt_vector(p, keys, u, L, 1)
    cv = S.encrypt_vector(p, keys, v, L, 2)
    assert cu.digest() == d["enc_u"]
    assert cv.digest() == d["enc_v"]
    c3 = S.encrypt(p, keys, S.encode(p, u[:768], 3, p.scale), 3, p.scale, 3)
    assert c3.digest() == d["enc_l3"]
    prod = S.mult(p, keys, cu, cv)
    assert prod.digest() == d["mult"]
    assert np.array_equal(S.decrypt_vector(p, keys, prod)[:64], np.array(d["mult_dec"]))
    assert S.ct_add(p, cu, cv).digest() == d["add"]
    assert S.ct_sub(p, cu, cv).digest() == d["sub"]
    half = S.mult_plain(p, cu, S.const_pt(p, 0.5, L, p.scale), p.scale, rescale_after=False)
    assert S.rescale(p, half).digest() == d["rescale"]
    assert S.mult_plain(p, cu, S.encode(p, v, L, p.scale), p.scale).digest() == d["mult_plain_vec"]
    assert S.add_plain_const(p, cu, 0.25).digest() == d["add_plain_const"]
    assert S.mod_down(cu, max(1, L // 2)).digest() == d["mod_down"]
    assert S.ct_add(p, prod, S.mod_down(cv, prod.level - 1)).digest() == d["add_aligned"]
    if full:
        for s in d["rotation_steps"]:
            assert S.rotate(p, keys, cu, s).digest() == d[f"rot_{s}"]
        assert S.rotate(p, keys, cu, 3).digest() == d["rot_3"]
        if "conj" in d:
            assert S.conjugate(p, keys, cu).digest() == d["conj_ct"]


DESK_TEXT = """hebert-preset v1
scale 0x1.0000000000000p+40
security insecure-test-only
dnum 3
secret_hamming_weight 0
error_sigma 0x1.999999999999ap+1
hebert-ring-config v1
name desk
N 8192
moduli 0xfffffffffffc001 0xfffffdc001 0xfffff4c001 0xfffff3c001 0xffffe80001 0xffffe74001 0xffffd6c001 0xffffd44001 0xffffd0c001
special 0xffffffffffe8001 0xffffffffffd8001 0xffffffffffc4001
"""


def test_oracle_desk(digests):
    _check_scheme("desk", digests["desk"], True)


def test_oracle_p14(digests):
    _check_scheme("p14", digests["p14"], True)


@pytest.mark.slow
def test_oracle_p16(digests):
    if OK.clib() is None:
        OK.build_c()
        OK._clib = None
    _check_scheme("p16", digests["p16"], False)


def test_oracle_mod_raise(digests):
    from paper_2210_02574_b200.ckks import params as P

    text = P.get_preset("desk-boot").to_config_text()
    p = S.Params.from_text(text)
    d = digests["boot_desk64"]
    keys = S.keygen(p, [], 11, conj=False)  # pk precedes every switch key in the RNG stream
    v = golden_npz("boot_desk64.npz")["v"]
    ct = S.encrypt_vector(p, keys, v, 0, 21)
    assert ct.digest() == d["enc"]
    assert S.mod_raise(p, ct).digest() == d["mod_raise"]
