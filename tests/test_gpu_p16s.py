"""The 128-bit-secure N = 2^16 bootstrappable preset (p16s: sparse secret
h = 192, scale 2^45, 45-bit rescale primes, 50-bit q0, 60-bit CoeffToSlot
and special primes, logQP = 1430).  Its scheme ops are pinned
bit-exact to the reference in test_gpu_ckks.py; here: full-slot and sparse
bootstrapping within the north-star 1e-3, with the double-angle EvalMod that
the wider h = 192 range (K = 25) needs."""

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

from paper_2210_02574_b200 import bootstrap as bs, ckks  # noqa: E402


@pytest.fixture(scope="module")
def secure():
    params = ckks.get_preset("p16s")
    full = bs.build_context(params, n_slots=params.slot_count)
    sparse = bs.build_context(params, n_slots=1024, input_periodic=True)
    steps = sorted(set(full.required_rotation_steps()) | set(bs.refresh_rotation_steps(sparse)))
    keys = ckks.keygen(params, rotation_steps=steps, rng_seed=7)
    return params, full, sparse, keys


def test_p16s_context(secure):
    params, full, sparse, keys = secure
    assert params.secret_hamming_weight == 192 and params.default_scale == 2.0 ** 45
    assert full.range_k == 25 and full.double_angle == 4 and full.evalmod_poly.degree == 31
    assert full.output_level == sparse.output_level == params.max_level - 12 == 9


def test_p16s_full_slot_bootstrap_within_1e3(secure):
    params, full, _, keys = secure
    rng = np.random.default_rng(1003)
    vs = [rng.uniform(-1, 1, params.slot_count) for _ in range(2)]
    cts = [ckks.encrypt_vector(params, v, keys, level=0, rng_seed=60 + i) for i, v in enumerate(vs)]
    outs = bs.bootstrap_many(cts, full, keys)
    errs = [float(np.max(np.abs(ckks.decrypt_vector(o, keys) - v))) for o, v in zip(outs, vs)]
    print(f"p16s full-slot bootstrap errors {errs}")
    assert all(o.level == full.output_level for o in outs)
    assert max(errs) <= 1e-3


def test_p16s_sparse_refresh_within_1e3(secure):
    params, _, sparse, keys = secure
    rng = np.random.default_rng(1004)
    vs = [np.tile(rng.uniform(-1, 1, 1024), params.slot_count // 1024) for _ in range(2)]
    cts = [ckks.encrypt_vector(params, v, keys, level=1, rng_seed=70 + i) for i, v in enumerate(vs)]
    outs = bs.BootstrapRefresher(sparse, keys).refresh_many(cts)  # packed pair
    errs = [float(np.max(np.abs(ckks.decrypt_vector(o, keys) - v))) for o, v in zip(outs, vs)]
    print(f"p16s packed sparse refresh errors {errs}")
    assert max(errs) <= 1e-3
