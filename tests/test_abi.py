"""The C-ABI boundary: libhegpu.so builds, loads and exports every entry point
include/hegpu.h declares (no compute: CPU only)."""

import re

import pytest

from paper_2210_02574_b200 import _lib, build


@pytest.fixture(scope="module")
def lib():
    build.build_lib()
    return _lib.load()


def declared():
    text = open(_lib.HEADER_PATH).read()
    return sorted(set(re.findall(r"\b(hegpu_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_kernel_table():
    names = declared()
    table = [
        "ntt_forward_inplace", "ntt_inverse_inplace", "elementwise_mont", "elementwise_mulmod",
        "rowwise_mont", "addmod_rows", "submod_rows", "base_convert", "fma_inplace",
        "fma_gather_inplace",
    ]
    for t in table:  # the ten functions of hebert._kernels (_kernels.py:319-328)
        assert f"hegpu_k_{t}" in names


def test_every_declared_symbol_is_exported(lib):
    for name in declared():
        assert hasattr(lib, name), name


def test_bindings_cover_the_header(lib):
    assert set(declared()) == set(_lib.SIGNATURES)
    assert set(_lib.exported_symbols()) == set(_lib.SIGNATURES)


def test_version_and_error_channel(lib):
    assert b"sm_100a" in lib.hegpu_version()
    assert isinstance(_lib.last_error(), str)
    assert lib.hegpu_device_count() >= 0


def test_bad_arguments_fail_loudly(lib):
    import ctypes

    handle = ctypes.c_void_p()
    # ring degree 2^3 is rejected before any device work
    rc = lib.hegpu_ring_create(3, None, 0, None, 0, ctypes.byref(handle))
    assert rc != 0
    assert "ring degree" in _lib.last_error()
    assert lib.hegpu_ring_destroy(None) == 0


def test_kernel_table_module_matches_reference_surface():
    from paper_2210_02574_b200 import _kernels

    for name in ("ntt_forward_inplace", "ntt_inverse_inplace", "elementwise_mont",
                 "elementwise_mulmod", "base_convert", "rowwise_mont", "addmod_rows",
                 "submod_rows", "fma_inplace", "fma_gather_inplace"):
        assert callable(getattr(_kernels, name))


def test_no_gpu_means_loud_failure():
    """Without a CUDA device the product raises instead of falling back to CPU."""
    from paper_2210_02574_b200 import ckks
    from paper_2210_02574_b200.errors import DeviceError

    if _lib.load().hegpu_device_count() > 0:
        pytest.skip("a GPU is present")
    params = ckks.get_preset("desk")
    with pytest.raises(DeviceError):
        ckks.keygen(params, rotation_steps=[1])
