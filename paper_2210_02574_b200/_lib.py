"""ctypes binding of libhegpu.so (the C ABI declared in include/hegpu.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is visible, every device entry point raises DeviceError.  Symbol
presence can be checked without a GPU (`exported_symbols`).
"""

import ctypes
import os
import threading

from .errors import DeviceError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HEGPU_LIB") or os.path.join(_HERE, "libhegpu.so")  # override: experiments
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "hegpu.h")

(OP_ADD, OP_SUB, OP_MUL, OP_MONT, OP_NEG, OP_SCALAR, OP_ROWMONT, OP_FMA, OP_COPY, OP_ADDC,
 OP_REDUCE) = range(11)

_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_U64 = ctypes.c_uint64

# name -> argtypes (restype is int unless listed in _RESTYPES)
SIGNATURES = {
    "hegpu_version": [],
    "hegpu_last_error": [],
    "hegpu_device_count": [],
    "hegpu_launch_count": [],
    "hegpu_bench_modmul_peak": [_I, _P],
    "hegpu_bench_fp_modmul_peak": [_I, _P],
    "hegpu_profile_enable": [_I],
    "hegpu_profile_read": [_P, _P, _P, _P, _I],
    "hegpu_ring_create": [_I, _P, _I, _P, _I, _P],
    "hegpu_ring_destroy": [_P],
    "hegpu_ring_get_tables": [_P, _I, _P],
    "hegpu_ntt": [_P, _I, _P, _I64, _P, _I64, _I, _I, _P, _P],
    "hegpu_elementwise": [_P, _I, _P, _I64, _P, _I64, _P, _I64, _I, _I, _P, _P, _P],
    "hegpu_lift_signed": [_P, _P, _I64, _P, _I64, _I, _I, _P, _P],
    "hegpu_lift_centered": [_P, _P, _I64, _I, _P, _I64, _I, _I, _P, _P],
    "hegpu_automorphism": [_P, _I, _U64, _P, _I64, _P, _I64, _I, _I, _P, _P],
    "hegpu_encode_diags": [_P, _I, _I, ctypes.c_double, ctypes.c_double, _I, _P, _P, _P, _P,
                           _P, _P],
    "hegpu_encode_overflow": [_P, _P],
    "hegpu_ntt_from_signed": [_P, _P, _I64, _P, _I64, _I, _I, _P, _P],
    "hegpu_pcg64_uniform": [_U64, _U64, _U64, _U64, _P, _I, _I, _P, _I64, _P, _P],
    "hegpu_sample_encrypt": [_P, _I, _U64, ctypes.c_double, _P],
    "hegpu_tensor": [_P, _P, _P, _I64, _P, _P, _I64, _P, _P, _P, _I64, _I, _I, _P],
    "hegpu_ks_apply": [_P, _I, _I, _P, _I64, _I, _P, _P, _I, _P, _P, _I64, _I, _P],
    "hegpu_tensor_periodic": [_P, _P, _P, _I64, _I, _P, _P, _I64, _P, _P, _P, _I64, _I, _I, _P],
    "hegpu_ks_rotsum": [_P, _I, _I, _P, _I64, _I64, _I, _I, _P, _P, _P, _I, _P, _I64, _I64, _P],
    "hegpu_ks_apply_rescale": [_P, _I, _I, _P, _I64, _I, _P, _P, _I, _P, _I64, _I64, _P, _I64,
                               _I64, _P],
    "hegpu_ks_hoisted": [_P, _I, _I, _P, _I64, _I64, _I, _I, _P, _P, _P, _I, _P, _I, _P],
    "hegpu_bsgs_giants": [_P, _I, _I, _P, _I64, _I, _I, _P, _P, _P, _I, _P, _I, _I, _P],
    "hegpu_moddown_rescale_ext": [_P, _I, _I, _P, _I, _P, _P],
    "hegpu_set_allocator": [_P, _P],
    "hegpu_rescale": [_P, _I, _P, _I64, _P, _I64, _I, _P],
    "hegpu_mod_raise": [_P, _P, _I64, _P, _I64, _I, _I, _P],
    "hegpu_encrypt_combine": [_P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P],
    "hegpu_diag_mac": [_P, _P, _I64, _I64, _P, _I, _I, _P, _I64, _I64, _I, _I, _P],
    "hegpu_bsgs": [_P, _P, _I, _I64, _I64, _I, _P, _I64, _I, _P, _I, _P, _I64, _I, _I, _P],
    "hegpu_k_ntt_forward_inplace": [_P, _I, _I, _P, _P, _P],
    "hegpu_k_ntt_inverse_inplace": [_P, _I, _I, _P, _P, _P, _P],
    "hegpu_k_elementwise_mont": [_P, _P, _P, _I, _I, _P, _P],
    "hegpu_k_elementwise_mulmod": [_P, _P, _P, _I, _I, _P, _P, _P],
    "hegpu_k_rowwise_mont": [_P, _P, _P, _I, _I, _P, _P],
    "hegpu_k_addmod_rows": [_P, _P, _P, _I, _I, _P],
    "hegpu_k_submod_rows": [_P, _P, _P, _I, _I, _P],
    "hegpu_k_base_convert": [_P, _I, _I, _P, _I, _P, _P, _P],
    "hegpu_k_fma_inplace": [_P, _P, _P, _I, _I, _P, _P, _P],
    "hegpu_k_fma_gather_inplace": [_P, _P, _P, _I, _P, _I, _I, _P, _P, _P],
}
_RESTYPES = {
    "hegpu_version": ctypes.c_char_p,
    "hegpu_last_error": ctypes.c_char_p,
    "hegpu_launch_count": ctypes.c_longlong,
}
PROF_CLASSES = ("ntt", "elementwise", "lift", "automorphism", "tensor", "conv", "ks_ip",
                "diag_mac", "encrypt", "encode",
                # subsets of "ntt" by the step that issued them (not additive)
                "ntt_modup", "ntt_moddown", "ntt_rescale")

_lock = threading.Lock()
_lib = None


def load():
    """Load libhegpu.so (raises DeviceError if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise DeviceError(
                f"libhegpu.so not built at {LIB_PATH}; run __graft_entry__.build() "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, ctypes.c_int)
        _lib = lib
    return _lib


def exported_symbols():
    """Names from SIGNATURES that the built library exports (no GPU needed)."""
    lib = load()
    return [n for n in SIGNATURES if hasattr(lib, n)]


def last_error():
    return load().hegpu_last_error().decode("utf-8", "replace")


def check(rc, what=""):
    if rc != 0:
        raise DeviceError(f"hegpu{(' ' + what) if what else ''} failed (code {rc}): {last_error()}")


_gpu_checked = [False]


def require_gpu():
    """Fail loudly when no CUDA device is present (no CPU fallback)."""
    if _gpu_checked[0]:
        return
    lib = load()
    if lib.hegpu_device_count() < 1:
        raise DeviceError("no CUDA device visible: the B200 CKKS engine has no CPU path")
    _gpu_checked[0] = True


def call(name, *args):
    fn = getattr(load(), name)
    check(fn(*args), name)


def launch_count():
    return int(load().hegpu_launch_count())


def profile_enable(on=True):
    call("hegpu_profile_enable", 1 if on else 0)


def profile_read():
    """{class: {ms, launches, bytes, modmuls}} since profile_enable (syncs the device)."""
    import numpy as np

    n = len(PROF_CLASSES)
    ms = np.zeros(n, dtype=np.float64)
    cnt = np.zeros(n, dtype=np.int64)
    by = np.zeros(n, dtype=np.float64)
    mm = np.zeros(n, dtype=np.float64)
    call("hegpu_profile_read", ms.ctypes.data, cnt.ctypes.data, by.ctypes.data, mm.ctypes.data,
         n)
    return {c: {"ms": float(ms[i]), "launches": int(cnt[i]), "bytes": float(by[i]),
                "modmuls": float(mm[i])} for i, c in enumerate(PROF_CLASSES)}


def modmul_peak(iters=4096):
    """Measured INT64 Shoup modmul/s of the current GPU."""
    out = ctypes.c_double()
    call("hegpu_bench_modmul_peak", iters, ctypes.byref(out))
    return out.value


def fp_modmul_peak(iters=4096):
    """Measured FP64-pipe modmul/s (primes < 2^46) of the current GPU."""
    out = ctypes.c_double()
    call("hegpu_bench_fp_modmul_peak", iters, ctypes.byref(out))
    return out.value
