"""Drop-in for the reference kernel seam `hebert._kernels` (_kernels.py:319-328).

The ten functions take and return host numpy uint64 arrays with the
reference's exact signatures and ownership rules (*_inplace mutate their first
argument and return it; the others return a new array) and run on the GPU
through the hegpu_k_* entry points of libhegpu (include/hegpu.h).  Callers
that bind the kernel table keep working; the engine itself uses the
device-resident entry points instead.
"""

import numpy as np

from . import _lib

USE_NUMBA = False  # reference flag; this table always runs on the GPU


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


def _vec(v):
    return np.ascontiguousarray(np.asarray(v, dtype=np.uint64).ravel())


def ntt_forward_inplace(a, psi_rev, q_vec, qinv_vec):
    """In-place forward negacyclic NTT (natural -> bit-reversed), _kernels.py:144-171."""
    if not (a.flags.c_contiguous and a.dtype == np.uint64):
        raise ValueError("a must be a C-contiguous uint64 array")
    k, n = a.shape
    psi = _u64(psi_rev)
    q, qi = _vec(q_vec), _vec(qinv_vec)
    _lib.call("hegpu_k_ntt_forward_inplace", a.ctypes.data, k, n, psi.ctypes.data,
              q.ctypes.data, qi.ctypes.data)
    return a


def ntt_inverse_inplace(a, ipsi_rev, ninv_vec, q_vec, qinv_vec):
    """In-place inverse NTT (bit-reversed -> natural, times N^-1), _kernels.py:173-204."""
    if not (a.flags.c_contiguous and a.dtype == np.uint64):
        raise ValueError("a must be a C-contiguous uint64 array")
    k, n = a.shape
    ipsi = _u64(ipsi_rev)
    ninv, q, qi = _vec(ninv_vec), _vec(q_vec), _vec(qinv_vec)
    _lib.call("hegpu_k_ntt_inverse_inplace", a.ctypes.data, k, n, ipsi.ctypes.data,
              ninv.ctypes.data, q.ctypes.data, qi.ctypes.data)
    return a


def elementwise_mont(a, b, q_vec, qinv_vec):
    a, b = _u64(a), _u64(b)
    out = np.empty_like(a)
    q, qi = _vec(q_vec), _vec(qinv_vec)
    _lib.call("hegpu_k_elementwise_mont", a.ctypes.data, b.ctypes.data, out.ctypes.data,
              a.shape[0], a.shape[1], q.ctypes.data, qi.ctypes.data)
    return out


def elementwise_mulmod(a, b, q_vec, qinv_vec, r2_vec):
    a, b = _u64(a), _u64(b)
    out = np.empty_like(a)
    q, qi, r2 = _vec(q_vec), _vec(qinv_vec), _vec(r2_vec)
    _lib.call("hegpu_k_elementwise_mulmod", a.ctypes.data, b.ctypes.data, out.ctypes.data,
              a.shape[0], a.shape[1], q.ctypes.data, qi.ctypes.data, r2.ctypes.data)
    return out


def rowwise_mont(a, c_vec, q_vec, qinv_vec):
    a = _u64(a)
    out = np.empty_like(a)
    c, q, qi = _vec(c_vec), _vec(q_vec), _vec(qinv_vec)
    _lib.call("hegpu_k_rowwise_mont", a.ctypes.data, c.ctypes.data, out.ctypes.data,
              a.shape[0], a.shape[1], q.ctypes.data, qi.ctypes.data)
    return out


def addmod_rows(a, b, q_vec):
    a, b = _u64(a), _u64(b)
    out = np.empty_like(a)
    q = _vec(q_vec)
    _lib.call("hegpu_k_addmod_rows", a.ctypes.data, b.ctypes.data, out.ctypes.data,
              a.shape[0], a.shape[1], q.ctypes.data)
    return out


def submod_rows(a, b, q_vec):
    a, b = _u64(a), _u64(b)
    out = np.empty_like(a)
    q = _vec(q_vec)
    _lib.call("hegpu_k_submod_rows", a.ctypes.data, b.ctypes.data, out.ctypes.data,
              a.shape[0], a.shape[1], q.ctypes.data)
    return out


def base_convert(hat, punc_to, q_to, qinv_to):
    """acc[j] = sum_i hat[i] * punc_to[i, j] (Montgomery) mod q_to[j], _kernels.py:300-317."""
    hat = _u64(hat)
    punc = _u64(punc_to)
    q, qi = _vec(q_to), _vec(qinv_to)
    l, n = hat.shape
    kt = q.shape[0]
    out = np.zeros((kt, n), dtype=np.uint64)
    _lib.call("hegpu_k_base_convert", hat.ctypes.data, l, n, punc.ctypes.data, kt,
              q.ctypes.data, qi.ctypes.data, out.ctypes.data)
    return out


def fma_inplace(acc, a, b, q_vec, qinv_vec, r2_vec):
    """acc += a*b mod q in place (_kernels.py:255-269)."""
    if not (acc.flags.c_contiguous and acc.dtype == np.uint64):
        raise ValueError("acc must be a C-contiguous uint64 array")
    a, b = _u64(a), _u64(b)
    q, qi, r2 = _vec(q_vec), _vec(qinv_vec), _vec(r2_vec)
    _lib.call("hegpu_k_fma_inplace", acc.ctypes.data, a.ctypes.data, b.ctypes.data,
              acc.shape[0], acc.shape[1], q.ctypes.data, qi.ctypes.data, r2.ctypes.data)
    return acc


def fma_gather_inplace(acc, a, key, rows, q_vec, qinv_vec, r2_vec):
    """acc[i] += a[i] * key[rows[i]] mod q in place (_kernels.py:271-286)."""
    if not (acc.flags.c_contiguous and acc.dtype == np.uint64):
        raise ValueError("acc must be a C-contiguous uint64 array")
    a, key = _u64(a), _u64(key)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    q, qi, r2 = _vec(q_vec), _vec(qinv_vec), _vec(r2_vec)
    _lib.call("hegpu_k_fma_gather_inplace", acc.ctypes.data, a.ctypes.data, key.ctypes.data,
              key.shape[0], rows.ctypes.data, acc.shape[0], acc.shape[1], q.ctypes.data,
              qi.ctypes.data, r2.ctypes.data)
    return acc
