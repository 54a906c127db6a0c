"""TEST INFRASTRUCTURE ONLY -- CPU kernel table of the oracle.

numpy restatement of hebert/_kernels.py (numpy twins :29-113 and the numba
kernels :122-317), with an optional OpenMP C build of the same kernels
(oracle/csrc/hekernels.c -> oracle/_build/libhekernels.so) for speed.  Both
paths are bit-identical (modular arithmetic is exact); tests pin both.
"""

import ctypes
import os

import numpy as np

_U32 = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)

_HERE = os.path.dirname(os.path.abspath(__file__))
C_LIB_PATH = os.path.join(_HERE, "_build", "libhekernels.so")
_clib = None
_force_numpy = os.environ.get("ORACLE_NUMPY_ONLY", "") != ""


def build_c(verbose=False):
    """Compile the C kernel table (gcc -O3 -fopenmp)."""
    import subprocess

    os.makedirs(os.path.dirname(C_LIB_PATH), exist_ok=True)
    src = os.path.join(_HERE, "csrc", "hekernels.c")
    cmd = ["gcc", "-O3", "-march=x86-64-v3", "-fopenmp", "-fPIC", "-shared", "-o", C_LIB_PATH, src]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return C_LIB_PATH


def clib():
    global _clib
    if _force_numpy:
        return None
    if _clib is None and os.path.exists(C_LIB_PATH):
        lib = ctypes.CDLL(C_LIB_PATH)
        P, I = ctypes.c_void_p, ctypes.c_int
        sigs = {
            "ok_ntt_forward": [P, I, I, P, P, P],
            "ok_ntt_inverse": [P, I, I, P, P, P, P],
            "ok_mulmod": [P, P, P, I, I, P, P, P],
            "ok_mont": [P, P, P, I, I, P, P],
            "ok_rowwise": [P, P, P, I, I, P, P],
            "ok_addmod": [P, P, P, I, I, P],
            "ok_submod": [P, P, P, I, I, P],
            "ok_fma_gather": [P, P, P, P, I, I, P, P, P],
            "ok_base_convert": [P, I, I, P, I, P, P, P],
        }
        for name, args in sigs.items():
            getattr(lib, name).argtypes = args
            getattr(lib, name).restype = None
        _clib = lib
    return _clib


def _c(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


# ---------------------------------------------------------------------------
# numpy restatement (_kernels.py:29-113)
# ---------------------------------------------------------------------------


def mulhi(a, b):
    """High 64 bits of a*b from 32-bit partial products (_kernels.py:29-39)."""
    a_lo, a_hi = a & _U32, a >> _S32
    b_lo, b_hi = b & _U32, b >> _S32
    ll, lh, hl = a_lo * b_lo, a_lo * b_hi, a_hi * b_lo
    mid = (ll >> _S32) + (lh & _U32) + (hl & _U32)
    return a_hi * b_hi + (lh >> _S32) + (hl >> _S32) + (mid >> _S32)


def mont(a, b, q, qinv):
    """REDC a*b*2^-64 mod q (_kernels.py:42-46)."""
    t_lo = a * b
    m = t_lo * qinv
    r = mulhi(a, b) + mulhi(m, q) + (t_lo != 0).astype(np.uint64)
    return r - q * (r >= q)


def ntt_forward_inplace(a, psi_rev, q_vec, qinv_vec):
    """CT forward NTT, natural -> bit-reversed (_kernels.py:48-65 / :144-171)."""
    lib = clib()
    if lib is not None and a.flags.c_contiguous:
        k, n = a.shape
        psi, q, qi = _c(psi_rev[:k]), _c(q_vec), _c(qinv_vec)
        lib.ok_ntt_forward(a.ctypes.data, k, n, psi.ctypes.data, q.ctypes.data, qi.ctypes.data)
        return a
    k, n = a.shape
    q = q_vec[:, None, None]
    qi = qinv_vec[:, None, None]
    t, m = n, 1
    while m < n:
        t >>= 1
        view = a.reshape(k, m, 2 * t)
        s = psi_rev[:, m : 2 * m, None]
        u = view[:, :, :t].copy()
        v = mont(view[:, :, t:], s, q, qi)
        sm = u + v
        view[:, :, :t] = sm - q * (sm >= q)
        df = u + (q - v)
        view[:, :, t:] = df - q * (df >= q)
        m <<= 1
    return a


def ntt_inverse_inplace(a, ipsi_rev, ninv_vec, q_vec, qinv_vec):
    """GS inverse NTT then N^-1 (_kernels.py:68-88 / :173-204)."""
    lib = clib()
    if lib is not None and a.flags.c_contiguous:
        k, n = a.shape
        ipsi, ninv, q, qi = _c(ipsi_rev[:k]), _c(ninv_vec), _c(q_vec), _c(qinv_vec)
        lib.ok_ntt_inverse(a.ctypes.data, k, n, ipsi.ctypes.data, ninv.ctypes.data,
                           q.ctypes.data, qi.ctypes.data)
        return a
    k, n = a.shape
    q = q_vec[:, None, None]
    qi = qinv_vec[:, None, None]
    t, m = 1, n
    while m > 1:
        h = m >> 1
        view = a.reshape(k, h, 2 * t)
        s = ipsi_rev[:, h : 2 * h, None]
        u = view[:, :, :t].copy()
        v = view[:, :, t:].copy()
        sm = u + v
        view[:, :, :t] = sm - q * (sm >= q)
        df = u + (q - v)
        df -= q * (df >= q)
        view[:, :, t:] = mont(df, s, q, qi)
        t <<= 1
        m = h
    a[:] = mont(a, ninv_vec[:, None], q_vec[:, None], qinv_vec[:, None])
    return a


def elementwise_mont(a, b, q_vec, qinv_vec):
    lib = clib()
    if lib is not None:
        a, b = _c(a), _c(b)
        out = np.empty_like(a)
        q, qi = _c(q_vec), _c(qinv_vec)
        lib.ok_mont(a.ctypes.data, b.ctypes.data, out.ctypes.data, a.shape[0], a.shape[1],
                    q.ctypes.data, qi.ctypes.data)
        return out
    return mont(a, b, q_vec[:, None], qinv_vec[:, None])


def elementwise_mulmod(a, b, q_vec, qinv_vec, r2_vec):
    """a*b mod q = mont(mont(a,b), R^2) (_kernels.py:288-298)."""
    lib = clib()
    if lib is not None:
        a, b = _c(a), _c(b)
        out = np.empty_like(a)
        q, qi, r2 = _c(q_vec), _c(qinv_vec), _c(r2_vec)
        lib.ok_mulmod(a.ctypes.data, b.ctypes.data, out.ctypes.data, a.shape[0], a.shape[1],
                      q.ctypes.data, qi.ctypes.data, r2.ctypes.data)
        return out
    ab = mont(a, b, q_vec[:, None], qinv_vec[:, None])
    return mont(ab, r2_vec[:, None], q_vec[:, None], qinv_vec[:, None])


def rowwise_mont(a, c_vec, q_vec, qinv_vec):
    lib = clib()
    if lib is not None:
        a = _c(a)
        out = np.empty_like(a)
        c, q, qi = _c(c_vec), _c(q_vec), _c(qinv_vec)
        lib.ok_rowwise(a.ctypes.data, c.ctypes.data, out.ctypes.data, a.shape[0], a.shape[1],
                       q.ctypes.data, qi.ctypes.data)
        return out
    return mont(a, c_vec[:, None], q_vec[:, None], qinv_vec[:, None])


def addmod_rows(a, b, q_vec):
    lib = clib()
    if lib is not None:
        a, b = _c(a), _c(b)
        out = np.empty_like(a)
        q = _c(q_vec)
        lib.ok_addmod(a.ctypes.data, b.ctypes.data, out.ctypes.data, a.shape[0], a.shape[1],
                      q.ctypes.data)
        return out
    s = a + b
    return s - q_vec[:, None] * (s >= q_vec[:, None])


def submod_rows(a, b, q_vec):
    lib = clib()
    if lib is not None:
        a, b = _c(a), _c(b)
        out = np.empty_like(a)
        q = _c(q_vec)
        lib.ok_submod(a.ctypes.data, b.ctypes.data, out.ctypes.data, a.shape[0], a.shape[1],
                      q.ctypes.data)
        return out
    s = a + (q_vec[:, None] - b)
    return s - q_vec[:, None] * (s >= q_vec[:, None])


def base_convert(hat, punc_to, q_to, qinv_to):
    """out_j = sum_i mont(hat_i, punc_ij) mod p_j (_kernels.py:95-113 / :300-317)."""
    lib = clib()
    l, n = hat.shape
    kt = q_to.shape[0]
    if lib is not None:
        hat, punc = _c(hat), _c(punc_to)
        q, qi = _c(q_to), _c(qinv_to)
        out = np.empty((kt, n), dtype=np.uint64)
        lib.ok_base_convert(hat.ctypes.data, l, n, punc.ctypes.data, kt, q.ctypes.data,
                            qi.ctypes.data, out.ctypes.data)
        return out
    out = np.zeros((kt, n), dtype=np.uint64)
    for j in range(kt):
        q, qi = q_to[j], qinv_to[j]
        acc = np.zeros(n, dtype=np.uint64)
        for i in range(l):
            s = acc + mont(hat[i], punc_to[i, j], q, qi)
            acc = s - q * (s >= q)
        out[j] = acc
    return out


def fma_inplace(acc, a, b, q_vec, qinv_vec, r2_vec):
    acc[:] = addmod_rows(acc, elementwise_mulmod(a, b, q_vec, qinv_vec, r2_vec), q_vec)
    return acc


def fma_gather_inplace(acc, a, key, rows, q_vec, qinv_vec, r2_vec):
    """acc[i] += a[i]*key[rows[i]] mod q (_kernels.py:271-286)."""
    lib = clib()
    if lib is not None and acc.flags.c_contiguous:
        a, key = _c(a), _c(key)
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        q, qi, r2 = _c(q_vec), _c(qinv_vec), _c(r2_vec)
        lib.ok_fma_gather(acc.ctypes.data, a.ctypes.data, key.ctypes.data, rows.ctypes.data,
                          acc.shape[0], acc.shape[1], q.ctypes.data, qi.ctypes.data,
                          r2.ctypes.data)
        return acc
    return fma_inplace(acc, a, key[rows], q_vec, qinv_vec, r2_vec)
