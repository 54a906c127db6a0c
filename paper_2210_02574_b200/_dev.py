"""Device memory / stream plumbing (PyTorch is used only as the allocator and
stream provider; all arithmetic runs in libhegpu).

Residue limbs live in torch.int64 CUDA tensors that are bit-identical to the
reference's uint64 limb matrices (ring.py:257-279).  A "poly group" tensor has
shape (..., k, N) with unit stride along N and stride N along limbs; its
leading dimensions must be uniformly strided so one C-ABI call covers them.
"""

import numpy as np

from . import _lib
from .errors import CryptoError, DeviceError

try:  # torch is the device allocator; importing it is cheap after warm-up
    import torch
except Exception as exc:  # pragma: no cover - torch is part of the image
    torch = None
    _TORCH_ERR = exc
else:
    _TORCH_ERR = None

_PRIME_CACHE = {}


def require():
    if torch is None:
        raise DeviceError(f"torch unavailable: {_TORCH_ERR}")
    _lib.require_gpu()
    if not torch.cuda.is_available():
        raise DeviceError("torch sees no CUDA device")
    if not _ALLOCATOR:
        _install_allocator()


_ALLOCATOR = []  # keeps the ctypes callbacks alive


def _install_allocator():
    """Route libhegpu's scratch buffers through torch's caching allocator
    (hegpu_set_allocator): one pool for tensors and scratch, so a large
    workload (e.g. the full-slot ingest next to ~100 GB of keys and data)
    does not strand memory in one allocator that the other needs.
    HEGPU_DRIVER_SCRATCH=1 keeps the driver's stream-ordered pool."""
    import ctypes
    import os

    if os.environ.get("HEGPU_DRIVER_SCRATCH") == "1":
        _ALLOCATOR.append(None)
        return
    alloc_t = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
    free_t = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)

    def _alloc(nbytes, stream):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), torch.cuda.current_device(),
                                                      int(stream or 0))
        except Exception:  # noqa: BLE001 -- OOM becomes HEGPU_E_NOMEM in the library
            return None

    def _free(ptr, nbytes, stream):
        torch.cuda.caching_allocator_delete(ptr)

    fa, ff = alloc_t(_alloc), free_t(_free)
    _lib.call("hegpu_set_allocator", ctypes.cast(fa, ctypes.c_void_p),
              ctypes.cast(ff, ctypes.c_void_p))
    _ALLOCATOR.extend([fa, ff])


def device():
    return torch.device("cuda", torch.cuda.current_device())


def stream():
    return torch.cuda.current_stream().cuda_stream


def empty(*shape):
    return torch.empty(shape, dtype=torch.int64, device=device())


def zeros(*shape):
    return torch.zeros(shape, dtype=torch.int64, device=device())


def ptr(t):
    return t.data_ptr()


def to_device(arr):
    """numpy uint64/int64 array -> device int64 tensor (H2D copy)."""
    a = np.ascontiguousarray(arr)
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    elif a.dtype != np.int64:
        a = a.astype(np.int64)
    return torch.from_numpy(a).to(device(), non_blocking=False)


def to_host(t):
    """device int64 tensor -> numpy uint64 (D2H copy)."""
    return t.detach().to("cpu").contiguous().numpy().view(np.uint64)


def group(t, k, n):
    """(ptr, n_polys, poly_stride) of a (..., k, N) tensor with uniform strides."""
    if t.dtype != torch.int64 or not t.is_cuda:
        raise CryptoError("limbs must be a CUDA int64 tensor")
    if t.shape[-2:] != (k, n):
        raise CryptoError(f"limb shape {tuple(t.shape)} inconsistent with ({k}, {n})")
    if t.stride(-1) != 1 or (k > 1 and t.stride(-2) != n):
        raise CryptoError("limbs must be contiguous within a poly")
    lead = t.shape[:-2]
    if len(lead) == 0:
        return t.data_ptr(), 1, k * n
    count = 1
    for s in lead:
        count *= s
    if count == 1:
        return t.data_ptr(), 1, k * n
    # collapse leading dims: require a single uniform stride
    strides = [t.stride(i) for i in range(len(lead))]
    inner = strides[-1]
    expect = inner
    for i in range(len(lead) - 1, 0, -1):
        expect *= lead[i]
        if lead[i - 1] > 1 and strides[i - 1] != expect:
            raise CryptoError("poly group is not uniformly strided")
    return t.data_ptr(), count, inner


def prime_array(key, values):
    """Cached int32 numpy array of global prime indices (kept alive for ctypes)."""
    arr = _PRIME_CACHE.get(key)
    if arr is None:
        arr = np.ascontiguousarray(values, dtype=np.int32)
        _PRIME_CACHE[key] = arr
    return arr


def chain_primes(k):
    return prime_array(("chain", k), range(k))


def ext_primes(level, n_chain, n_special):
    return prime_array(
        ("ext", level, n_chain, n_special),
        list(range(level + 1)) + [n_chain + i for i in range(n_special)],
    )


class PtCache:
    """Bounded LRU cache of device plaintexts (encoded masks and constants).

    Keys may carry per-input values (a bootstrap's scale correction), so an
    unbounded dict grows with every distinct input scale.  Entries read while
    a CUDA graph is captured must outlive the graph: captured objects keep
    the list `pin_cached()` returns (every live entry at capture time)."""

    _ALL = []

    def __init__(self, maxsize=64):
        from collections import OrderedDict

        self.maxsize = maxsize
        self._d = OrderedDict()
        PtCache._ALL.append(self)

    def get(self, key):
        v = self._d.get(key)
        if v is not None:
            self._d.move_to_end(key)
            _note_capture(v)
        return v

    def __setitem__(self, key, value):
        self._d[key] = value
        self._d.move_to_end(key)
        _note_capture(value)
        while len(self._d) > self.maxsize:
            self._d.popitem(last=False)

    def __getitem__(self, key):
        return self._d[key]

    def __len__(self):
        return len(self._d)

    def clear(self):
        self._d.clear()


_CAPTURE_REFS = []


def _note_capture(v):
    if torch is not None and torch.cuda.is_available() and torch.cuda.is_current_stream_capturing():
        _CAPTURE_REFS.append(v)


def pin_cached():
    """Strong references to every cached plaintext plus every one read during
    the capture that just ended (held by captured graphs)."""
    refs = [v for c in PtCache._ALL for v in c._d.values()] + _CAPTURE_REFS
    _CAPTURE_REFS.clear()
    return refs


def driver_scratch():
    """True when libhegpu's scratch uses the driver pool, not torch's allocator."""
    return bool(_ALLOCATOR) and _ALLOCATOR[0] is None


def release_cached(min_free_bytes=48 << 30):
    """Return torch's cached free blocks to the driver when less than
    `min_free_bytes` of device memory is free (not while a graph is
    captured): libhegpu's scratch comes from the stream-ordered pool
    (cudaMallocAsync), which cannot reuse memory torch's allocator caches.
    Releasing unconditionally costs the next call its re-allocations."""
    if torch is None or not torch.cuda.is_available() or \
            torch.cuda.is_current_stream_capturing():
        return
    if torch.cuda.mem_get_info()[0] < min_free_bytes:
        torch.cuda.empty_cache()
