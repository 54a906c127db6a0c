"""Homomorphic operations (mirror of hebert/ckks/ops.py), GPU resident.

Level/scale bookkeeping is the reference's, statement for statement (float64
scales, the exact-1.0 alignment multiply, BSGS skip thresholds), so results
are bit-identical; the arithmetic underneath is libhegpu.  Ciphertexts are
stored packed: c0 and c1 are views of one (..., 2, level+1, N) tensor, so
whole-ciphertext kernels (rescale, automorphism) cover both components in a
single launch.  A Ciphertext may be batched (leading dimension B): every op
then processes all B ciphertexts per launch and key switches stream each key
once per batch.  Batched and unbatched operands broadcast (a shared weight
ciphertext against a batch of data ciphertexts).
"""

import contextlib
import logging
import math
import threading
from dataclasses import dataclass

import numpy as np
import torch

from .. import _dev
from .. import _lib
from .. import _stats
from .. import ring as rg
from ..errors import CryptoError, LevelMismatchError, OutOfLevelsError, ScaleMismatchError
from . import keys as keysmod
from .encoding import Plaintext, decode, decode_real, encode, encode_coeffs

log = logging.getLogger(__name__)

_mode = threading.local()


@contextlib.contextmanager
def fused_rescale(enabled=True):
    """Inside this context `mult(..., rescale_after=True)` relinearizes and
    rescales with ONE ModDown from the basis {q_level} + P
    (hegpu_ks_apply_rescale) instead of the reference's ModDown-then-rescale:
    same message and scale, limbs differ by the conversion rounding, and the
    separate rescale's INTT/NTT of every limb disappears.  The public API is
    reference-exact by default; the bootstrap and the trainer use this for
    their internal products (their results are tolerance-checked)."""
    prev = getattr(_mode, "fused", False)
    _mode.fused = enabled
    try:
        yield
    finally:
        _mode.fused = prev


def fused_rescale_enabled():
    return getattr(_mode, "fused", False)


SCALE_MATCH_RTOL = 2.0 ** -10
SCALE_EXACT_RTOL = 1e-9
_COEFF_SKIP_REL = 1e-13


@dataclass
class Ciphertext:
    """Pair of ring elements with level/scale/slot bookkeeping (ops.py:25-52).

    `insecure_provenance` is sticky: it marks anything that passed through
    the decrypt-reencrypt debug refresher.
    """

    c0: rg.RnsPoly
    c1: rg.RnsPoly
    scale: float
    slot_count: int
    params: object
    insecure_provenance: bool = False

    @property
    def level(self):
        return self.c0.level

    @property
    def batch(self):
        return self.c0.batch

    def copy(self):
        out = _packed(self.params, _lead(self), self.level)
        out[..., 0, :, :].copy_(self.c0.data)
        out[..., 1, :, :].copy_(self.c1.data)
        return _ct(out, self.level, self.scale, self.slot_count, self.params,
                   self.insecure_provenance)

    def __getitem__(self, i):
        """i-th ciphertext of a batch (a view)."""
        if self.batch is None:
            raise CryptoError("not a batched ciphertext")
        return Ciphertext(
            rg.RnsPoly(self.params.ring, self.c0.data[i], self.c0.form, self.level),
            rg.RnsPoly(self.params.ring, self.c1.data[i], self.c1.form, self.level),
            self.scale, self.slot_count, self.params, self.insecure_provenance,
        )

    def __len__(self):
        return 0 if self.batch is None else self.batch

    def narrow(self, lo, hi):
        """Batched view of ciphertexts lo..hi-1."""
        if self.batch is None:
            raise CryptoError("not a batched ciphertext")
        return Ciphertext(
            rg.RnsPoly(self.params.ring, self.c0.data[lo:hi], self.c0.form, self.level),
            rg.RnsPoly(self.params.ring, self.c1.data[lo:hi], self.c1.form, self.level),
            self.scale, self.slot_count, self.params, self.insecure_provenance,
        )


# ---------------------------------------------------------------------------
# packing helpers
# ---------------------------------------------------------------------------


def _lead(ct):
    return tuple(ct.c0.data.shape[:-2])


def _packed(params, lead, level):
    return _dev.empty(*(tuple(lead) + (2, level + 1, params.ring_degree)))


def _ct(t, level, scale, slot_count, params, insecure=False):
    ring = params.ring
    return Ciphertext(
        rg.RnsPoly(ring, t[..., 0, :, :], rg.EVAL, level),
        rg.RnsPoly(ring, t[..., 1, :, :], rg.EVAL, level),
        scale, slot_count, params, insecure,
    )


def _pair_group(ct):
    """(ptr, n_polys, stride) covering c0 and c1 of every batch element, if packed."""
    k = ct.level + 1
    n = ct.params.ring_degree
    p0, cnt, s0 = _dev.group(ct.c0.data, k, n)
    p1, _, s1 = _dev.group(ct.c1.data, k, n)
    if p1 - p0 != k * n * 8:
        return None
    if cnt > 1 and not (s0 == s1 == 2 * k * n):
        return None
    return p0, 2 * cnt, k * n


def _packed_view(ct):
    """The (lead..., 2, k, N) tensor holding c0 and c1 when they are packed
    back to back (one contiguous copy instead of two), else None."""
    if _pair_group(ct) is None:
        return None
    k = ct.level + 1
    n = ct.params.ring_degree
    lead = tuple(_lead(ct))
    if len(lead) > 1 or (lead and ct.c0.data.stride(0) != 2 * k * n):
        return None
    shape = lead + (2, k, n)
    stride = ((2 * k * n,) if lead else ()) + (k * n, n, 1)
    return ct.c0.data.as_strided(shape, stride)


def stack(cts):
    """Batch a list of same-level, same-scale ciphertexts into one (B, ...) ciphertext."""
    if not cts:
        raise CryptoError("cannot stack an empty list")
    first = cts[0]
    for c in cts[1:]:
        if c.level != first.level:
            raise LevelMismatchError("stacked ciphertexts must share a level")
        _check_scales(first.scale, c.scale)
    out = _packed(first.params, (len(cts),), first.level)
    for i, c in enumerate(cts):
        pv = _packed_view(c)
        if pv is not None:
            out[i].copy_(pv)
        else:
            out[i, 0].copy_(c.c0.data)
            out[i, 1].copy_(c.c1.data)
    return _ct(out, first.level, first.scale, first.slot_count, first.params,
               any(c.insecure_provenance for c in cts))


def unstack(ct):
    return [ct[i] for i in range(len(ct))]


def concat(cts):
    """Concatenate batched and/or single ciphertexts along the batch dimension."""
    parts = [c if c.batch is not None else stack([c]) for c in cts]
    first = parts[0]
    for c in parts[1:]:
        if c.level != first.level:
            raise LevelMismatchError("concatenated ciphertexts must share a level")
        _check_scales(first.scale, c.scale)
    total = sum(c.batch for c in parts)
    out = _packed(first.params, (total,), first.level)
    pos = 0
    for c in parts:
        pv = _packed_view(c)
        if pv is not None:
            out[pos : pos + c.batch].copy_(pv)
        else:
            out[pos : pos + c.batch, 0].copy_(c.c0.data)
            out[pos : pos + c.batch, 1].copy_(c.c1.data)
        pos += c.batch
    return _ct(out, first.level, first.scale, first.slot_count, first.params,
               any(c.insecure_provenance for c in parts))


def _ew_group(params, op, a_ptr, a_stride, b_ptr, b_stride, o_ptr, o_stride, cnt, k, consts=None):
    _lib.call(
        "hegpu_elementwise", params.ring.device(), op, a_ptr, a_stride, b_ptr, b_stride, o_ptr,
        o_stride, cnt, k, _dev.chain_primes(k).ctypes.data,
        None if consts is None else consts.ctypes.data, _dev.stream(),
    )


def _poly_binary(op, a, b, out_t):
    """out_t (tensor) = a op b with broadcasting of an unbatched operand."""
    rg._binary(op, a, b, out_t)


def _ct_scalar_op(ct, op, consts, both=True):
    """Per-limb scalar op on c0 (and c1) into a fresh packed ciphertext."""
    k = ct.level + 1
    n = ct.params.ring_degree
    out = _packed(ct.params, _lead(ct), ct.level)
    res = _ct(out, ct.level, ct.scale, ct.slot_count, ct.params, ct.insecure_provenance)
    grp = _pair_group(ct)
    if both and grp is not None:
        p, cnt, s = grp
        _ew_group(ct.params, op, p, s, None, 0, out.data_ptr(), k * n, cnt, k, consts)
        return res
    for src, dst, apply in ((ct.c0, res.c0, True), (ct.c1, res.c1, both)):
        sp, cnt, ss = src._group()
        dp, _, ds = dst._group()
        _ew_group(ct.params, op if apply else _lib.OP_COPY, sp, ss, None, 0, dp, ds, cnt, k,
                  consts if apply else None)
    return res


# ---------------------------------------------------------------------------
# encode / encrypt / decrypt
# ---------------------------------------------------------------------------


def encode_const(params, value, level, scale):
    """Constant plaintext without the FFT round (ops.py:55-66)."""
    scaled = float(value) * scale
    if abs(scaled) >= float(1 << 62):
        raise CryptoError("constant too large for the coefficient word")
    return Plaintext.constant(params, int(np.rint(scaled)), level, scale)


def encrypt(pt, keyset, target_level=None, rng_seed=None, min_circuit_level=None):
    """Public-key encryption at target_level (ops.py:69-123).

    The randomness v, e0, e1 is drawn on the host in the reference's order,
    so a seeded encryption is bit-identical; lifts, NTTs and the combine
    c0 = v*b + e0 + m, c1 = v*a + e1 run on the GPU.
    """
    params = pt._params
    level = pt.level if target_level is None else int(target_level)
    if level > params.max_level:
        raise CryptoError(f"target level {level} exceeds max {params.max_level}")
    if min_circuit_level is not None and level < min_circuit_level:
        log.warning(
            "encrypting at level %d below the declared circuit need %d; "
            "a refresh will be required before use", level, min_circuit_level,
        )
    if pt.level < level:
        raise CryptoError("plaintext level below requested ciphertext level")
    if rng_seed is None and DEVICE_UNSEEDED_RANDOMNESS:
        # the reference seeds numpy from OS entropy here (never reproducible):
        # expand 64 bits of OS entropy on the device instead of drawing and
        # uploading 3 N samples
        return _encrypt_from_samples(pt, keyset, level, device_samples(params))
    rng = np.random.default_rng(None if rng_seed is None else np.random.PCG64(rng_seed))
    ring = params.ring
    v = rg._sample_signed(ring, "ternary", rng)
    e0 = rg._sample_signed(ring, "discrete_gaussian", rng, sigma=params.error_sigma)
    e1 = rg._sample_signed(ring, "discrete_gaussian", rng, sigma=params.error_sigma)
    return _encrypt_from_samples(pt, keyset, level, np.stack([v, e0, e1]))


# unseeded encryptions draw v, e0, e1 on the device (hegpu_sample_encrypt);
# False restores the host numpy draws for them too
DEVICE_UNSEEDED_RANDOMNESS = True


def device_samples(params, seed=None):
    """(3, N) int64 device tensor: ternary v and rounded-Gaussian e0, e1
    (ring.py:499-509 distributions) expanded from a 64-bit seed (default:
    OS entropy) by the device Philox generator."""
    import os as _os

    n = params.ring_degree
    if seed is None:
        seed = int.from_bytes(_os.urandom(8), "little")
    out = _dev.empty(3, n)
    _lib.call("hegpu_sample_encrypt", out.data_ptr(), n, int(seed) & ((1 << 64) - 1),
              float(params.error_sigma), _dev.stream())
    return out


def _encrypt_from_samples(pt, keyset, level, samples):
    params = pt._params
    ring = params.ring
    n = params.ring_degree
    k = level + 1
    sel = _dev.chain_primes(k)
    dev_samples = samples if isinstance(samples, torch.Tensor) else _dev.to_device(samples)
    lifted = rg._lift_signed_dev(ring, dev_samples, sel)  # (3, k, N)
    rg._ntt_dev(ring, lifted, lifted, k, sel, False)
    b_full, a_full = keyset.public_key
    out = _packed(params, (), level)
    m = pt.poly.data[:k]
    _lib.call(
        "hegpu_encrypt_combine", ring.device(), lifted[0].data_ptr(), lifted[1].data_ptr(),
        lifted[2].data_ptr(), m.data_ptr(), b_full.data[:k].data_ptr(), a_full.data[:k].data_ptr(),
        out[0].data_ptr(), out[1].data_ptr(), k, _dev.stream(),
    )
    return _ct(out, level, pt.scale, params.slot_count, params)


def decrypt(ct, keyset):
    """m = c0 + c1*s (ops.py:126-133); batched ciphertexts decrypt together."""
    params = ct.params
    s = keyset.secret_at_level(ct.level)
    m = rg.poly_add(ct.c0, rg.poly_mul(ct.c1, s))
    pt = Plaintext(m, ct.scale)
    pt._params = params
    return pt


def decrypt_vector(ct, keyset, length=None):
    return decode_real(decrypt(ct, keyset), length)


def encrypt_vector(params, values, keyset, level=None, scale=None, rng_seed=None):
    level = params.max_level if level is None else level
    return encrypt(encode(params, values, level, scale), keyset, level, rng_seed)


# ---------------------------------------------------------------------------
# level management
# ---------------------------------------------------------------------------


def mod_down(ct, target_level):
    """Drop limbs to target_level; message and scale are preserved (ops.py:145-161)."""
    if target_level > ct.level:
        raise LevelMismatchError(
            f"mod_down target {target_level} above current level {ct.level}"
        )
    if target_level == ct.level:
        return ct
    k = target_level + 1
    out = _packed(ct.params, _lead(ct), target_level)
    out[..., 0, :, :].copy_(ct.c0.data[..., :k, :])
    out[..., 1, :, :].copy_(ct.c1.data[..., :k, :])
    return _ct(out, target_level, ct.scale, ct.slot_count, ct.params, ct.insecure_provenance)


def _rescale_polys(params, level, in_ptr, in_stride, out_ptr, out_stride, cnt):
    _stats.count("rescale_poly", level, cnt)
    _lib.call(
        "hegpu_rescale", params.ring.device(), level, in_ptr, in_stride, out_ptr, out_stride, cnt,
        _dev.stream(),
    )


def _poly_rescale(poly, params):
    """Divide by the top limb's prime with centered rounding; level - 1."""
    level = poly.level
    n = params.ring_degree
    out = _dev.empty(*(tuple(poly.data.shape[:-2]) + (level, n)))
    ip, cnt, is_ = poly._group()
    _rescale_polys(params, level, ip, is_, out.data_ptr(), level * n, cnt)
    return rg.RnsPoly(params.ring, out, rg.EVAL, level - 1)


def rescale(ct):
    """Divide the message scale by the dropped prime; consumes one level."""
    if ct.level == 0:
        raise OutOfLevelsError("rescale at level 0")
    params = ct.params
    q_l = params.ring.moduli_chain[ct.level]
    n = params.ring_degree
    out = _packed(params, _lead(ct), ct.level - 1)
    res = _ct(out, ct.level - 1, ct.scale / q_l, ct.slot_count, params, ct.insecure_provenance)
    grp = _pair_group(ct)
    if grp is not None:
        p, cnt, s = grp
        _rescale_polys(params, ct.level, p, s, out.data_ptr(), ct.level * n, cnt)
    else:
        for src, dst in ((ct.c0, res.c0), (ct.c1, res.c1)):
            sp, cnt, ss = rg.to_eval(src)._group()
            dp, _, ds = dst._group()
            _rescale_polys(params, ct.level, sp, ss, dp, ds, cnt)
    return res


def _align(ct1, ct2):
    """Equalize levels and (where a spare level allows) scales exactly (ops.py:210-231)."""
    s1, s2 = ct1.scale, ct2.scale
    if ct1.level == ct2.level and abs(s1 - s2) <= SCALE_EXACT_RTOL * max(s1, s2):
        return ct1, ct2
    hi, lo = (ct1, ct2) if ct1.level >= ct2.level else (ct2, ct1)
    if hi.level > lo.level and abs(hi.scale - lo.scale) > SCALE_EXACT_RTOL * lo.scale:
        hi = mod_down(hi, lo.level + 1)
        q = hi.params.ring.moduli_chain[hi.level]
        pt = encode_const(hi.params, 1.0, hi.level, lo.scale * q / hi.scale)
        hi = mult_plain(hi, pt)
        hi.scale = lo.scale
    else:
        hi = mod_down(hi, lo.level)
    return (hi, lo) if ct1.level >= ct2.level else (lo, hi)


def _check_scales(s1, s2):
    if abs(s1 - s2) > SCALE_MATCH_RTOL * max(s1, s2):
        raise ScaleMismatchError(f"scales differ beyond 2^-10: {s1} vs {s2}")


def _combine(op, ct1, ct2):
    lead = _lead(ct1) if len(_lead(ct1)) >= len(_lead(ct2)) else _lead(ct2)
    out = _packed(ct1.params, lead, ct1.level)
    res = _ct(out, ct1.level, ct1.scale, ct1.slot_count, ct1.params,
              ct1.insecure_provenance or ct2.insecure_provenance)
    g1, g2 = _pair_group(ct1), _pair_group(ct2)
    if g1 is not None and g2 is not None and g1[1] == g2[1]:
        k = ct1.level + 1
        n = ct1.params.ring_degree
        _ew_group(ct1.params, op, g1[0], g1[2], g2[0], g2[2], out.data_ptr(), k * n, g1[1], k)
        return res
    _poly_binary(op, ct1.c0, ct2.c0, res.c0.data)
    _poly_binary(op, ct1.c1, ct2.c1, res.c1.data)
    return res


def add(ct1, ct2):
    """Slot-wise sum; the higher-level operand is mod-downed automatically."""
    ct1, ct2 = _align(ct1, ct2)
    _check_scales(ct1.scale, ct2.scale)
    return _combine(_lib.OP_ADD, ct1, ct2)


def sub(ct1, ct2):
    ct1, ct2 = _align(ct1, ct2)
    _check_scales(ct1.scale, ct2.scale)
    if ct1.batch is None and ct2.batch is not None:
        return add(negate(ct2), ct1)
    return _combine(_lib.OP_SUB, ct1, ct2)


def negate(ct):
    return _ct_scalar_op(ct, _lib.OP_NEG, None)


# ---------------------------------------------------------------------------
# plaintext operations
# ---------------------------------------------------------------------------


def _as_plaintext(ct, values_or_pt, scale=None):
    if isinstance(values_or_pt, Plaintext):
        return values_or_pt
    if np.isscalar(values_or_pt):
        return encode_const(
            ct.params, values_or_pt, ct.level, scale if scale else ct.params.default_scale
        )
    return encode(ct.params, values_or_pt, ct.level, scale if scale else ct.params.default_scale)


def add_plain(ct, values_or_pt):
    """ct + plaintext; the plaintext is encoded at the ciphertext's scale (ops.py:277-304)."""
    if isinstance(values_or_pt, Plaintext):
        pt = values_or_pt
        _check_scales(ct.scale, pt.scale)
    elif np.isscalar(values_or_pt):
        pt = encode_const(ct.params, values_or_pt, ct.level, ct.scale)
    else:
        pt = encode(ct.params, values_or_pt, ct.level, ct.scale)
    k = ct.level + 1
    if pt.level < ct.level:
        raise LevelMismatchError("plaintext level below ciphertext level")
    cres = pt.const_residues(k)
    if cres is not None:
        # constant in every slot: c0 + c, c1 copied
        return _ct_scalar_op(ct, _lib.OP_ADDC, cres, both=False)
    ppoly = rg.RnsPoly(ct.params.ring, pt.poly.data[:k], rg.EVAL, ct.level)
    out = _packed(ct.params, _lead(ct), ct.level)
    res = _ct(out, ct.level, ct.scale, ct.slot_count, ct.params, ct.insecure_provenance)
    _poly_binary(_lib.OP_ADD, ct.c0, ppoly, res.c0.data)
    res.c1.data.copy_(ct.c1.data)
    return res


def sub_plain(ct, values_or_pt):
    neg = values_or_pt
    if isinstance(values_or_pt, Plaintext):
        p = values_or_pt
        cres = p.const_residues(p.level + 1)
        if cres is not None:
            neg = Plaintext.constant(p._params, -p._const[0], p._const[1], p.scale)
        else:
            neg = Plaintext(rg.poly_neg(p.poly), p.scale)
            neg._params = p._params
    elif np.isscalar(values_or_pt):
        neg = -values_or_pt
    else:
        neg = -np.asarray(values_or_pt)
    return add_plain(ct, neg)


def mult_plain(ct, values_or_pt, rescale_after=True):
    """Slot-wise product with a plaintext, rescaled back to ~default scale (ops.py:323-343)."""
    if ct.level == 0:
        raise OutOfLevelsError("mult_plain at level 0")
    pt = _as_plaintext(ct, values_or_pt)
    if pt.level < ct.level:
        raise LevelMismatchError("plaintext level below ciphertext level")
    k = ct.level + 1
    cres = pt.const_residues(k)
    if cres is not None:
        out = _ct_scalar_op(ct, _lib.OP_SCALAR, cres)
        out.scale = ct.scale * pt.scale
    else:
        ppoly = rg.RnsPoly(ct.params.ring, pt.poly.data[:k], rg.EVAL, ct.level)
        t = _packed(ct.params, _lead(ct), ct.level)
        out = _ct(t, ct.level, ct.scale * pt.scale, ct.slot_count, ct.params,
                  ct.insecure_provenance)
        grp = _pair_group(ct)
        if grp is not None:
            n = ct.params.ring_degree
            p, cnt, s = grp
            _ew_group(ct.params, _lib.OP_MUL, p, s, ppoly.data.data_ptr(), 0, t.data_ptr(), k * n,
                      cnt, k)
        else:
            _poly_binary(_lib.OP_MUL, ct.c0, ppoly, out.c0.data)
            _poly_binary(_lib.OP_MUL, ct.c1, ppoly, out.c1.data)
    return rescale(out) if rescale_after else out


# ---------------------------------------------------------------------------
# key-switched operations
# ---------------------------------------------------------------------------


def _tensor(ct1, ct2):
    """(d0, d1, d2) packed as (..., 3, k, N)."""
    params = ct1.params
    k = ct1.level + 1
    n = params.ring_degree
    a0p, acnt, as_ = ct1.c0._group()
    a1p, _, _ = ct1.c1._group()
    b0p, bcnt, bs = ct2.c0._group()
    b1p, _, _ = ct2.c1._group()
    cnt = max(acnt, bcnt)
    period = cnt
    if acnt == 1 and cnt > 1:  # the product is symmetric: put the batch first
        a0p, a1p, as_, b0p, b1p, bs = b0p, b1p, bs, a0p, a1p, 0
    elif bcnt == 1 and cnt > 1:
        bs = 0
    elif acnt != bcnt:
        # one batch against several stacked copies of its shape: the smaller
        # operand repeats with period min(acnt, bcnt) (level-batched polynomial
        # evaluation multiplies one giant power by every node of a level)
        lo_cnt, hi_cnt = min(acnt, bcnt), max(acnt, bcnt)
        if hi_cnt % lo_cnt:
            raise CryptoError("batch size mismatch")
        if bcnt < acnt:
            a0p, a1p, as_, b0p, b1p, bs = b0p, b1p, bs, a0p, a1p, as_
        period = lo_cnt
    lead = _lead(ct1) if acnt >= bcnt else _lead(ct2)
    d = _dev.empty(*(tuple(lead) + (3, k, n)))
    _lib.call(
        "hegpu_tensor_periodic", params.ring.device(), a0p, a1p, as_, period, b0p, b1p, bs,
        d[..., 0, :, :].data_ptr(), d[..., 1, :, :].data_ptr(), d[..., 2, :, :].data_ptr(),
        3 * k * n, cnt, k, _dev.stream(),
    )
    return d


def mult(ct1, ct2, relin_key_or_keyset, rescale_after=True):
    """Slot-wise ciphertext product with relinearization and rescale (ops.py:346-367)."""
    keyset = relin_key_or_keyset
    if not isinstance(keyset, keysmod.KeySet):
        raise CryptoError("mult needs the KeySet (for the KS precompute cache)")
    ct1, ct2 = _align(ct1, ct2)
    if ct1.level == 0:
        raise OutOfLevelsError("mult at level 0")
    params = ct1.params
    level = ct1.level
    d = _tensor(ct1, ct2)  # (..., 3, k, N): d0, d1, d2
    ring = params.ring
    k = level + 1
    n = params.ring_degree
    d2 = rg.RnsPoly(ring, d[..., 2, :, :], rg.EVAL, level)
    if rescale_after and fused_rescale_enabled():
        out = _packed(params, tuple(d.shape[:-3]), level - 1)
        dp, cnt, ds = d2._group()
        kb, ka = keyset.relin_key.ptr_arrays()
        _stats.count("ks", level, cnt)
        _stats.count("rescale_poly", level, 2 * cnt)
        _lib.call(
            "hegpu_ks_apply_rescale", ring.device(), level, params.digit_size, dp, ds, cnt, kb, ka,
            keyset.relin_key.dnum, d.data_ptr(), 3 * k * n, k * n, out.data_ptr(),
            2 * level * n, level * n, _dev.stream(),
        )
        q_l = ring.moduli_chain[level]
        return _ct(out, level - 1, ct1.scale * ct2.scale / q_l, ct1.slot_count, params,
                   ct1.insecure_provenance or ct2.insecure_provenance)
    # (d0, d1) += KS(d2): the ModDown epilogue accumulates in place
    keysmod.ks_apply_into(keyset, keyset.relin_key, d2, d[..., 0, :, :].data_ptr(),
                          d[..., 1, :, :].data_ptr(), 3 * k * n, 3)
    res = Ciphertext(
        rg.RnsPoly(ring, d[..., 0, :, :], rg.EVAL, level),
        rg.RnsPoly(ring, d[..., 1, :, :], rg.EVAL, level),
        ct1.scale * ct2.scale, ct1.slot_count, params,
        ct1.insecure_provenance or ct2.insecure_provenance,
    )
    return rescale(res) if rescale_after else res


def square(ct, keyset, rescale_after=True):
    return mult(ct, ct, keyset, rescale_after)


def _automorph_ct(ct, g):
    """Both components through X -> X^g (eval form), packed output."""
    params = ct.params
    k = ct.level + 1
    n = params.ring_degree
    out = _packed(params, _lead(ct), ct.level)
    res = _ct(out, ct.level, ct.scale, ct.slot_count, params, ct.insecure_provenance)
    grp = _pair_group(ct)
    if grp is not None:
        p, cnt, s = grp
        _lib.call(
            "hegpu_automorphism", params.ring.device(), 1, g % (2 * n), p, s, out.data_ptr(),
            k * n, cnt, k, _dev.chain_primes(k).ctypes.data, _dev.stream(),
        )
    else:
        res.c0.data.copy_(rg.poly_automorphism_eval(rg.to_eval(ct.c0), g).data)
        res.c1.data.copy_(rg.poly_automorphism_eval(rg.to_eval(ct.c1), g).data)
    return res


def _switch_after_automorph(ct, g, key, keyset):
    """(c0∘σ + KS(c1∘σ).b, KS(c1∘σ).a) (ops.py:374-388 / :401-416); the b half
    is accumulated into c0∘σ and the a half overwrites c1∘σ in place."""
    r = _automorph_ct(ct, g)
    k = ct.level + 1
    n = ct.params.ring_degree
    keysmod.ks_apply_into(keyset, key, r.c1, r.c0.data.data_ptr(), r.c1.data.data_ptr(),
                          2 * k * n, 1)
    return r


def _rotate_once(ct, step, keyset):
    params = ct.params
    g = keysmod.galois_exponent_for_step(params, step)
    key = keysmod.rotation_key_for(keyset, step)
    return _switch_after_automorph(ct, g, key, keyset)


def rotate(ct, step, keyset):
    """Cyclic left shift of the slot vector by `step` (negative = right)."""
    step = int(step) % ct.slot_count
    if step == 0:
        return ct.copy()
    for part in keysmod.decompose_rotation(keyset, step, ct.slot_count):
        ct = _rotate_once(ct, part, keyset)
    return ct


def rotate_hoisted(ct, steps, keyset):
    """Rotations of one (batched) ciphertext by several keyed steps sharing
    one ModUp of c1 (hoisting).  Each output decrypts like `rotate(ct, s)`;
    its limbs are not bit-identical to it (see hegpu_ks_hoisted), so the
    public `rotate` keeps the reference's per-rotation key switch.  Used for
    the bootstrap's baby steps.  Step 0 returns ct itself."""
    import ctypes

    params = ct.params
    n = params.ring_degree
    k = ct.level + 1
    out = {}
    todo = []
    for s in steps:
        s = int(s) % ct.slot_count
        if s == 0:
            out[0] = ct
        elif s in keyset.rotation_keys or s - ct.slot_count in keyset.rotation_keys:
            todo.append(s)
        else:
            out[s] = rotate(ct, s, keyset)
    if not todo:
        return [out[int(s) % ct.slot_count] for s in steps]
    src = ct if _pair_group(ct) is not None else ct.copy()
    cnt = 1 if src.batch is None else src.batch
    keys = [keysmod.rotation_key_for(keyset, s if s in keyset.rotation_keys else s - ct.slot_count)
            for s in todo]
    dnum = keys[0].dnum
    gal = np.array([keysmod.galois_exponent_for_step(params, s) % (2 * n) for s in todo],
                   dtype=np.uint64)
    kb = (ctypes.c_void_p * (len(todo) * dnum))(
        *[kk.b[j].data_ptr() for kk in keys for j in range(dnum)])
    ka = (ctypes.c_void_p * (len(todo) * dnum))(
        *[kk.a[j].data_ptr() for kk in keys for j in range(dnum)])
    # one tensor, rotation-major: the library batches the ModDowns of all rotations
    allout = _dev.empty(*((len(todo),) + tuple(_lead(ct)) + (2, k, n)))
    outs = [allout[i] for i in range(len(todo))]
    optr = (ctypes.c_void_p * len(todo))(*[o.data_ptr() for o in outs])
    for _ in todo:
        _stats.count("ks", ct.level, cnt)
    _lib.call(
        "hegpu_ks_hoisted", params.ring.device(), ct.level, params.digit_size,
        src.c0.data.data_ptr(), 2 * k * n, k * n, cnt, len(todo), gal.ctypes.data, kb, ka, dnum,
        optr, 0, _dev.stream(),
    )
    for s, o in zip(todo, outs):
        out[s] = _ct(o, ct.level, ct.scale, ct.slot_count, params, ct.insecure_provenance)
    return [out[int(s) % ct.slot_count] for s in steps]


def p_mod_chain(params, k):
    """P mod q_i (P = product of the special primes) for chain limbs i < k."""
    p = 1
    for s in params.ring.special_moduli:
        p *= int(s)
    return np.array([p % int(q) for q in params.ring.moduli_chain[:k]], dtype=np.uint64)


def to_extended(ct):
    """P-scaled extended-basis copy of ct: (P c0, P c1) on the chain limbs and
    0 on the special limbs, packed (..., 2, level+1+K, N) -- the form of a
    double-hoisted rotation by 0."""
    params = ct.params
    k = ct.level + 1
    n = params.ring_degree
    K = len(params.ring.special_moduli)
    src = ct if _pair_group(ct) is not None else ct.copy()
    cnt = 1 if src.batch is None else src.batch
    out = _dev.zeros(*(tuple(_lead(ct)) + (2, k + K, n)))
    _ew_group(params, _lib.OP_SCALAR, src.c0.data.data_ptr(), k * n, None, 0, out.data_ptr(),
              (k + K) * n, 2 * cnt, k, p_mod_chain(params, k))
    return out


def rotate_hoisted_ext(ct, steps, keyset):
    """Double-hoisted rotations: one ModUp, then every rotation's inner
    product stays in the extended basis (no ModDown): returns a packed
    (len(steps), ..., 2, level+1+K, N) tensor of P-scaled rotations
    (hegpu_ks_hoisted with pq_out).  Steps must be keyed (or 0)."""
    import ctypes

    params = ct.params
    n = params.ring_degree
    k = ct.level + 1
    K = len(params.ring.special_moduli)
    src = ct if _pair_group(ct) is not None else ct.copy()
    cnt = 1 if src.batch is None else src.batch
    steps = [int(s) % ct.slot_count for s in steps]
    out = _dev.empty(*((len(steps),) + tuple(_lead(ct)) + (2, k + K, n)))
    todo = [i for i, s in enumerate(steps) if s]
    for i, s in enumerate(steps):
        if not s:
            out[i].copy_(to_extended(ct))
    if not todo:
        return out
    if not can_rotate_sum(keyset, [steps[i] for i in todo], ct.slot_count):
        raise CryptoError("double-hoisted rotations need a key for every step")
    keys = [keysmod.rotation_key_for(keyset, steps[i] if steps[i] in keyset.rotation_keys
                                     else steps[i] - ct.slot_count) for i in todo]
    dnum = keys[0].dnum
    gal = np.array([keysmod.galois_exponent_for_step(params, steps[i]) % (2 * n) for i in todo],
                   dtype=np.uint64)
    kb = (ctypes.c_void_p * (len(todo) * dnum))(
        *[kk.b[j].data_ptr() for kk in keys for j in range(dnum)])
    ka = (ctypes.c_void_p * (len(todo) * dnum))(
        *[kk.a[j].data_ptr() for kk in keys for j in range(dnum)])
    # the rotated outputs must be packed back to back: a contiguous run of
    # nonzero steps (e.g. babies 1..n1-1 after step 0) is computed in place;
    # otherwise into a dense block that is scattered afterwards
    if todo == list(range(todo[0], todo[0] + len(todo))):
        block = out[todo[0]: todo[0] + len(todo)]
    else:
        block = _dev.empty(*((len(todo),) + tuple(_lead(ct)) + (2, k + K, n)))
    optr = (ctypes.c_void_p * len(todo))(*[block[i].data_ptr() for i in range(len(todo))])
    for _ in todo:
        _stats.count("ks", ct.level, cnt)
    _lib.call(
        "hegpu_ks_hoisted", params.ring.device(), ct.level, params.digit_size,
        src.c0.data.data_ptr(), 2 * k * n, k * n, cnt, len(todo), gal.ctypes.data, kb, ka, dnum,
        optr, 1, _dev.stream(),
    )
    if block.data_ptr() != out[todo[0]].data_ptr():
        for j, i in enumerate(todo):
            out[i].copy_(block[j])
    return out


def _keyed(keyset, s, slot_count):
    return s in keyset.rotation_keys or s - slot_count in keyset.rotation_keys


def can_rotate_sum(keyset, steps, slot_count):
    return all(_keyed(keyset, int(s) % slot_count, slot_count) for s in steps
               if int(s) % slot_count)


def rotate_sum(ct, steps, keyset):
    """ct + sum_s rotate(ct, s) with ONE ModUp and ONE ModDown
    (hegpu_ks_rotsum): the rotations' inner products accumulate in the
    extended basis.  Decrypts like the sequential rotate-and-add (the
    reference's loops, logreg.py:202-229); limbs differ.  Every nonzero step
    must have its own rotation key (can_rotate_sum)."""
    import ctypes

    params = ct.params
    n = params.ring_degree
    k = ct.level + 1
    todo = [int(s) % ct.slot_count for s in steps]
    zeros = sum(1 for s in todo if s == 0)
    todo = [s for s in todo if s]
    if not can_rotate_sum(keyset, todo, ct.slot_count):
        raise CryptoError("rotate_sum needs a rotation key for every step")
    src = ct if _pair_group(ct) is not None else ct.copy()
    cnt = 1 if src.batch is None else src.batch
    out = _packed(params, _lead(ct), ct.level)
    if todo:
        keys = [keysmod.rotation_key_for(keyset, s if s in keyset.rotation_keys
                                         else s - ct.slot_count) for s in todo]
        dnum = keys[0].dnum
        gal = np.array([keysmod.galois_exponent_for_step(params, s) % (2 * n) for s in todo],
                       dtype=np.uint64)
        kb = (ctypes.c_void_p * (len(todo) * dnum))(
            *[kk.b[j].data_ptr() for kk in keys for j in range(dnum)])
        ka = (ctypes.c_void_p * (len(todo) * dnum))(
            *[kk.a[j].data_ptr() for kk in keys for j in range(dnum)])
        for _ in todo:
            _stats.count("ks", ct.level, cnt)
    else:
        gal, kb, ka, dnum = np.zeros(1, dtype=np.uint64), None, None, 1
    _lib.call(
        "hegpu_ks_rotsum", params.ring.device(), ct.level, params.digit_size,
        src.c0.data.data_ptr(), 2 * k * n, k * n, cnt, len(todo), gal.ctypes.data, kb, ka, dnum,
        out.data_ptr(), 2 * k * n, k * n, _dev.stream(),
    )
    res = _ct(out, ct.level, ct.scale, ct.slot_count, params, ct.insecure_provenance)
    for _ in range(zeros):  # rotation by 0 adds ct itself
        res = add(res, ct)
    return res


def conjugate(ct, keyset):
    if keyset.conj_key is None:
        raise CryptoError("key set has no conjugation key")
    n = ct.params.ring_degree
    return _switch_after_automorph(ct, 2 * n - 1, keyset.conj_key, keyset)


# ---------------------------------------------------------------------------
# Chebyshev-basis polynomial evaluation (ops.py:424-506)
# ---------------------------------------------------------------------------


def bsgs_depth(degree, prescaled=False):
    """Levels consumed: ceil(log2(degree+1)) plus one for the domain affine."""
    return math.ceil(math.log2(degree + 1)) + (0 if prescaled else 1)


def eval_poly_bsgs(ct, poly, keyset, input_prescaled=False):
    """Apply a Chebyshev-basis polynomial slot-wise (divide and conquer over
    power-of-two giants T_{2^i}; the reference's recursion and skip rules,
    ops.py:432-506, so the op sequence and results are identical)."""
    degree = poly.degree
    need = bsgs_depth(degree, input_prescaled)
    if ct.level < need:
        raise OutOfLevelsError(f"polynomial evaluation needs {need} levels, have {ct.level}")
    coeffs = np.asarray(poly.cheb_coeffs, dtype=np.float64)

    if input_prescaled:
        y = ct
    else:
        a, b = poly.domain
        y = mult_plain(ct, 2.0 / (b - a))
        shift = -(a + b) / (b - a)
        if abs(shift) > 0:
            y = add_plain(y, shift)
    if degree == 0:
        return add_plain(mult_plain(y, 0.0), float(coeffs[0]))

    skip = _COEFF_SKIP_REL * float(np.max(np.abs(coeffs)))

    giants = {1: y}
    g = 1
    while 2 * g <= degree:
        sq = square(giants[g], keyset)
        giants[2 * g] = add_plain(add(sq, sq), -1.0)
        g *= 2

    # The reference's recursion (ops.py:432-506) is planned first and then run
    # level by level: every leaf's scalar product shares one rescale launch and
    # all products of one giant power share one key switch.  Each op sees the
    # same operands as in the recursive order, so the limbs are identical.
    def plan(c):
        d = len(c) - 1
        while d > 0 and abs(c[d]) <= skip:
            d -= 1
        if d == 0:
            return ["const", float(c[0])]
        if d == 1:
            return ["leaf", float(c[0]), float(c[1])]
        g = 1 << (math.ceil(math.log2(d + 1)) - 1)
        r = np.zeros(d - g + 1)
        r[0] = c[g]
        r[1:] = 2.0 * c[g + 1 : d + 1]
        q = c[:g].copy()
        for j in range(1, d - g + 1):
            q[g - j] -= c[g + j]
        return ["node", g, plan(r), plan(q)]

    root = plan(coeffs.copy())
    leaves, nodes = [], []

    def walk(t):
        if t[0] == "leaf":
            leaves.append(t)
        elif t[0] == "node":
            walk(t[2])
            walk(t[3])
            nodes.append(t)

    walk(root)
    values = {}

    def value(t):
        return t[1] if t[0] == "const" else values[id(t)]

    if leaves:
        cat = _scalar_products(giants[1], [lf[2] for lf in leaves])
        if cat is None:
            cat = _cat_batch([mult_plain(giants[1], lf[2], rescale_after=False) for lf in leaves])
        for lf, v in zip(leaves, _split_batch(rescale(cat), len(leaves), y)):
            values[id(lf)] = add_plain(v, lf[1])
    for g in sorted({t[1] for t in nodes}):
        level_nodes = [t for t in nodes if t[1] == g]
        groups = {}
        for t in level_nodes:
            r_val = value(t[2])
            if not isinstance(r_val, float):
                groups.setdefault((r_val.level, r_val.scale), []).append(t)
        terms = {}
        for members in groups.values():
            operands = [value(t[2]) for t in members]
            prod = mult(giants[g], _cat_batch(operands), keyset)
            for t, v in zip(members, _split_batch(prod, len(members), y)):
                terms[id(t)] = v
        adds = {}
        for t in level_nodes:
            r_val, q_val = value(t[2]), value(t[3])
            if isinstance(r_val, float):
                term = None if abs(r_val) <= skip else mult_plain(giants[g], r_val)
            else:
                term = terms[id(t)]
            if term is None:
                values[id(t)] = q_val
            elif isinstance(q_val, float):
                values[id(t)] = add_plain(term, q_val) if q_val else term
            else:  # batched below: the level alignment of q_val is shared
                key = (term.level, term.scale, q_val.level, q_val.scale)
                adds.setdefault(key, []).append((t, term, q_val))
        for members in adds.values():
            summed = add(_cat_batch([m[1] for m in members]),
                         _cat_batch([m[2] for m in members]))
            for m, v in zip(members, _split_batch(summed, len(members), y)):
                values[id(m[0])] = v

    result = value(root)
    if isinstance(result, float):
        result = add_plain(mult_plain(y, 0.0), result)
    return result


def _scalar_products(ct, scalars):
    """_cat_batch([mult_plain(ct, c, rescale_after=False) for c in scalars])
    written straight into one packed batch (same scalar launches, no gather
    copy); None when a scalar does not encode as a constant."""
    if len(scalars) < 2 or _pair_group(ct) is None or len(_lead(ct)) > 1:
        return None
    k = ct.level + 1
    n = ct.params.ring_degree
    pts = [_as_plaintext(ct, float(c)) for c in scalars]
    cres = [pt.const_residues(k) for pt in pts]
    if any(c is None for c in cres) or len({pt.scale for pt in pts}) != 1:
        return None
    b = _lead(ct)[0] if _lead(ct) else 1
    t = _dev.empty(len(scalars) * b, 2, k, n)
    p, cnt, stride = _pair_group(ct)
    for i, c in enumerate(cres):
        _ew_group(ct.params, _lib.OP_SCALAR, p, stride, None, 0, t[i * b].data_ptr(), k * n, cnt,
                  k, c)
    if not _lead(ct):
        t = t.view(len(scalars), 2, k, n)
    return _ct(t, ct.level, ct.scale * pts[0].scale, ct.slot_count, ct.params,
               ct.insecure_provenance)


def _cat_batch(cts):
    """Stack same-shape ciphertexts (each unbatched or with batch B) into one
    batch of len(cts) (or len(cts) * B); a single one passes through.  Parts
    that already sit back to back in one packed tensor (the slices
    _split_batch made of an earlier batched result, in order) are returned as
    a view of it instead of copied (read-only use inside eval_poly_bsgs)."""
    if len(cts) == 1:
        return cts[0]
    view = _adjacent_view(cts)
    if view is not None:
        first = cts[0]
        return _ct(view, first.level, first.scale, first.slot_count, first.params,
                   any(c.insecure_provenance for c in cts))
    if cts[0].batch is None:
        return stack(cts)
    return concat(cts)


def _adjacent_view(cts):
    """(total, 2, k, N) view over ciphertexts packed consecutively in memory
    with the same level and scale, else None."""
    first = cts[0]
    views = []
    for c in cts:
        if c.level != first.level or c.scale != first.scale:
            return None
        v = _packed_view(c)
        if v is None:
            return None
        views.append(v)
    ptr = views[0].data_ptr()
    base = views[0].untyped_storage().data_ptr()
    for v in views:  # same allocation (adjacent allocations do not count)
        if v.data_ptr() != ptr or v.untyped_storage().data_ptr() != base:
            return None
        ptr += v.numel() * v.element_size()
    k, n = first.level + 1, first.params.ring_degree
    total = sum(1 if c.batch is None else c.batch for c in cts)
    return views[0].as_strided((total, 2, k, n), (2 * k * n, k * n, n, 1))


def _split_batch(ct, n, like):
    """Inverse of _cat_batch for n parts shaped like `like`."""
    if n == 1:
        return [ct]
    if like.batch is None:
        return [ct[i] for i in range(n)]
    b = like.batch
    return [ct.narrow(i * b, (i + 1) * b) for i in range(n)]
