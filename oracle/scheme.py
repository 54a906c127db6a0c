"""TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference CKKS scheme.

Follows /root/reference/pkg/src/hebert step by step on host numpy arrays:
ring tables (ring.py:60-128), RNS polynomial arithmetic (ring.py:287-482),
encoding (ckks/encoding.py:17-143), key generation (ckks/keys.py:103-249),
hybrid key switching (ckks/keys.py:19-49, 264-339), encryption/decryption,
rescale, alignment, products and rotations (ckks/ops.py:55-416) and ModRaise
(bootstrap.py:260-275).  Kernels come from oracle.kernels.  Pinned against
the reference's own outputs by tests/test_oracle_golden.py.
"""

import hashlib
import math

import numpy as np

from . import kernels as K

# ---------------------------------------------------------------------------
# parameters (ckks/params.py:59-96)
# ---------------------------------------------------------------------------


class Params:
    def __init__(self, n, chain, special, scale, dnum, hamming, sigma, text=None):
        self.n = n
        self.chain = tuple(chain)
        self.special = tuple(special)
        self.scale = scale
        self.dnum = dnum
        self.hamming = hamming
        self.sigma = sigma
        self.text = text
        self._tabs = {}

    @classmethod
    def from_text(cls, text):
        lines = [ln.strip() for ln in text.strip().splitlines()
                 if ln.strip() and not ln.startswith("#")]
        f = {}
        for ln in lines[1:]:
            key, _, rest = ln.partition(" ")
            f.setdefault(key, rest.strip())
        hw = int(f["secret_hamming_weight"])
        return cls(int(f["N"]), [int(x, 16) for x in f["moduli"].split()],
                   [int(x, 16) for x in f.get("special", "").split()],
                   float.fromhex(f["scale"]), int(f["dnum"]), hw or None,
                   float.fromhex(f["error_sigma"]), text)

    @property
    def max_level(self):
        return len(self.chain) - 1

    @property
    def slots(self):
        return self.n // 2

    @property
    def digit_size(self):
        return -(-(self.max_level + 1) // self.dnum)

    def digit_groups(self, level):
        idx = list(range(level + 1))
        sz = self.digit_size
        return [idx[i : i + sz] for i in range(0, len(idx), sz)]

    @property
    def ext(self):
        return self.chain + self.special

    # -- per-prime tables (ring.py:81-108) --------------------------------
    def table(self, q):
        t = self._tabs.get(q)
        if t is None:
            t = _PrimeTab(q, self.n)
            self._tabs[q] = t
        return t

    def stack(self, primes):
        key = ("stack",) + tuple(primes)
        s = self._tabs.get(key)
        if s is None:
            tabs = [self.table(q) for q in primes]
            s = {
                "q": np.array(primes, dtype=np.uint64),
                "qinv": np.array([t.qinv for t in tabs], dtype=np.uint64),
                "r2": np.array([t.r2 for t in tabs], dtype=np.uint64),
                "ninv": np.array([t.ninv for t in tabs], dtype=np.uint64),
                "psi": np.stack([t.psi_rev for t in tabs]),
                "ipsi": np.stack([t.ipsi_rev for t in tabs]),
            }
            self._tabs[key] = s
        return s


def find_psi(q, two_n):
    """First base in [2, 10^4) with an order-2N power (ring.py:69-78)."""
    e = (q - 1) // two_n
    for base in range(2, 10000):
        cand = pow(base, e, q)
        if pow(cand, two_n // 2, q) == q - 1:
            return cand
    raise ValueError("no primitive root")


def bitrev(n):
    bits = n.bit_length() - 1
    idx = np.arange(n)
    rev = np.zeros(n, dtype=np.int64)
    for b in range(bits):
        rev |= ((idx >> b) & 1) << (bits - 1 - b)
    return rev


class _PrimeTab:
    def __init__(self, q, n):
        self.q = q
        self.qinv = (-pow(q, -1, 1 << 64)) % (1 << 64)
        r = (1 << 64) % q
        self.r = r
        self.r2 = r * r % q
        psi = find_psi(q, 2 * n)
        rev = bitrev(n)
        self.psi_rev = _mont_powers(psi, r, q, n)[rev].copy()
        self.ipsi_rev = _mont_powers(pow(psi, -1, q), r, q, n)[rev].copy()
        self.ninv = pow(n, -1, q) * r % q


def _mont_powers(base, r, q, n):
    """[base^i * R mod q for i < n] (Montgomery form, ring.py:96-105)."""
    out = np.empty(n, dtype=np.uint64)
    out[0] = r % q
    qq = np.uint64(q)
    qinv = np.uint64((-pow(q, -1, 1 << 64)) % (1 << 64))
    span = 1
    bp = base % q
    while span < n:
        step = min(span, n - span)
        # out[span+i] = out[i] * base^span: mont(out[i], base^span R) stays in Montgomery form
        bs_r = np.uint64(pow(bp, span, q) * r % q)
        out[span : span + step] = K.mont(out[:step], bs_r, qq, qinv)
        span += step
    return out


# ---------------------------------------------------------------------------
# ring operations on (k, N) limb arrays
# ---------------------------------------------------------------------------


def ntt_fwd(p, limbs, primes):
    s = p.stack(primes)
    a = np.ascontiguousarray(limbs, dtype=np.uint64).copy()
    return K.ntt_forward_inplace(a, s["psi"], s["q"], s["qinv"])


def ntt_inv(p, limbs, primes):
    s = p.stack(primes)
    a = np.ascontiguousarray(limbs, dtype=np.uint64).copy()
    return K.ntt_inverse_inplace(a, s["ipsi"], s["ninv"], s["q"], s["qinv"])


def mul(p, a, b, primes):
    s = p.stack(primes)
    return K.elementwise_mulmod(a, b, s["q"], s["qinv"], s["r2"])


def add(p, a, b, primes):
    return K.addmod_rows(a, b, np.array(primes, dtype=np.uint64))


def sub(p, a, b, primes):
    return K.submod_rows(a, b, np.array(primes, dtype=np.uint64))


def neg(a, primes):
    q = np.array(primes, dtype=np.uint64)[:, None]
    return np.where(a == 0, a, q - a)


def from_signed(coeffs, primes):
    """limbs_from_signed (ring.py:381-387)."""
    c = np.asarray(coeffs, dtype=np.int64)
    out = np.empty((len(primes), c.shape[-1]), dtype=np.uint64)
    for i, q in enumerate(primes):
        out[i] = np.mod(c, np.int64(q)).astype(np.uint64)
    return out


def auto_eval(limbs, g, n):
    """Eval-form automorphism as a slot gather (ring.py:440-482)."""
    exps = 2 * bitrev(n) + 1  # slot exponents of this NTT ordering
    pos = np.full(2 * n, -1, dtype=np.int64)
    pos[exps] = np.arange(n)
    return limbs[:, pos[(exps * (g % (2 * n))) % (2 * n)]].copy()


def sha(arr):
    return hashlib.sha256(np.ascontiguousarray(arr, dtype="<u8").tobytes()).hexdigest()


# ---------------------------------------------------------------------------
# encoding (ckks/encoding.py:17-143)
# ---------------------------------------------------------------------------


def _emb(n):
    j = np.arange(n)
    zeta = np.exp(1j * np.pi * j / n)
    m = np.empty(n // 2, dtype=np.int64)
    g = 1
    for i in range(n // 2):
        m[i] = g
        g = (g * 5) % (2 * n)
    slot_idx = (m - 1) // 2
    return zeta, slot_idx, n - 1 - slot_idx


def encode_coeffs(p, values, scale):
    n = p.n
    v = np.asarray(values, dtype=np.complex128).ravel()
    full = np.zeros(p.slots, dtype=np.complex128)
    full[: v.size] = v
    zeta, si, ci = _emb(n)
    spec = np.zeros(n, dtype=np.complex128)
    spec[si] = full * scale
    spec[ci] = np.conj(full * scale)
    coeffs = np.real(np.fft.fft(spec) / n * np.conj(zeta))
    return np.rint(coeffs).astype(np.int64)


def encode(p, values, level, scale):
    primes = p.chain[: level + 1]
    return ntt_fwd(p, from_signed(encode_coeffs(p, values, scale), primes), primes)


def decode(p, limbs_eval, level, scale):
    primes = p.chain[: level + 1]
    c = ntt_inv(p, limbs_eval, primes)
    q0 = p.chain[0]
    if level == 0:
        x0 = c[0]
        f = np.where(x0 > q0 // 2, x0.astype(np.float64) - float(q0), x0.astype(np.float64))
    else:
        q1 = p.chain[1]
        x0, x1 = c[0], c[1]
        diff = (x1.astype(object) - (x0 % np.uint64(q1)).astype(object)) % q1
        t = np.array([(int(d) * pow(q0, -1, q1)) % q1 for d in diff], dtype=np.uint64)
        tc = np.where(t > q1 // 2, t.astype(np.float64) - float(q1), t.astype(np.float64))
        f = x0.astype(np.float64) + float(q0) * tc
    zeta, si, _ = _emb(p.n)
    ev = p.n * np.fft.ifft(f * zeta)
    return np.real(ev[si] / scale)


# ---------------------------------------------------------------------------
# keys (ckks/keys.py:103-249)
# ---------------------------------------------------------------------------


class Keys:
    pass


def _uniform(rng, primes, n):
    out = np.empty((len(primes), n), dtype=np.uint64)
    for i, q in enumerate(primes):
        out[i] = rng.integers(0, q, size=n, dtype=np.uint64)
    return out


def _switch_key(p, s_from, s_ext, rng):
    ext = p.ext
    pprod = math.prod(p.special)
    bs, as_ = [], []
    for group in p.digit_groups(p.max_level):
        a = _uniform(rng, ext, p.n)
        e = ntt_fwd(p, from_signed(np.rint(rng.normal(0.0, p.sigma, size=p.n)).astype(np.int64),
                                   ext), ext)
        b = sub(p, e, mul(p, a, s_ext, ext), ext)
        for j in group:
            q = p.chain[j]
            b[j] = (b[j].astype(object) + (s_from[j].astype(object) * (pprod % q)) % q) % q
        bs.append(b.astype(np.uint64))
        as_.append(a)
    return bs, as_


def _auto_ext(p, coeffs, g):
    n = p.n
    j = np.arange(n, dtype=np.int64)
    e = (j * (g % (2 * n))) % (2 * n)
    out = np.zeros(n, dtype=np.int64)
    out[e % n] = coeffs * np.where(e >= n, -1, 1)
    return ntt_fwd(p, from_signed(out, p.ext), p.ext)


def keygen(p, steps, seed, conj=True):
    rng = np.random.default_rng(np.random.PCG64(seed))
    n = p.n
    steps = tuple(dict.fromkeys(int(s) for s in steps))
    if p.hamming is None:
        s = rng.integers(-1, 2, size=n).astype(np.int64)
    else:
        s = np.zeros(n, dtype=np.int64)
        pos = rng.choice(n, size=p.hamming, replace=False)
        s[pos] = rng.choice(np.array([-1, 1]), size=p.hamming)
    k = Keys()
    k.s_ext = ntt_fwd(p, from_signed(s, p.ext), p.ext)
    nc = len(p.chain)
    a_pk = _uniform(rng, p.chain, n)
    e = ntt_fwd(p, from_signed(np.rint(rng.normal(0.0, p.sigma, size=n)).astype(np.int64),
                               p.chain), p.chain)
    k.pk = (sub(p, e, mul(p, a_pk, k.s_ext[:nc], p.chain), p.chain), a_pk)
    k.relin = _switch_key(p, mul(p, k.s_ext, k.s_ext, p.ext), k.s_ext, rng)
    k.rot = {}
    for st in steps:
        g = pow(5, st % (n // 2), 2 * n)
        k.rot[st] = _switch_key(p, _auto_ext(p, s, g), k.s_ext, rng)
    k.conj = _switch_key(p, _auto_ext(p, s, 2 * n - 1), k.s_ext, rng) if conj else None
    k.steps = steps
    return k


# ---------------------------------------------------------------------------
# key switching (ckks/keys.py:19-49, 264-339)
# ---------------------------------------------------------------------------


def _convert(p, limbs, src, dst):
    qs = math.prod(src)
    inv = np.array([pow(qs // q, -1, q) * p.table(q).r % q for q in src], dtype=np.uint64)
    mat = np.array([[(qs // q) % d * p.table(d).r % d for d in dst] for q in src],
                   dtype=np.uint64)
    ss, ds = p.stack(src), p.stack(dst)
    hat = K.rowwise_mont(limbs, inv, ss["q"], ss["qinv"])
    return K.base_convert(hat, mat, ds["q"], ds["qinv"])


def ks_apply(p, swk, d_eval, level):
    chain, specials = p.chain, p.special
    n, ksp = p.n, len(specials)
    d_coeff = ntt_inv(p, d_eval, chain[: level + 1])
    ext = tuple(chain[: level + 1]) + tuple(specials)
    es = p.stack(ext)
    n_ext = level + 1 + ksp
    rows = np.asarray(list(range(level + 1)) + [len(chain) + i for i in range(ksp)], dtype=np.int64)
    acc_b = np.zeros((n_ext, n), dtype=np.uint64)
    acc_a = np.zeros((n_ext, n), dtype=np.uint64)
    for gi, group in enumerate(p.digit_groups(level)):
        src = tuple(chain[j] for j in group)
        dst_rows = [r for r in range(n_ext) if (r < level + 1 and r not in group) or r >= level + 1]
        dst = tuple(ext[r] for r in dst_rows)
        digit = np.empty((n_ext, n), dtype=np.uint64)
        digit[group] = d_eval[group]
        if dst:
            digit[dst_rows] = ntt_fwd(p, _convert(p, d_coeff[group], src, dst), dst)
        K.fma_gather_inplace(acc_b, digit, swk[0][gi], rows, es["q"], es["qinv"], es["r2"])
        K.fma_gather_inplace(acc_a, digit, swk[1][gi], rows, es["q"], es["qinv"], es["r2"])
    cprimes = chain[: level + 1]
    cs = p.stack(cprimes)
    pprod = math.prod(specials)
    pinv = np.array([pow(pprod, -1, q) * p.table(q).r % q for q in cprimes], dtype=np.uint64)
    out = []
    for acc in (acc_b, acc_a):
        sp = ntt_inv(p, acc[level + 1 :], specials)
        corr = ntt_fwd(p, _convert(p, sp, specials, cprimes), cprimes)
        diff = K.submod_rows(acc[: level + 1], corr, cs["q"])
        out.append(K.rowwise_mont(diff, pinv, cs["q"], cs["qinv"]))
    return out[0], out[1]


# ---------------------------------------------------------------------------
# ciphertext operations (ckks/ops.py)
# ---------------------------------------------------------------------------


class Ct:
    def __init__(self, c0, c1, level, scale):
        self.c0, self.c1, self.level, self.scale = c0, c1, level, scale

    def digest(self):
        return {"c0": sha(self.c0), "c1": sha(self.c1), "level": self.level,
                "scale": float(self.scale).hex()}


def encrypt(p, keys, m_eval, level, scale, seed):
    """ops.py:69-123 (RNG order v, e0, e1)."""
    rng = np.random.default_rng(None if seed is None else np.random.PCG64(seed))
    n = p.n
    primes = p.chain[: level + 1]
    k = level + 1
    v = ntt_fwd(p, from_signed(rng.integers(-1, 2, size=n).astype(np.int64), primes), primes)
    e0 = ntt_fwd(p, from_signed(np.rint(rng.normal(0.0, p.sigma, size=n)).astype(np.int64),
                                primes), primes)
    e1 = ntt_fwd(p, from_signed(np.rint(rng.normal(0.0, p.sigma, size=n)).astype(np.int64),
                                primes), primes)
    c0 = add(p, add(p, mul(p, v, keys.pk[0][:k], primes), e0, primes), m_eval[:k], primes)
    c1 = add(p, mul(p, v, keys.pk[1][:k], primes), e1, primes)
    return Ct(c0, c1, level, scale)


def encrypt_vector(p, keys, values, level, seed, scale=None):
    scale = p.scale if scale is None else scale
    return encrypt(p, keys, encode(p, values, level, scale), level, scale, seed)


def decrypt_vector(p, keys, ct):
    primes = p.chain[: ct.level + 1]
    m = add(p, ct.c0, mul(p, ct.c1, keys.s_ext[: ct.level + 1], primes), primes)
    return decode(p, m, ct.level, ct.scale)


def _rescale_poly(p, limbs, level):
    """ops.py:164-189."""
    chain = p.chain
    ql = chain[level]
    top = ntt_inv(p, limbs[level : level + 1], (ql,))
    c = top[0].astype(np.int64)
    c = np.where(c > ql // 2, c - ql, c)
    rest = ntt_fwd(p, from_signed(c, chain[:level]), chain[:level])
    diff = K.submod_rows(limbs[:level], rest, np.array(chain[:level], dtype=np.uint64))
    inv = np.array([pow(ql, -1, q) * p.table(q).r % q for q in chain[:level]], dtype=np.uint64)
    s = p.stack(chain[:level])
    return K.rowwise_mont(diff, inv, s["q"], s["qinv"])


def rescale(p, ct):
    ql = p.chain[ct.level]
    return Ct(_rescale_poly(p, ct.c0, ct.level), _rescale_poly(p, ct.c1, ct.level),
              ct.level - 1, ct.scale / ql)


def mod_down(ct, level):
    if level == ct.level:
        return ct
    return Ct(ct.c0[: level + 1].copy(), ct.c1[: level + 1].copy(), level, ct.scale)


def const_pt(p, value, level, scale):
    """encode_const (ops.py:55-66)."""
    coeffs = np.zeros(p.n, dtype=np.int64)
    coeffs[0] = int(np.rint(float(value) * scale))
    primes = p.chain[: level + 1]
    return ntt_fwd(p, from_signed(coeffs, primes), primes)


def mult_plain(p, ct, pt_eval, pt_scale, rescale_after=True):
    primes = p.chain[: ct.level + 1]
    k = ct.level + 1
    out = Ct(mul(p, ct.c0, pt_eval[:k], primes), mul(p, ct.c1, pt_eval[:k], primes), ct.level,
             ct.scale * pt_scale)
    return rescale(p, out) if rescale_after else out


def add_plain_const(p, ct, value):
    pt = const_pt(p, value, ct.level, ct.scale)
    primes = p.chain[: ct.level + 1]
    return Ct(add(p, ct.c0, pt, primes), ct.c1.copy(), ct.level, ct.scale)


def _align(p, a, b):
    """ops.py:210-231."""
    s1, s2 = a.scale, b.scale
    if a.level == b.level and abs(s1 - s2) <= 1e-9 * max(s1, s2):
        return a, b
    hi, lo = (a, b) if a.level >= b.level else (b, a)
    if hi.level > lo.level and abs(hi.scale - lo.scale) > 1e-9 * lo.scale:
        hi = mod_down(hi, lo.level + 1)
        q = p.chain[hi.level]
        sc = lo.scale * q / hi.scale
        hi = mult_plain(p, hi, const_pt(p, 1.0, hi.level, sc), sc)
        hi.scale = lo.scale
    else:
        hi = mod_down(hi, lo.level)
    return (hi, lo) if a.level >= b.level else (lo, hi)


def ct_add(p, a, b):
    a, b = _align(p, a, b)
    primes = p.chain[: a.level + 1]
    return Ct(add(p, a.c0, b.c0, primes), add(p, a.c1, b.c1, primes), a.level, a.scale)


def ct_sub(p, a, b):
    a, b = _align(p, a, b)
    primes = p.chain[: a.level + 1]
    return Ct(sub(p, a.c0, b.c0, primes), sub(p, a.c1, b.c1, primes), a.level, a.scale)


def mult(p, keys, a, b, rescale_after=True):
    """ops.py:346-367."""
    a, b = _align(p, a, b)
    primes = p.chain[: a.level + 1]
    d0 = mul(p, a.c0, b.c0, primes)
    d1 = add(p, mul(p, a.c0, b.c1, primes), mul(p, a.c1, b.c0, primes), primes)
    d2 = mul(p, a.c1, b.c1, primes)
    kb, ka = ks_apply(p, keys.relin, d2, a.level)
    out = Ct(add(p, d0, kb, primes), add(p, d1, ka, primes), a.level, a.scale * b.scale)
    return rescale(p, out) if rescale_after else out


def _switch(p, ct, g, swk):
    c0r, c1r = auto_eval(ct.c0, g, p.n), auto_eval(ct.c1, g, p.n)
    kb, ka = ks_apply(p, swk, c1r, ct.level)
    return Ct(add(p, c0r, kb, p.chain[: ct.level + 1]), ka, ct.level, ct.scale)


def decompose_rotation(keys, step, slots):
    """keys.py:348-377."""
    step = step % slots
    if step == 0:
        return []
    if step in keys.rot:
        return [step]
    if step - slots in keys.rot:
        return [step - slots]
    remaining = min(step, step - slots, key=abs)
    parts = []
    avail = sorted((s for s in keys.rot if s != 0), key=abs, reverse=True)
    while remaining != 0:
        best = None
        for s in avail:
            if abs(remaining - s) < abs(remaining) and (
                best is None or abs(remaining - s) < abs(remaining - best)
            ):
                best = s
        if best is None:
            raise ValueError("step cannot be decomposed")
        parts.append(best)
        remaining -= best
    return parts


def rotate(p, keys, ct, step):
    for part in decompose_rotation(keys, int(step), p.slots):
        ct = _switch(p, ct, pow(5, part % (p.n // 2), 2 * p.n), keys.rot[part])
    return ct


def conjugate(p, keys, ct):
    return _switch(p, ct, 2 * p.n - 1, keys.conj)


def mod_raise(p, ct):
    """bootstrap.py:260-275."""
    q0 = p.chain[0]
    out = []
    for poly in (ct.c0, ct.c1):
        c = ntt_inv(p, poly[:1], (q0,))[0].astype(np.int64)
        c = np.where(c > q0 // 2, c - q0, c)
        out.append(ntt_fwd(p, from_signed(c, p.chain), p.chain))
    return Ct(out[0], out[1], p.max_level, ct.scale)
