// Device-side modular arithmetic and shared launch descriptors for the
// B200 CKKS engine (sm_100a).
//
// Residues are uint64 words modulo primes q < 2^62 (the reference validates
// this bound in RingParams.__post_init__, /root/reference/pkg/src/hebert/
// ring.py:145-159).  Every value that leaves a kernel is fully reduced to
// [0, q); inside kernels we keep Harvey-style lazy ranges ([0, 2q) / [0, 4q)),
// which is legal because 4q < 2^64.
//
// Two multiplication flavours are used:
//  * Montgomery REDC (R = 2^64) for data x data products and for
//    accumulate-then-reduce inner products.  Same constants as the reference
//    (qinv_neg = -q^-1 mod 2^64, R^2 mod q; ring.py:87-90), so the modular
//    value produced is identical to hebert._kernels._mont (_kernels.py:134).
//  * Shoup multiplication by a known constant w with w' = floor(w 2^64 / q)
//    for twiddles and per-limb scalars (1 mulhi + 2 mullo).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hegpu {

constexpr int kMaxPrimes = 64;  // chain + special primes per ring
constexpr int kMaxSeg = 8;      // independent operand groups per launch

struct PrimeConst {
  uint64_t q;
  uint64_t qinv_neg;  // -q^{-1} mod 2^64
  uint64_t r2;        // R^2 mod q, R = 2^64
  uint64_t bar;       // floor(2^64 / q): Shoup constant of w = 1
  uint64_t ninv;      // N^{-1} mod q
  uint64_t ninv_sh;
  uint64_t ilast;     // ipsi_rev[1] * N^{-1} mod q (fused last inverse stage)
  uint64_t ilast_sh;
};

// ---------------------------------------------------------------------------
// scalar helpers
// ---------------------------------------------------------------------------

// REDC of the 128-bit value hi*2^64 + lo, which must be < q * 2^64.
// Returns (hi*2^64+lo) * 2^-64 mod q in [0, q).
__device__ __forceinline__ uint64_t redc128(uint64_t hi, uint64_t lo, uint64_t q,
                                            uint64_t qneg) {
  uint64_t m = lo * qneg;
  uint64_t r = hi + __umul64hi(m, q) + (lo != 0ull);
  return r >= q ? r - q : r;
}

__device__ __forceinline__ uint64_t mont_mul(uint64_t a, uint64_t b, uint64_t q,
                                             uint64_t qneg) {
  return redc128(__umul64hi(a, b), a * b, q, qneg);
}

// a*b mod q for a, b < q (two REDCs, the second one by R^2).
__device__ __forceinline__ uint64_t mul_mod(uint64_t a, uint64_t b, const PrimeConst& c) {
  return mont_mul(mont_mul(a, b, c.q, c.qinv_neg), c.r2, c.q, c.qinv_neg);
}

// Shoup: a*w mod q, lazily in [0, 2q), valid for any a < 2^64 and w < q.
__device__ __forceinline__ uint64_t shoup_lazy(uint64_t a, uint64_t w, uint64_t wsh,
                                               uint64_t q) {
  return a * w - __umul64hi(a, wsh) * q;
}

__device__ __forceinline__ uint64_t shoup(uint64_t a, uint64_t w, uint64_t wsh, uint64_t q) {
  uint64_t r = shoup_lazy(a, w, wsh, q);
  return r >= q ? r - q : r;
}

__device__ __forceinline__ uint64_t add_mod(uint64_t a, uint64_t b, uint64_t q) {
  uint64_t s = a + b;
  return s >= q ? s - q : s;
}

__device__ __forceinline__ uint64_t sub_mod(uint64_t a, uint64_t b, uint64_t q) {
  uint64_t s = a + (q - b);
  return s >= q ? s - q : s;
}

// x mod q for any x < 2^64.
__device__ __forceinline__ uint64_t reduce64(uint64_t x, const PrimeConst& c) {
  uint64_t r = x - __umul64hi(x, c.bar) * c.q;
  return r >= c.q ? r - c.q : r;
}

// numpy-style np.mod(v, q) for a signed 64-bit v (result in [0, q)).
__device__ __forceinline__ uint64_t signed_mod(int64_t v, const PrimeConst& c) {
  if (v >= 0) return reduce64(static_cast<uint64_t>(v), c);
  uint64_t r = reduce64(static_cast<uint64_t>(-v), c);
  return r ? c.q - r : 0ull;
}

// 128-bit accumulator kept below q * 2^64 (precondition of redc128):
// after each add of a product < q*2^62 subtract q*2^64 when hi >= q.
struct Acc128 {
  uint64_t hi, lo;
  __device__ __forceinline__ void zero() { hi = lo = 0; }
  __device__ __forceinline__ void mac(uint64_t a, uint64_t b, uint64_t q) {
    uint64_t plo = a * b;
    uint64_t phi = __umul64hi(a, b);
    uint64_t nlo = lo + plo;
    hi = hi + phi + (nlo < lo);
    lo = nlo;
    if (hi >= q) hi -= q;
  }
};

// ---------------------------------------------------------------------------
// operand descriptors
// ---------------------------------------------------------------------------

// A group of n_polys polynomials of k limbs each; limb l of poly p lives at
// ptr + p*stride + l*N.  Limb l uses global prime sel[seg][l].
struct Seg {
  const uint64_t* in;
  uint64_t* out;
  int64_t in_stride;
  int64_t out_stride;
  const uint64_t* other;  // epilogue operand (forward NTT only)
  uint64_t* eout;         // epilogue destination
  int64_t other_stride;
  int64_t eout_stride;
  int n_polys;
  int k;
  int row_start;  // first global (poly, limb) row of this segment
  // fused basis-conversion prologue (forward register NTT): the input of limb
  // t of poly p is REDC(sum_i csrc[p*csrc_stride + i*N + x] * cpunc[i*cpunc_ld + t])
  const uint64_t* csrc;
  int64_t csrc_stride;
  const uint64_t* cpunc;
  int c_nsrc;
  int cpunc_ld;
  int eacc;  // epilogue accumulates: eout = eout + (other - y) * c
  // cmode 1: the prologue instead lifts one coefficient-form limb (modulus
  // csrc_q, at csrc + p*csrc_stride) centered into every limb (rescale/ModRaise)
  int cmode;
  uint64_t csrc_q;
};

struct SegSet {
  int n_seg;
  int n_rows;
  Seg seg[kMaxSeg];
  uint8_t sel[kMaxSeg][kMaxPrimes];
};

__device__ __forceinline__ int find_seg(const SegSet& S, int row) {
  int s = 0;
#pragma unroll 1
  while (s + 1 < S.n_seg && row >= S.seg[s + 1].row_start) ++s;
  return s;
}

}  // namespace hegpu
