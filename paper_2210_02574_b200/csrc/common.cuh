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
  // FP64-pipe twiddles (w, w/q) for primes below kFpMaxBits bits, forward
  // [0, N) then inverse [N, 2N); nullptr: this prime takes the integer path
  const double2* twf;
  uint64_t pad_;
};

// ---------------------------------------------------------------------------
// FP64 modular arithmetic for primes q < 2^kFpMaxBits (sm_100a runs DFMA at
// 64 lanes/clk/SM; a modmul below is 6 FP64 ops, ~2.7x the measured rate of
// the 64-bit integer Shoup product, tools/fpmodpeak.cu).  Residues are
// integers held exactly in doubles, in signed lazy ranges.
//   h = a*w, l = fma(a, w, -h)     exact: a*w = h + l
//   t = rint(a * (w/q))            quotient estimate, |a*w/q - t| < 0.75
//   r = fma(-t, q, h) + l          exact (|r| < q < 2^53), r in (-q, q)
// Valid for |a| < 2^51 and w < q; results identical as residues to the
// integer path, so the transforms stay bit-exact once normalised.
// ---------------------------------------------------------------------------
constexpr int kFpMaxBits = 46;
constexpr double kFpMagic = 6755399441055744.0;  // 1.5 * 2^52: rint by addition
constexpr long long kFpMagicBits = 0x4338000000000000LL;

__device__ __forceinline__ double fp_mulmod(double a, double w, double wq, double q) {
  const double h = a * w;
  const double l = fma(a, w, -h);
  const double t = fma(a, wq, kFpMagic) - kFpMagic;
  return fma(-t, q, h) + l;
}
// centered reduction: |result| <= q/2 (+1), for |x| < 2^51
__device__ __forceinline__ double fp_reduce(double x, double q, double qinv) {
  const double t = fma(x, qinv, kFpMagic) - kFpMagic;
  return fma(-t, q, x);
}
// Split products for primes q < 2^46: a residue x is held as (h, l) =
// (rint(x / 2^23), x - 2^23 h), |h| <= 2^23, |l| <= 2^22, so
//   x y = 2^46 h h' + 2^23 (h l' + l h') + l l'
// with every partial product <= 2^46: three FP64 accumulators stay exact for
// 64 products, each product costing 4 DFMA.
struct FpSplitAcc {
  double h, m, l;
  __device__ __forceinline__ void zero() { h = m = l = 0.0; }
  __device__ __forceinline__ void add(double2 x, double2 y) {
    h = fma(x.x, y.x, h);
    m = fma(x.x, y.y, m);
    m = fma(x.y, y.x, m);
    l = fma(x.y, y.y, l);
  }
};
struct FpSplitConst {
  double q, qinv, c23, c23q, c46, c46q;  // 2^23, 2^46 mod q and their quotients
};
__device__ __forceinline__ FpSplitConst fp_split_const(uint64_t qi) {
  FpSplitConst c;
  c.q = (double)qi;
  c.qinv = 1.0 / c.q;
  c.c23 = (double)((1ull << 23) % qi);
  c.c46 = (double)((1ull << 46) % qi);
  c.c23q = c.c23 / c.q;
  c.c46q = c.c46 / c.q;
  return c;
}

// signed 64-bit integer <-> double, exact for |x| < 2^51
__device__ __forceinline__ double fp_from_s64(uint64_t x) {
  return __longlong_as_double(static_cast<long long>(x) + kFpMagicBits) - kFpMagic;
}
__device__ __forceinline__ uint64_t fp_to_s64(double x) {
  return static_cast<uint64_t>(__double_as_longlong(x + kFpMagic) - kFpMagicBits);
}
// x in (-q, q) -> residue in [0, q)
__device__ __forceinline__ uint64_t fp_to_residue_small(double x, double q) {
  return fp_to_s64(x < 0.0 ? x + q : x);
}
// any |x| < 2^51 -> residue in [0, q)
__device__ __forceinline__ uint64_t fp_to_residue(double x, double q, double qinv) {
  return fp_to_residue_small(fp_reduce(x, q, qinv), q);
}
// residue (< 2^46) -> (h, l) split
__device__ __forceinline__ double2 fp_split23(uint64_t w) {
  const double x = fp_from_s64(w);
  const double h = fma(x, 0x1p-23, kFpMagic) - kFpMagic;
  return make_double2(h, fma(-h, 0x1p23, x));
}
// value of a split accumulator, centred-reduced: |result| <= q/2 + 1
__device__ __forceinline__ double fp_split_fold(const FpSplitAcc& a, const FpSplitConst& c) {
  const double v = fp_mulmod(fp_reduce(a.h, c.q, c.qinv), c.c46, c.c46q, c.q) +
                   fp_mulmod(fp_reduce(a.m, c.q, c.qinv), c.c23, c.c23q, c.q) +
                   fp_reduce(a.l, c.q, c.qinv);
  return fp_reduce(v, c.q, c.qinv);
}

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

// 128-bit multiply-accumulator with deferred carries: 4 IMAD.WIDE + 1 IADD3.X
// per product (the portable 64-bit formulation costs ~18 SASS instructions).
// Value = W + M * 2^32 + c * 2^96 with W = H:L, M (the two
// cross products) and C the count of M's carries out.  Inputs must be < 2^62.
// Invariant: after fold() the value is < q * 2^64; from there kMacFold more
// products (< 2^124 each) keep it below 2^128, so callers fold at least every
// kMacFold products.
constexpr int kMacFold = 8;

struct Mac128 {
  // 64-bit halves keep the IMAD.WIDE operands in aligned register pairs
  uint64_t L, H, M;  // W = H:L, M = m1:m0
  uint32_t c;
  __device__ __forceinline__ void zero() {
    L = H = M = 0;
    c = 0;
  }
  __device__ __forceinline__ void add(uint64_t a, uint64_t b) {
    asm("{\n\t.reg .u32 a0, a1, b0, b1, l0, l1, h0, h1, m0, m1;\n\t"
        "mov.b64 {a0, a1}, %4;\n\tmov.b64 {b0, b1}, %5;\n\t"
        "mov.b64 {l0, l1}, %0;\n\tmov.b64 {h0, h1}, %1;\n\tmov.b64 {m0, m1}, %2;\n\t"
        "mad.lo.cc.u32 l0, a0, b0, l0;\n\tmadc.hi.cc.u32 l1, a0, b0, l1;\n\t"
        "madc.lo.cc.u32 h0, a1, b1, h0;\n\tmadc.hi.u32 h1, a1, b1, h1;\n\t"
        "mad.lo.cc.u32 m0, a0, b1, m0;\n\tmadc.hi.cc.u32 m1, a0, b1, m1;\n\taddc.u32 %3, %3, 0;\n\t"
        "mad.lo.cc.u32 m0, a1, b0, m0;\n\tmadc.hi.cc.u32 m1, a1, b0, m1;\n\taddc.u32 %3, %3, 0;\n\t"
        "mov.b64 %0, {l0, l1};\n\tmov.b64 %1, {h0, h1};\n\tmov.b64 %2, {m0, m1};\n\t}"
        : "+l"(L), "+l"(H), "+l"(M), "+r"(c)
        : "l"(a), "l"(b));
  }
  // exact 128-bit value (hi, lo)
  __device__ __forceinline__ void value(uint64_t& hi, uint64_t& lo) const {
    lo = L + (M << 32);
    hi = H + (M >> 32) + (static_cast<uint64_t>(c) << 32) + (lo < L);
  }
  // hi <- hi mod q (value mod q*2^64 unchanged modulo q); bar = floor(2^64/q)
  __device__ __forceinline__ void fold(uint64_t q, uint64_t bar) {
    uint64_t hi, lo;
    value(hi, lo);
    uint64_t r = hi - __umul64hi(hi, bar) * q;
    L = lo;
    H = r >= q ? r - q : r;
    M = 0;
    c = 0;
  }
  // value * 2^-64 mod q, in [0, q)
  __device__ __forceinline__ uint64_t redc(const PrimeConst& pc) const {
    uint64_t hi, lo;
    value(hi, lo);
    uint64_t r = hi - __umul64hi(hi, pc.bar) * pc.q;
    r = r >= pc.q ? r - pc.q : r;
    return redc128(r, lo, pc.q, pc.qinv_neg);
  }
};

// 16-byte global -> shared copy that does not occupy registers (LDGSTS).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// --- mbarrier + bulk-copy (TMA engine) helpers ------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared, completing `bytes` of transactions on bar
// (bytes and both addresses 16-byte aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// generic-proxy accesses of shared memory before later async-proxy ones
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

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
  int eacc;  // epilogue: 1 -> eout += (other - y) * c; 2 -> eout = ein * s + (other - y) * c
  const uint64_t* ein;
  int64_t ein_stride;
  // cmode 1: the prologue instead lifts one coefficient-form limb (modulus
  // csrc_q, at csrc + p*csrc_stride) centered into every limb (rescale/ModRaise)
  // cmode 3: the prologue reads signed int64 coefficients (csrc + p*csrc_stride)
  // and reduces them into every limb (numpy np.mod semantics)
  // cmode 2: conversion of the CENTERED representative: the overflow count
  // e = round(sum_i hat_i / d_i) is estimated in fp32 from (hat_i >> cfs[i]) *
  // cfw[i] (cfw = 2^cfs / d_i; both read at stride 2, one per 64-bit word)
  // and e * cnegd[t] (= -D R mod p_t) is added
  int cmode;
  // every conversion source prime is < 2^kFpMaxBits: the prologue may run
  // part of its products on the FP64 pipe (split products, above)
  int c_fp_src;
  uint64_t csrc_q;
  const uint64_t* cnegd;
  const float* cfw;
  const int32_t* cfs;
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
