// Register-resident radix NTT passes (sm_100a), used for N >= 2^12.
//
// Same decomposition as ntt.cu (forward: column pass over the first a stages,
// block pass over the rest; inverse reversed), but each S-point sub-transform
// (S = 2^LOGS in {64..512}) is owned by ONE warp: every lane keeps E = S/32
// elements in registers and runs log2(E) butterfly stages per round without
// any barrier; between rounds the warp re-distributes its elements through a
// warp-private shared-memory buffer (__syncwarp only).  The element index j
// of (lane, e) in a round whose register window starts at bit `lo` is
//     j = (lane & (2^lo - 1)) | (e << lo) | ((lane >> lo) << (lo + log2 E)),
// so a butterfly at distance t = 2^p pairs registers e and e + 2^(p - lo).
// Twiddle indices are the reference's psi_rev[m + i] / ipsi_rev[h + i]
// (hebert/_kernels.py:152-203) expressed in global stage/group terms, so the
// output is bit-identical to the CT/GS transforms.
//
// The kernels stage the twiddles a CTA needs in shared memory first (the
// round functions index `tw` with the same formulas, on a re-based table),
// so the butterflies' twiddle reads are shared-memory loads instead of
// long-latency global loads on the dependency chain.
#pragma once
#include "common.cuh"

namespace hegpu {

template <int LOGS>
struct RegShape {
  static constexpr int S = 1 << LOGS;
  static constexpr int EB = LOGS - 5;  // log2(elements per lane)
  static constexpr int E = 1 << EB;
  static constexpr int ROUNDS = (LOGS + EB - 1) / EB;
  static constexpr int PAD_S = S + S / 16;  // warp buffer with 1 pad word per 16
};

__device__ __forceinline__ int reg_j(int lane, int e, int lo, int eb) {
  return (lane & ((1 << lo) - 1)) | (e << lo) | ((lane >> lo) << (lo + eb));
}
__device__ __forceinline__ int padi(int j) { return j + (j >> 4); }
// warp-buffer slot of element j: 64-bit accesses are served per half-warp, so
// a half-warp's 16 words must hit 16 distinct bank pairs.  For the round
// windows of S = 128 / 256 the XOR swizzle j ^ ((j >> 3) & 15) is
// conflict-free in every round (1 padded word per 16 leaves 2-way conflicts);
// for S = 512 the padding is.
template <int LOGS>
__device__ __forceinline__ int shf_idx(int j) {
  if constexpr (LOGS == 7 || LOGS == 8)
    return j ^ ((j >> 3) & 15);
  else
    return padi(j);
}
// shared-memory slot of staged twiddle i (16-byte entries, served per quarter
// warp): late stages read twiddles at a lane stride of 2..8 entries, which the
// swizzle spreads over the 8 bank groups (4x fewer wavefronts at stride 4)
__device__ __forceinline__ int tw_sw(int i) { return i ^ ((i >> 3) & 7); }


// Forward CT butterflies on register window [lo, lo+EB) for bit positions
// p = phi down to plo (t = 2^p within the sub-transform).  Twiddle index of
// the butterfly whose lower element is j at local stage st (t = 2^(LOGS-1-st))
// is tw_base(st) + (j >> (p + 1)), tw_base(st) = (1 << (g0 + st)) + (blk << st).
template <int LOGS>
__device__ __forceinline__ void fwd_round(uint64_t (&x)[RegShape<LOGS>::E], int lane, int lo,
                                          int phi, int plo, int g0, int blk,
                                          const ulonglong2* __restrict__ tw, uint64_t q) {
  constexpr int E = RegShape<LOGS>::E, EB = RegShape<LOGS>::EB;
  const uint64_t q2 = q << 1;
#pragma unroll
  for (int p = LOGS - 1; p >= 0; --p) {
    if (p > phi || p < plo) continue;
    const int st = LOGS - 1 - p;
    const int d = 1 << (p - lo);
    const int base = (1 << (g0 + st)) + (blk << st);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (e & d) continue;
      const int j = reg_j(lane, e, lo, EB);
      const int ti = base + (j >> (p + 1));
      uint64_t u = x[e];
      u = u >= q2 ? u - q2 : u;
      const ulonglong2 wp = tw[tw_sw(ti)];
      const uint64_t v = shoup_lazy(x[e + d], wp.x, wp.y, q);
      x[e] = u + v;
      x[e + d] = u - v + q2;
    }
  }
}

// Inverse GS butterflies for bit positions p = plo up to phi.  Twiddle index
// is hbase(p) + (blk << (LOGS - p - 1)) + (j >> (p + 1)) with
// hbase(p) = N >> (gshift + p + 1), gshift the global bit offset of this pass.
// The final stage (global t = N/2) multiplies the sum by fin_s and the
// difference by fin_d: (N^-1, ipsi_rev[1] N^-1), optionally times a per-limb
// post-scale (the ModUp / ModDown punctured-product inverse).
template <int LOGS>
__device__ __forceinline__ void inv_round(uint64_t (&x)[RegShape<LOGS>::E], int lane, int lo,
                                          int plo, int phi, int log_n, int gshift, int blk,
                                          const ulonglong2* __restrict__ tw,
                                          const PrimeConst& pc, const ulonglong2 fin_s,
                                          const ulonglong2 fin_d) {
  constexpr int E = RegShape<LOGS>::E, EB = RegShape<LOGS>::EB;
  const uint64_t q = pc.q, q2 = q << 1;
#pragma unroll
  for (int p = 0; p < LOGS; ++p) {
    if (p < plo || p > phi) continue;
    const int d = 1 << (p - lo);
    const bool last = (gshift + p == log_n - 1);
    const int base = (1 << (log_n - gshift - p - 1)) + (blk << (LOGS - p - 1));
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (e & d) continue;
      const uint64_t a = x[e], b = x[e + d];
      uint64_t s = a + b;
      s = s >= q2 ? s - q2 : s;
      const uint64_t df = a - b + q2;
      if (!last) {
        const int j = reg_j(lane, e, lo, EB);
        const int ti = base + (j >> (p + 1));
        x[e] = s;
        const ulonglong2 wp = tw[tw_sw(ti)];
        x[e + d] = shoup_lazy(df, wp.x, wp.y, q);
      } else {
        x[e] = shoup(s, fin_s.x, fin_s.y, q);
        x[e + d] = shoup(df, fin_d.x, fin_d.y, q);
      }
    }
  }
}

// Re-distribute the warp's elements from window lo_from to window lo_to.
template <int LOGS, typename T>
__device__ __forceinline__ void reg_shuffle(T (&x)[RegShape<LOGS>::E], T* buf,
                                            int lane, int lo_from, int lo_to) {
  constexpr int E = RegShape<LOGS>::E, EB = RegShape<LOGS>::EB;
  if (lo_from == lo_to) return;
#pragma unroll
  for (int e = 0; e < E; ++e) buf[shf_idx<LOGS>(reg_j(lane, e, lo_from, EB))] = x[e];
  __syncwarp();
#pragma unroll
  for (int e = 0; e < E; ++e) x[e] = buf[shf_idx<LOGS>(reg_j(lane, e, lo_to, EB))];
  __syncwarp();
}

// Full S-point forward sub-transform in registers; input layout window
// lo_in, output layout window lo_out.
template <int LOGS>
__device__ __forceinline__ void fwd_sub(uint64_t (&x)[RegShape<LOGS>::E], uint64_t* buf,
                                        int lane, int lo_in, int lo_out, int g0, int blk,
                                        const ulonglong2* tw, uint64_t q) {
  constexpr int EB = RegShape<LOGS>::EB, R = RegShape<LOGS>::ROUNDS;
  int cur = lo_in;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int phi = LOGS - 1 - r * EB;
    const int plo = phi - EB + 1 < 0 ? 0 : phi - EB + 1;
    const int lo = LOGS - (r + 1) * EB < 0 ? 0 : LOGS - (r + 1) * EB;
    reg_shuffle<LOGS>(x, buf, lane, cur, lo);
    cur = lo;
    fwd_round<LOGS>(x, lane, lo, phi, plo, g0, blk, tw, q);
  }
  reg_shuffle<LOGS>(x, buf, lane, cur, lo_out);
}

template <int LOGS>
__device__ __forceinline__ void inv_sub(uint64_t (&x)[RegShape<LOGS>::E], uint64_t* buf,
                                        int lane, int lo_in, int lo_out, int log_n, int gshift,
                                        int blk, const ulonglong2* tw, const PrimeConst& pc,
                                        const ulonglong2 fin_s, const ulonglong2 fin_d) {
  constexpr int EB = RegShape<LOGS>::EB, R = RegShape<LOGS>::ROUNDS;
  int cur = lo_in;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int plo = r * EB;
    const int phi = plo + EB - 1 > LOGS - 1 ? LOGS - 1 : plo + EB - 1;
    const int lo = plo + EB > LOGS ? LOGS - EB : plo;
    reg_shuffle<LOGS>(x, buf, lane, cur, lo);
    cur = lo;
    inv_round<LOGS>(x, lane, lo, plo, phi, log_n, gshift, blk, tw, pc, fin_s, fin_d);
  }
  reg_shuffle<LOGS>(x, buf, lane, cur, lo_out);
}

// Two independent sub-transforms in lockstep (the same twiddles: the same
// limb of two polys): each round runs both register sets back to back so the
// scheduler interleaves two independent butterfly streams (2x ILP), and the
// two re-distributions share one pair of __syncwarp.
template <int LOGS>
__device__ __forceinline__ void reg_shuffle2(uint64_t (&x0)[RegShape<LOGS>::E],
                                             uint64_t (&x1)[RegShape<LOGS>::E], uint64_t* b0,
                                             uint64_t* b1, int lane, int lo_from, int lo_to) {
  constexpr int E = RegShape<LOGS>::E, EB = RegShape<LOGS>::EB;
  if (lo_from == lo_to) return;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int j = shf_idx<LOGS>(reg_j(lane, e, lo_from, EB));
    b0[j] = x0[e];
    b1[j] = x1[e];
  }
  __syncwarp();
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int j = shf_idx<LOGS>(reg_j(lane, e, lo_to, EB));
    x0[e] = b0[j];
    x1[e] = b1[j];
  }
  __syncwarp();
}

template <int LOGS>
__device__ __forceinline__ void fwd_sub2(uint64_t (&x0)[RegShape<LOGS>::E],
                                         uint64_t (&x1)[RegShape<LOGS>::E], uint64_t* b0,
                                         uint64_t* b1, int lane, int lo_in, int lo_out, int g0,
                                         int blk, const ulonglong2* tw, uint64_t q) {
  constexpr int EB = RegShape<LOGS>::EB, R = RegShape<LOGS>::ROUNDS;
  int cur = lo_in;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int phi = LOGS - 1 - r * EB;
    const int plo = phi - EB + 1 < 0 ? 0 : phi - EB + 1;
    const int lo = LOGS - (r + 1) * EB < 0 ? 0 : LOGS - (r + 1) * EB;
    reg_shuffle2<LOGS>(x0, x1, b0, b1, lane, cur, lo);
    cur = lo;
    fwd_round<LOGS>(x0, lane, lo, phi, plo, g0, blk, tw, q);
    fwd_round<LOGS>(x1, lane, lo, phi, plo, g0, blk, tw, q);
  }
  reg_shuffle2<LOGS>(x0, x1, b0, b1, lane, cur, lo_out);
}

template <int LOGS>
__device__ __forceinline__ void inv_sub2(uint64_t (&x0)[RegShape<LOGS>::E],
                                         uint64_t (&x1)[RegShape<LOGS>::E], uint64_t* b0,
                                         uint64_t* b1, int lane, int lo_in, int lo_out, int log_n,
                                         int gshift, int blk, const ulonglong2* tw,
                                         const PrimeConst& pc, const ulonglong2 fin_s,
                                         const ulonglong2 fin_d) {
  constexpr int EB = RegShape<LOGS>::EB, R = RegShape<LOGS>::ROUNDS;
  int cur = lo_in;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int plo = r * EB;
    const int phi = plo + EB - 1 > LOGS - 1 ? LOGS - 1 : plo + EB - 1;
    const int lo = plo + EB > LOGS ? LOGS - EB : plo;
    reg_shuffle2<LOGS>(x0, x1, b0, b1, lane, cur, lo);
    cur = lo;
    inv_round<LOGS>(x0, lane, lo, plo, phi, log_n, gshift, blk, tw, pc, fin_s, fin_d);
    inv_round<LOGS>(x1, lane, lo, plo, phi, log_n, gshift, blk, tw, pc, fin_s, fin_d);
  }
  reg_shuffle2<LOGS>(x0, x1, b0, b1, lane, cur, lo_out);
}

// ---------------------------------------------------------------------------
// FP64-pipe variants (primes q < 2^kFpMaxBits, common.cuh): elements are
// integers held in doubles in signed lazy ranges, twiddles are (w, w/q).
// Forward CT: u + v, u - v with v = w*x in (-q, q): the bound grows by q per
// stage (<= (stages + 1) q, < 2^51 over both passes of N <= 2^17).
// Inverse GS: the sum doubles per stage, so it is centred-reduced after every
// 4th stage and at the end of a non-final pass (bound <= 16 q < 2^50).
// ---------------------------------------------------------------------------
template <int LOGS>
__device__ __forceinline__ void fwd_round_fp(double (&x)[RegShape<LOGS>::E], int lane, int lo,
                                             int phi, int plo, int g0, int blk,
                                             const double2* __restrict__ tw, double q) {
  constexpr int E = RegShape<LOGS>::E, EB = RegShape<LOGS>::EB;
#pragma unroll
  for (int p = LOGS - 1; p >= 0; --p) {
    if (p > phi || p < plo) continue;
    const int st = LOGS - 1 - p;
    const int d = 1 << (p - lo);
    const int base = (1 << (g0 + st)) + (blk << st);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (e & d) continue;
      const int j = reg_j(lane, e, lo, EB);
      const double2 wp = tw[tw_sw(base + (j >> (p + 1)))];
      const double v = fp_mulmod(x[e + d], wp.x, wp.y, q);
      const double u = x[e];
      x[e] = u + v;
      x[e + d] = u - v;
    }
  }
}

template <int LOGS>
__device__ __forceinline__ void inv_round_fp(double (&x)[RegShape<LOGS>::E], int lane, int lo,
                                             int plo, int phi, int log_n, int gshift, int blk,
                                             const double2* __restrict__ tw, double q,
                                             double qinv, const double2 fin_s,
                                             const double2 fin_d) {
  constexpr int E = RegShape<LOGS>::E, EB = RegShape<LOGS>::EB;
#pragma unroll
  for (int p = 0; p < LOGS; ++p) {
    if (p < plo || p > phi) continue;
    const int d = 1 << (p - lo);
    const bool last = (gshift + p == log_n - 1);
    const bool red = (p & 3) == 3 || p == LOGS - 1;
    const int base = (1 << (log_n - gshift - p - 1)) + (blk << (LOGS - p - 1));
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (e & d) continue;
      const double a = x[e], b = x[e + d];
      double s = a + b;
      const double df = a - b;
      if (!last) {
        const int j = reg_j(lane, e, lo, EB);
        const double2 wp = tw[tw_sw(base + (j >> (p + 1)))];
        x[e] = red ? fp_reduce(s, q, qinv) : s;
        x[e + d] = fp_mulmod(df, wp.x, wp.y, q);
      } else {
        x[e] = fp_mulmod(s, fin_s.x, fin_s.y, q);
        x[e + d] = fp_mulmod(df, fin_d.x, fin_d.y, q);
      }
    }
  }
}

template <int LOGS>
__device__ __forceinline__ void fwd_sub_fp(double (&x)[RegShape<LOGS>::E], double* buf, int lane,
                                           int lo_in, int lo_out, int g0, int blk,
                                           const double2* tw, double q) {
  constexpr int EB = RegShape<LOGS>::EB, R = RegShape<LOGS>::ROUNDS;
  int cur = lo_in;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int phi = LOGS - 1 - r * EB;
    const int plo = phi - EB + 1 < 0 ? 0 : phi - EB + 1;
    const int lo = LOGS - (r + 1) * EB < 0 ? 0 : LOGS - (r + 1) * EB;
    reg_shuffle<LOGS>(x, buf, lane, cur, lo);
    cur = lo;
    fwd_round_fp<LOGS>(x, lane, lo, phi, plo, g0, blk, tw, q);
  }
  reg_shuffle<LOGS>(x, buf, lane, cur, lo_out);
}

template <int LOGS>
__device__ __forceinline__ void inv_sub_fp(double (&x)[RegShape<LOGS>::E], double* buf, int lane,
                                           int lo_in, int lo_out, int log_n, int gshift, int blk,
                                           const double2* tw, double q, double qinv,
                                           const double2 fin_s, const double2 fin_d) {
  constexpr int EB = RegShape<LOGS>::EB, R = RegShape<LOGS>::ROUNDS;
  int cur = lo_in;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int plo = r * EB;
    const int phi = plo + EB - 1 > LOGS - 1 ? LOGS - 1 : plo + EB - 1;
    const int lo = plo + EB > LOGS ? LOGS - EB : plo;
    reg_shuffle<LOGS>(x, buf, lane, cur, lo);
    cur = lo;
    inv_round_fp<LOGS>(x, lane, lo, plo, phi, log_n, gshift, blk, tw, q, qinv, fin_s, fin_d);
  }
  reg_shuffle<LOGS>(x, buf, lane, cur, lo_out);
}

}  // namespace hegpu
