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
// The kernels stage the twiddles a CTA needs in shared memory first, in the
// order the lanes consume them (TwLayout), so the butterflies' twiddle reads
// are shared-memory loads at compile-time offsets instead of long-latency
// global loads on the dependency chain.
#pragma once
#include "common.cuh"

namespace hegpu {

template <int LOGS>
struct RegShape {
  static constexpr int S = 1 << LOGS;
  static constexpr int EB = LOGS - 5;  // log2(elements per lane)
  static constexpr int E = 1 << EB;
  static constexpr int ROUNDS = (LOGS + EB - 1) / EB;
  // warp buffer: element j of a shuffle lives at j + (j >> s), s >= SMIN (shf_shift)
  static constexpr int SMIN = LOGS - 5;
  static constexpr int PAD_S = S + (S >> SMIN);
};

__device__ __forceinline__ int reg_j(int lane, int e, int lo, int eb) {
  return (lane & ((1 << lo) - 1)) | (e << lo) | ((lane >> lo) << (lo + eb));
}
__device__ __forceinline__ int padi(int j) { return j + (j >> 4); }


// ---------------------------------------------------------------------------
// Twiddles in consumption order.  Round r of a sub-transform works on register
// window [lo, lo + EB); its butterfly at bit p (lower element j) uses twiddle
// tree index (1 << st) + (j >> (p + 1)), st = LOGS - 1 - p, and
//   j >> (p + 1) = (e >> (p + 1 - lo)) | (g << (lo + EB - p - 1)),  g = lane >> lo,
// so a lane's twiddles of a round depend only on its group g.  The CTA stages
// them (once) as [round][group][stage][u]: a lane then reads its round's
// twiddles from one base address with compile-time offsets (no per-butterfly
// index arithmetic), and the 8 lanes of a quarter warp with distinct groups
// read slots cnt(r) apart, which spreads them over the bank groups.
// ---------------------------------------------------------------------------
template <int LOGS, bool INV>
struct TwLayout {
  static constexpr int EB = LOGS - 5, E = 1 << EB, R = (LOGS + EB - 1) / EB;
  static constexpr int plo(int r) {
    return INV ? r * EB : (LOGS - 1 - r * EB - EB + 1 < 0 ? 0 : LOGS - r * EB - EB);
  }
  static constexpr int phi(int r) {
    return INV ? (r * EB + EB - 1 > LOGS - 1 ? LOGS - 1 : r * EB + EB - 1) : LOGS - 1 - r * EB;
  }
  static constexpr int lo(int r) {
    return INV ? (r * EB + EB > LOGS ? LOGS - EB : r * EB)
               : (LOGS - (r + 1) * EB < 0 ? 0 : LOGS - (r + 1) * EB);
  }
  // distinct twiddles per group at bit p of round r
  static constexpr int kp(int r, int p) { return E >> (p + 1 - lo(r)); }
  static constexpr int cnt(int r) {
    int c = 0;
    for (int p = plo(r); p <= phi(r); ++p) c += kp(r, p);
    return c;
  }
  // offset of bit p inside a group's run (stages in execution order)
  static constexpr int pre(int r, int p) {
    int c = 0;
    if (INV) {
      for (int q = plo(r); q < p; ++q) c += kp(r, q);
    } else {
      for (int q = phi(r); q > p; --q) c += kp(r, q);
    }
    return c;
  }
  static constexpr int groups(int r) { return 32 >> lo(r); }
  static constexpr int off(int r) {
    int c = 0;
    for (int q = 0; q < r; ++q) c += groups(q) * cnt(q);
    return c;
  }
  static constexpr int total() { return off(R); }  // == S - 1
  // slot -> (st, local index within the stage); host/device, any slot < total()
  __host__ __device__ static void decode(int s, int& st, int& local) {
    int r = 0;
    while (r + 1 < R && s >= off(r + 1)) ++r;
    const int rel = s - off(r), g = rel / cnt(r);
    int rem = rel - g * cnt(r);
    int p = INV ? plo(r) : phi(r);
    while (rem >= kp(r, p)) {
      rem -= kp(r, p);
      p += INV ? 1 : -1;
    }
    st = LOGS - 1 - p;
    local = rem | (g << (lo(r) + EB - p - 1));
  }
};

// Forward CT butterflies of round r (bits phi down to plo); tw = this lane's
// twiddle run of the round.
template <int LOGS, int r>
__device__ __forceinline__ void fwd_round(uint64_t (&x)[RegShape<LOGS>::E],
                                          const ulonglong2* __restrict__ tw, uint64_t q) {
  using L = TwLayout<LOGS, false>;
  constexpr int E = RegShape<LOGS>::E, lo = L::lo(r);
  const uint64_t q2 = q << 1;
#pragma unroll
  for (int p = L::phi(r); p >= L::plo(r); --p) {
    const int d = 1 << (p - lo);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (e & d) continue;
      uint64_t u = x[e];
      u = u >= q2 ? u - q2 : u;
      const ulonglong2 wp = tw[L::pre(r, p) + (e >> (p + 1 - lo))];
      const uint64_t v = shoup_lazy(x[e + d], wp.x, wp.y, q);
      x[e] = u + v;
      x[e + d] = u - v + q2;
    }
  }
}

// Inverse GS butterflies of round r (bits plo up to phi).  The final stage
// (global t = N/2, `last_p` = its bit, -1 if not in this pass) multiplies the
// sum by fin_s and the difference by fin_d: (N^-1, ipsi_rev[1] N^-1),
// optionally times a per-limb post-scale (ModUp / ModDown).
template <int LOGS, int r>
__device__ __forceinline__ void inv_round(uint64_t (&x)[RegShape<LOGS>::E],
                                          const ulonglong2* __restrict__ tw, int last_p,
                                          const PrimeConst& pc, const ulonglong2 fin_s,
                                          const ulonglong2 fin_d) {
  using L = TwLayout<LOGS, true>;
  constexpr int E = RegShape<LOGS>::E, lo = L::lo(r);
  const uint64_t q = pc.q, q2 = q << 1;
#pragma unroll
  for (int p = L::plo(r); p <= L::phi(r); ++p) {
    const int d = 1 << (p - lo);
    const bool last = p == last_p;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (e & d) continue;
      const uint64_t a = x[e], b = x[e + d];
      uint64_t s = a + b;
      s = s >= q2 ? s - q2 : s;
      const uint64_t df = a - b + q2;
      if (!last) {
        x[e] = s;
        const ulonglong2 wp = tw[L::pre(r, p) + (e >> (p + 1 - lo))];
        x[e + d] = shoup_lazy(df, wp.x, wp.y, q);
      } else {
        x[e] = shoup(s, fin_s.x, fin_s.y, q);
        x[e + d] = shoup(df, fin_d.x, fin_d.y, q);
      }
    }
  }
}

// Padding shift of the warp buffer for a shuffle from window FROM to window TO:
// element j lives at j + (j >> s).  The lane bits and the register bits of j
// are disjoint, so the slot is base(lane) + c(e) with c a compile-time
// constant: no per-access index arithmetic.  s is chosen per (FROM, TO) for
// the fewest shared-memory wavefronts (64-bit words, served per half warp)
// over the store and the load: ideal for every shuffle of S = 64..512 except
// two of S = 256 / three of S = 64, 128 (1.5x).
template <int LOGS>
__host__ __device__ constexpr int shf_shift(int from, int to) {
  if (LOGS == 9) return 4;
  if (LOGS == 8) return (from == 0 && to == 5) || (from == 5 && to == 0) ? 4 : 3;
  if (LOGS == 7) return (from == 5 || to == 5) ? 4 : 2;
  // LOGS == 6
  return (from >= 3 && to >= 3) || from == 5 || to == 5 ? 4 : 1;
}

template <int LOGS, int W>
__device__ __forceinline__ int shf_base(int lane, int s) {
  constexpr int EB = RegShape<LOGS>::EB;
  const int a = (lane & ((1 << W) - 1)) | ((lane >> W) << (W + EB));
  return a + (a >> s);
}

// Re-distribute the warp's elements from window FROM to window TO.
template <int LOGS, int FROM, int TO, typename T>
__device__ __forceinline__ void reg_shuffle(T (&x)[RegShape<LOGS>::E], T* buf, int lane) {
  constexpr int E = RegShape<LOGS>::E;
  if constexpr (FROM != TO) {
    constexpr int s = shf_shift<LOGS>(FROM, TO);
    static_assert(s >= RegShape<LOGS>::SMIN, "warp buffer too small for this padding");
    T* bf = buf + shf_base<LOGS, FROM>(lane, s);
#pragma unroll
    for (int e = 0; e < E; ++e) bf[(e << FROM) + ((e << FROM) >> s)] = x[e];
    __syncwarp();
    const T* bt = buf + shf_base<LOGS, TO>(lane, s);
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = bt[(e << TO) + ((e << TO) >> s)];
    __syncwarp();
  }
}

// lane's twiddle run of round r in the staged table
template <int LOGS, bool INV, int r, typename TW>
__device__ __forceinline__ const TW* tw_run(const TW* tab, int lane) {
  using L = TwLayout<LOGS, INV>;
  return tab + L::off(r) + (lane >> L::lo(r)) * L::cnt(r);
}

// CUR: the window the elements are in; the sub-transform starts and ends in
// the strided window LOGS - EB (j = lane + 32 e)
template <int LOGS, int r = 0, int CUR = LOGS - RegShape<LOGS>::EB>
__device__ __forceinline__ void fwd_rounds(uint64_t (&x)[RegShape<LOGS>::E], uint64_t* buf,
                                           int lane, const ulonglong2* tab, uint64_t q) {
  using L = TwLayout<LOGS, false>;
  if constexpr (r < L::R) {
    reg_shuffle<LOGS, CUR, L::lo(r)>(x, buf, lane);
    fwd_round<LOGS, r>(x, tw_run<LOGS, false, r>(tab, lane), q);
    fwd_rounds<LOGS, r + 1, L::lo(r)>(x, buf, lane, tab, q);
  } else {
    reg_shuffle<LOGS, CUR, LOGS - RegShape<LOGS>::EB>(x, buf, lane);
  }
}

template <int LOGS, int r = 0, int CUR = LOGS - RegShape<LOGS>::EB>
__device__ __forceinline__ void inv_rounds(uint64_t (&x)[RegShape<LOGS>::E], uint64_t* buf,
                                           int lane, const ulonglong2* tab, int last_p,
                                           const PrimeConst& pc, const ulonglong2 fin_s,
                                           const ulonglong2 fin_d) {
  using L = TwLayout<LOGS, true>;
  if constexpr (r < L::R) {
    reg_shuffle<LOGS, CUR, L::lo(r)>(x, buf, lane);
    inv_round<LOGS, r>(x, tw_run<LOGS, true, r>(tab, lane), last_p, pc, fin_s, fin_d);
    inv_rounds<LOGS, r + 1, L::lo(r)>(x, buf, lane, tab, last_p, pc, fin_s, fin_d);
  } else {
    reg_shuffle<LOGS, CUR, LOGS - RegShape<LOGS>::EB>(x, buf, lane);
  }
}

// Full S-point sub-transforms in registers; input / output layout windows
// lo_in / lo_out; tab = the staged consumption-order twiddles (TwLayout).
template <int LOGS>
__device__ __forceinline__ void fwd_sub(uint64_t (&x)[RegShape<LOGS>::E], uint64_t* buf,
                                        int lane, int lo_in, int lo_out, const ulonglong2* tab,
                                        uint64_t q) {
  (void)lo_in;  // both are the strided window LOGS - EB
  (void)lo_out;
  fwd_rounds<LOGS>(x, buf, lane, tab, q);
}

template <int LOGS>
__device__ __forceinline__ void inv_sub(uint64_t (&x)[RegShape<LOGS>::E], uint64_t* buf,
                                        int lane, int lo_in, int lo_out, int last_p,
                                        const ulonglong2* tab, const PrimeConst& pc,
                                        const ulonglong2 fin_s, const ulonglong2 fin_d) {
  (void)lo_in;
  (void)lo_out;
  inv_rounds<LOGS>(x, buf, lane, tab, last_p, pc, fin_s, fin_d);
}

// ---------------------------------------------------------------------------
// FP64-pipe variants (primes q < 2^kFpMaxBits, common.cuh): elements are
// integers held in doubles in signed lazy ranges, twiddles are (w, w/q).
// Forward CT: u + v, u - v with v = w*x in (-q, q): the bound grows by q per
// stage (<= (stages + 1) q, < 2^51 over both passes of N <= 2^17).
// Inverse GS: the sum doubles per stage, so it is centred-reduced after every
// 4th stage and at the end of a non-final pass (bound <= 16 q < 2^50).
// ---------------------------------------------------------------------------
template <int LOGS, int r>
__device__ __forceinline__ void fwd_round_fp(double (&x)[RegShape<LOGS>::E],
                                             const double2* __restrict__ tw, double q) {
  using L = TwLayout<LOGS, false>;
  constexpr int E = RegShape<LOGS>::E, lo = L::lo(r);
#pragma unroll
  for (int p = L::phi(r); p >= L::plo(r); --p) {
    const int d = 1 << (p - lo);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (e & d) continue;
      const double2 wp = tw[L::pre(r, p) + (e >> (p + 1 - lo))];
      const double v = fp_mulmod(x[e + d], wp.x, wp.y, q);
      const double u = x[e];
      x[e] = u + v;
      x[e + d] = u - v;
    }
  }
}

template <int LOGS, int r>
__device__ __forceinline__ void inv_round_fp(double (&x)[RegShape<LOGS>::E],
                                             const double2* __restrict__ tw, int last_p,
                                             double q, double qinv, const double2 fin_s,
                                             const double2 fin_d) {
  using L = TwLayout<LOGS, true>;
  constexpr int E = RegShape<LOGS>::E, lo = L::lo(r);
#pragma unroll
  for (int p = L::plo(r); p <= L::phi(r); ++p) {
    const int d = 1 << (p - lo);
    const bool last = p == last_p;
    const bool red = (p & 3) == 3 || p == LOGS - 1;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (e & d) continue;
      const double a = x[e], b = x[e + d];
      const double s = a + b;
      const double df = a - b;
      if (!last) {
        const double2 wp = tw[L::pre(r, p) + (e >> (p + 1 - lo))];
        x[e] = red ? fp_reduce(s, q, qinv) : s;
        x[e + d] = fp_mulmod(df, wp.x, wp.y, q);
      } else {
        x[e] = fp_mulmod(s, fin_s.x, fin_s.y, q);
        x[e + d] = fp_mulmod(df, fin_d.x, fin_d.y, q);
      }
    }
  }
}

template <int LOGS, int r = 0, int CUR = LOGS - RegShape<LOGS>::EB>
__device__ __forceinline__ void fwd_rounds_fp(double (&x)[RegShape<LOGS>::E], double* buf,
                                              int lane, const double2* tab, double q) {
  using L = TwLayout<LOGS, false>;
  if constexpr (r < L::R) {
    reg_shuffle<LOGS, CUR, L::lo(r)>(x, buf, lane);
    fwd_round_fp<LOGS, r>(x, tw_run<LOGS, false, r>(tab, lane), q);
    fwd_rounds_fp<LOGS, r + 1, L::lo(r)>(x, buf, lane, tab, q);
  } else {
    reg_shuffle<LOGS, CUR, LOGS - RegShape<LOGS>::EB>(x, buf, lane);
  }
}

template <int LOGS, int r = 0, int CUR = LOGS - RegShape<LOGS>::EB>
__device__ __forceinline__ void inv_rounds_fp(double (&x)[RegShape<LOGS>::E], double* buf,
                                              int lane, const double2* tab, int last_p,
                                              double q, double qinv, const double2 fin_s,
                                              const double2 fin_d) {
  using L = TwLayout<LOGS, true>;
  if constexpr (r < L::R) {
    reg_shuffle<LOGS, CUR, L::lo(r)>(x, buf, lane);
    inv_round_fp<LOGS, r>(x, tw_run<LOGS, true, r>(tab, lane), last_p, q, qinv, fin_s, fin_d);
    inv_rounds_fp<LOGS, r + 1, L::lo(r)>(x, buf, lane, tab, last_p, q, qinv, fin_s, fin_d);
  } else {
    reg_shuffle<LOGS, CUR, LOGS - RegShape<LOGS>::EB>(x, buf, lane);
  }
}

template <int LOGS>
__device__ __forceinline__ void fwd_sub_fp(double (&x)[RegShape<LOGS>::E], double* buf, int lane,
                                           int lo_in, int lo_out, const double2* tab, double q) {
  (void)lo_in;
  (void)lo_out;
  fwd_rounds_fp<LOGS>(x, buf, lane, tab, q);
}

template <int LOGS>
__device__ __forceinline__ void inv_sub_fp(double (&x)[RegShape<LOGS>::E], double* buf, int lane,
                                           int lo_in, int lo_out, int last_p, const double2* tab,
                                           double q, double qinv, const double2 fin_s,
                                           const double2 fin_d) {
  (void)lo_in;
  (void)lo_out;
  inv_rounds_fp<LOGS>(x, buf, lane, tab, last_p, q, qinv, fin_s, fin_d);
}

}  // namespace hegpu
