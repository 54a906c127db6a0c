// Batched negacyclic NTT for sm_100a.
//
// Bit-exact with the reference transforms (hebert/_kernels.py:144-204): same
// psi (ring.py:69-78), same bit-reversed twiddle tables (ring.py:94-108), same
// natural -> bit-reversed (forward CT) / bit-reversed -> natural (inverse GS,
// times N^-1) orderings.  Modular arithmetic is exact, so any schedule of the
// same butterflies produces identical residues; ours is:
//
//   N = R * C with R = 2^a, a = ceil(log N / 2).
//   forward  pass A ("cols"):  stages 0..a-1 act on R-element columns
//                               (stride C), independent per column, same
//                               twiddles for every column;
//            pass B ("blocks"): stages a..logN-1 act on contiguous C-element
//                               blocks.
//   inverse  pass B first (stages with span < C), pass A last with N^-1 and
//            the last twiddle folded into the final butterfly.
//
// Each CTA stages a 4096-element tile (32 KiB) in shared memory; a limb of
// N = 2^16 is 16 tiles, so every launch has (16 x limbs x polys) CTAs.
// Intermediate values stay in Harvey lazy ranges ([0,4q) forward, [0,2q)
// inverse); outputs are fully reduced.
#include <cooperative_groups.h>

#include <mutex>
#include <vector>

#include "ntt_reg.cuh"
#include "ring.cuh"

namespace hegpu {

struct NttParams {
  SegSet S;
  const PrimeConst* pc;
  const uint64_t* tw;
  int log_n;
  int a;
  int tile_log;  // log2 of the CPB / BPC group size
  int epi;
  uint64_t c[kMaxPrimes];
  uint64_t csh[kMaxPrimes];
  uint64_t es[kMaxPrimes];  // eacc == 2 input scale (Shoup pairs)
  uint64_t essh[kMaxPrimes];
  // inverse with post-scale: final-stage constants per limb (sum, difference)
  int post;
  ulonglong2 fin_s[kMaxPrimes];
  ulonglong2 fin_d[kMaxPrimes];
  // register passes: blockIdx.y enumerates units (segment, limb, chunk of
  // ppb polys); all polys of a unit share the prime, hence the twiddles
  int ppb;
  int unit_start[kMaxSeg + 1];
  int unit0;  // first unit of this launch (L2-sized chunks of a large batch)
};

// unit -> (segment, limb, first poly, poly count)
struct UnitPos {
  int s, limb, p0, np;
};
__device__ __forceinline__ UnitPos unit_pos(const NttParams& P, int unit) {
  UnitPos u;
  int s = 0;
#pragma unroll 1
  while (s + 1 < P.S.n_seg && unit >= P.unit_start[s + 1]) ++s;
  const Seg& sg = P.S.seg[s];
  const int r = unit - P.unit_start[s];
  const int chunk = r / sg.k;
  u.s = s;
  u.limb = r - chunk * sg.k;
  u.p0 = chunk * P.ppb;
  u.np = min(P.ppb, sg.n_polys - u.p0);
  return u;
}

template <bool INV>
__global__ void __launch_bounds__(256) k_ntt_cols(const __grid_constant__ NttParams P) {
  extern __shared__ uint64_t sm[];
  const int log_n = P.log_n, N = 1 << log_n, a = P.a, R = 1 << a, C = N >> a;
  const int cpb_log = P.tile_log, CPB = 1 << cpb_log;
  const int row = blockIdx.y;
  const int s = find_seg(P.S, row);
  const Seg& sg = P.S.seg[s];
  const int rr = row - sg.row_start;
  const int poly = rr / sg.k, limb = rr - poly * sg.k;
  const int prime = P.S.sel[s][limb];
  const PrimeConst pc = P.pc[prime];
  const uint64_t q = pc.q, q2 = q << 1;
  // twiddles are (w, w') Shoup pairs, bit-reversed order, forward then inverse
  const ulonglong2* tw =
      reinterpret_cast<const ulonglong2*>(P.tw + (size_t)prime * 4 * N + (INV ? 2 * (size_t)N : 0));
  const uint64_t* src = INV ? (sg.out + poly * sg.out_stride + (size_t)limb * N)
                            : (sg.in + poly * sg.in_stride + (size_t)limb * N);
  uint64_t* dst = sg.out + poly * sg.out_stride + (size_t)limb * N;
  const int c0 = blockIdx.x << cpb_log;
  const int tile = R << cpb_log;
  for (int e = threadIdx.x; e < tile; e += blockDim.x) {
    const int r = e >> cpb_log, c = e & (CPB - 1);
    sm[e] = src[c0 + c + (size_t)C * r];
  }
  __syncthreads();
  const int nb = tile >> 1;
  if (!INV) {
    for (int st = 0; st < a; ++st) {
      const int hl = a - st - 1;  // log2 of the row distance
      const int hr = 1 << hl;
      for (int b = threadIdx.x; b < nb; b += blockDim.x) {
        const int c = b & (CPB - 1), bi = b >> cpb_log;
        const int grp = bi >> hl, off = bi & (hr - 1);
        const int r0 = (grp << (hl + 1)) + off;
        const int ti = (1 << st) + grp;
        const int i0 = (r0 << cpb_log) + c, i1 = i0 + (hr << cpb_log);
        uint64_t x = sm[i0];
        const uint64_t y = sm[i1];
        x = x >= q2 ? x - q2 : x;
        const ulonglong2 wp = tw[ti];
        const uint64_t v = shoup_lazy(y, wp.x, wp.y, q);
        sm[i0] = x + v;
        sm[i1] = x - v + q2;
      }
      __syncthreads();
    }
  } else {
    const int u0 = log_n - a;
    for (int st = 0; st < a; ++st) {
      const int u = u0 + st;
      const int tr = 1 << st;
      const int h = N >> (u + 1);
      const bool last = (st == a - 1);
      for (int b = threadIdx.x; b < nb; b += blockDim.x) {
        const int c = b & (CPB - 1), bi = b >> cpb_log;
        const int grp = bi >> st, off = bi & (tr - 1);
        const int r0 = (grp << (st + 1)) + off;
        const int i0 = (r0 << cpb_log) + c, i1 = i0 + (tr << cpb_log);
        const uint64_t x = sm[i0], y = sm[i1];
        uint64_t sum = x + y;
        sum = sum >= q2 ? sum - q2 : sum;
        const uint64_t d = x - y + q2;
        if (!last) {
          const int ti = h + grp;
          sm[i0] = sum;
          const ulonglong2 wp = tw[ti];
          sm[i1] = shoup_lazy(d, wp.x, wp.y, q);
        } else {
          sm[i0] = shoup(sum, pc.ninv, pc.ninv_sh, q);
          sm[i1] = shoup(d, pc.ilast, pc.ilast_sh, q);
        }
      }
      __syncthreads();
    }
  }
  for (int e = threadIdx.x; e < tile; e += blockDim.x) {
    const int r = e >> cpb_log, c = e & (CPB - 1);
    dst[c0 + c + (size_t)C * r] = sm[e];
  }
}

template <bool INV>
__global__ void __launch_bounds__(256) k_ntt_blocks(const __grid_constant__ NttParams P) {
  extern __shared__ uint64_t sm[];
  const int log_n = P.log_n, N = 1 << log_n, a = P.a;
  const int B = N >> a, blog = log_n - a;
  const int bpc_log = P.tile_log;
  const int row = blockIdx.y;
  const int s = find_seg(P.S, row);
  const Seg& sg = P.S.seg[s];
  const int rr = row - sg.row_start;
  const int poly = rr / sg.k, limb = rr - poly * sg.k;
  const int prime = P.S.sel[s][limb];
  const PrimeConst pc = P.pc[prime];
  const uint64_t q = pc.q, q2 = q << 1;
  // twiddles are (w, w') Shoup pairs, bit-reversed order, forward then inverse
  const ulonglong2* tw =
      reinterpret_cast<const ulonglong2*>(P.tw + (size_t)prime * 4 * N + (INV ? 2 * (size_t)N : 0));
  const uint64_t* src = INV ? (sg.in + poly * sg.in_stride + (size_t)limb * N)
                            : (sg.out + poly * sg.out_stride + (size_t)limb * N);
  uint64_t* dst = sg.out + poly * sg.out_stride + (size_t)limb * N;
  const int blk0 = blockIdx.x << bpc_log;
  const int tile = B << bpc_log;
  const size_t base = (size_t)blk0 * B;
  for (int e = threadIdx.x; e < tile; e += blockDim.x) sm[e] = src[base + e];
  __syncthreads();
  const int nb = tile >> 1;
  const int hb_log = blog - 1;  // log2(B/2)
  if (!INV) {
    for (int st = a; st < log_n; ++st) {
      const int tl = log_n - st - 1;  // log2 t
      const int t = 1 << tl;
      for (int b = threadIdx.x; b < nb; b += blockDim.x) {
        const int bl = b >> hb_log, bi = b & ((1 << hb_log) - 1);
        const int grp = bi >> tl, off = bi & (t - 1);
        const int l0 = (grp << (tl + 1)) + off;
        const int ti = (1 << st) + ((blk0 + bl) << (blog - tl - 1)) + grp;
        const int i0 = (bl << blog) + l0, i1 = i0 + t;
        uint64_t x = sm[i0];
        const uint64_t y = sm[i1];
        x = x >= q2 ? x - q2 : x;
        const ulonglong2 wp = tw[ti];
        const uint64_t v = shoup_lazy(y, wp.x, wp.y, q);
        sm[i0] = x + v;
        sm[i1] = x - v + q2;
      }
      __syncthreads();
    }
    if (P.epi) {
      const uint64_t* other = sg.other + poly * sg.other_stride + (size_t)limb * N + base;
      uint64_t* eout = sg.eout + poly * sg.eout_stride + (size_t)limb * N + base;
      const uint64_t cc = P.c[limb], ccsh = P.csh[limb];
      for (int e = threadIdx.x; e < tile; e += blockDim.x) {
        uint64_t y = sm[e];
        y = y >= q2 ? y - q2 : y;
        y = y >= q ? y - q : y;
        uint64_t r = shoup(other[e] + q - y, cc, ccsh, q);
        if (sg.eacc == 1) r = add_mod(r, eout[e], q);
        if (sg.eacc == 2) {
          const uint64_t* ein = sg.ein + poly * sg.ein_stride + (size_t)limb * N + base;
          r = add_mod(r, shoup(ein[e], P.es[limb], P.essh[limb], q), q);
        }
        eout[e] = r;
      }
      return;
    }
    for (int e = threadIdx.x; e < tile; e += blockDim.x) {
      uint64_t y = sm[e];
      y = y >= q2 ? y - q2 : y;
      y = y >= q ? y - q : y;
      dst[base + e] = y;
    }
  } else {
    for (int u = 0; u < blog; ++u) {
      const int t = 1 << u;
      const int h = N >> (u + 1);
      for (int b = threadIdx.x; b < nb; b += blockDim.x) {
        const int bl = b >> hb_log, bi = b & ((1 << hb_log) - 1);
        const int grp = bi >> u, off = bi & (t - 1);
        const int l0 = (grp << (u + 1)) + off;
        const int ti = h + ((blk0 + bl) << (blog - u - 1)) + grp;
        const int i0 = (bl << blog) + l0, i1 = i0 + t;
        const uint64_t x = sm[i0], y = sm[i1];
        uint64_t sum = x + y;
        sum = sum >= q2 ? sum - q2 : sum;
        sm[i0] = sum;
        const ulonglong2 wp = tw[ti];
        sm[i1] = shoup_lazy(x - y + q2, wp.x, wp.y, q);
      }
      __syncthreads();
    }
    for (int e = threadIdx.x; e < tile; e += blockDim.x) dst[base + e] = sm[e];
  }
}

// ---------------------------------------------------------------------------
// register-radix passes (N >= 2^12): one warp per S-point sub-transform
// ---------------------------------------------------------------------------

#ifndef HEGPU_REG_WARPS_LOG
#define HEGPU_REG_WARPS_LOG 3
#endif
constexpr int kRegWarpsLog = HEGPU_REG_WARPS_LOG;  // warps (sub-transforms) per CTA, log2
constexpr int kRegWarps = 1 << kRegWarpsLog;
constexpr int kRegMinBlocks = 8 / kRegWarps;  // scales the launch bounds below
#ifndef HEGPU_NTT_PPB
#define HEGPU_NTT_PPB 4
#endif
constexpr int kNttPolysPerCta = HEGPU_NTT_PPB;
// conversion prologue: up to this many source limbs take the unrolled path
// (all source words of a coefficient in flight at once)
constexpr int kConvMaxSrc = 8;
#ifndef HEGPU_NTT_BULK
#define HEGPU_NTT_BULK 0  // measured: 76.5 ms per train step with it, 75.1 without (3 vs 4 CTAs/SM)
#endif
#ifndef HEGPU_BLOCKS_MINB
// 3 with the bulk-prefetch buffers (their shared memory fits 3 CTAs per SM)
#define HEGPU_BLOCKS_MINB (HEGPU_NTT_BULK ? 3 : 4)
#endif
#ifndef HEGPU_CONV_HYBRID
#define HEGPU_CONV_HYBRID 0
#endif
// column passes at 4 CTAs/SM (64 registers): measured 95.5 ms per training
// step vs 96.9 at 5 (48 registers, the conversion prologues spilled)
#ifndef HEGPU_COLS_MINB
#define HEGPU_COLS_MINB 4
#endif

// slot -> (st << 16 | local) of TwLayout<6 + li, inv>, filled once by the host
// (the staging loops then do one table read per twiddle instead of a decode)
__device__ int32_t g_tw_slot[2][4][512];

template <int LOGS, bool INV>
__device__ __forceinline__ int tw_slot_index(int i, int blk_shift_base) {
  const int code = g_tw_slot[INV][LOGS - 6][i];
  const int st = code >> 16, local = code & 0xffff;
  return (1 << (blk_shift_base + st)) + local;
}

template <int LOGS, bool INV>
static void fill_tw_slots(std::vector<int32_t>& h) {
  for (int i = 0; i < (1 << LOGS) - 1; ++i) {
    int st, local;
    TwLayout<LOGS, INV>::decode(i, st, local);
    h[((INV ? 1 : 0) * 4 + (LOGS - 6)) * 512 + i] = (st << 16) | local;
  }
}

void ensure_tw_slots() {
  static std::once_flag once;
  std::call_once(once, [] {
    std::vector<int32_t> h(2 * 4 * 512, 0);
    fill_tw_slots<6, false>(h); fill_tw_slots<7, false>(h);
    fill_tw_slots<8, false>(h); fill_tw_slots<9, false>(h);
    fill_tw_slots<6, true>(h); fill_tw_slots<7, true>(h);
    fill_tw_slots<8, true>(h); fill_tw_slots<9, true>(h);
    check_cuda(cudaMemcpyToSymbol(g_tw_slot, h.data(), h.size() * sizeof(int32_t)),
               "twiddle slot table");
  });
}

// Shared memory of the register passes (bytes): the cols pass holds its
// S x 8 tile, the warp buffers and the S twiddle pairs of stages [0, LOGS);
// the blocks pass holds the warp buffers and its 8 blocks' twiddle pairs
// (8 * S, re-based so block-local index = (8 << st) + (warp << st) + i).
template <int LOGS>
constexpr size_t cols_r_smem() {
  return ((size_t)(1 << LOGS) * (kRegWarps + 1) + kRegWarps * RegShape<LOGS>::PAD_S) * 8 +
         (size_t)(1 << LOGS) * 16 + kConvMaxSrc * 3 * 8 + kConvMaxSrc * 16;
}
// blocks pass: each warp's next-poly block is prefetched into shared memory
// by a bulk copy (TMA engine) while the current one is transformed
template <int LOGS>
constexpr size_t blocks_r_smem() {
  return (size_t)kRegWarps * RegShape<LOGS>::PAD_S * 8 +
         (size_t)kRegWarps * (1 << LOGS) * 16 +
         (HEGPU_NTT_BULK ? (size_t)kRegWarps * ((1 << LOGS) * 8 + 16) : 0);
}

// CM: first-pass input -- 0 plain load, 1 centered lift of one limb
// (rescale / ModRaise), 2 fast basis conversion, 3 conversion of the centered
// representative (ModDown by q_l * P), 4 signed int64 coefficients
// (limbs_from_signed, ring.py:381-387: encoded plaintexts).  Compile-time so each variant carries
// only its own prologue.
template <int LOGS, bool INV, int CM>
__global__ void __launch_bounds__(32 * kRegWarps, (LOGS >= 9 ? 2 : HEGPU_COLS_MINB) * kRegMinBlocks) k_ntt_cols_r(const __grid_constant__ NttParams P) {
  static_assert(!INV || CM == 0, "prologues are forward-only");
  using Sh = RegShape<LOGS>;
  constexpr int S = Sh::S, E = Sh::E, EB = Sh::EB;
  constexpr int TS = kRegWarps + 1;  // padded tile row (conflict-free column reads)
  extern __shared__ uint64_t sm[];
  const int log_n = P.log_n, N = 1 << log_n, C = N >> LOGS;
  const UnitPos U = unit_pos(P, blockIdx.y + P.unit0);
  const Seg& sg = P.S.seg[U.s];
  const int limb = U.limb;
  const int prime = P.S.sel[U.s][limb];
  const PrimeConst pc = P.pc[prime];
  // twiddles are (w, w') Shoup pairs, bit-reversed order, forward then inverse
  const ulonglong2* tw =
      reinterpret_cast<const ulonglong2*>(P.tw + (size_t)prime * 4 * N + (INV ? 2 * (size_t)N : 0));
  uint64_t* tile = sm;
  // tile slot of (row r, column c): with 8 columns an XOR swizzle makes both
  // the row-wise fill and the column-wise register load conflict-free
  auto tix = [](int r, int c) {
    if constexpr (kRegWarps == 8) return r * 8 + (c ^ ((r >> 1) & 7));
    else return r * TS + c;
  };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* wbuf = sm + S * TS + warp * Sh::PAD_S;
  ulonglong2* stw = reinterpret_cast<ulonglong2*>(sm + S * TS + kRegWarps * Sh::PAD_S);
  // FP64 path for primes below 2^kFpMaxBits: (w, w/q) twiddles, same layout
  const bool fpp = pc.twf != nullptr;
  const ulonglong2* tws =
      fpp ? reinterpret_cast<const ulonglong2*>(pc.twf + (INV ? N : 0)) : tw;
  // every column transform of this pass uses twiddles [1, S) of its table,
  // staged in consumption order (TwLayout)
  for (int i = threadIdx.x; i < S - 1; i += blockDim.x)
    cp_async16(stw + i, tws + tw_slot_index<LOGS, INV>(i, 0));
  // conversion constants of this target limb: punc[i], fp32 weight, shift
  uint64_t* s_conv = reinterpret_cast<uint64_t*>(stw + S);
  const int nsrc = CM >= 2 ? sg.c_nsrc : 0;
  for (int i = threadIdx.x; i < nsrc && i < kConvMaxSrc; i += blockDim.x) {
    s_conv[i] = __ldg(sg.cpunc + i * sg.cpunc_ld + limb);
    if (CM == 2 && pc.twf != nullptr && sg.c_fp_src)  // natural-form constant, split
      reinterpret_cast<double2*>(s_conv + 3 * kConvMaxSrc)[i] =
          fp_split23(mont_mul(s_conv[i], 1, pc.q, pc.qinv_neg));
    if (CM == 3) {
      s_conv[kConvMaxSrc + i] = __ldg(reinterpret_cast<const uint64_t*>(sg.cfw) + i);
      s_conv[2 * kConvMaxSrc + i] = __ldg(reinterpret_cast<const uint64_t*>(sg.cfs) + i);
    }
  }
  __syncthreads();
  const int c0 = blockIdx.x * kRegWarps;
  constexpr bool centered = CM == 3;
  const uint64_t negd = centered ? __ldg(sg.cnegd + limb) : 0;
  const ulonglong2 fs = P.post ? P.fin_s[limb] : make_ulonglong2(pc.ninv, pc.ninv_sh);
  const ulonglong2 fd = P.post ? P.fin_d[limb] : make_ulonglong2(pc.ilast, pc.ilast_sh);
#pragma unroll 1
  for (int pi = 0; pi < U.np; ++pi) {
    const int poly = U.p0 + pi;
    const uint64_t* src = INV ? (sg.out + poly * sg.out_stride + (size_t)limb * N)
                              : (sg.in + poly * sg.in_stride + (size_t)limb * N);
    uint64_t* dst = sg.out + poly * sg.out_stride + (size_t)limb * N;
    if constexpr (CM == 4) {
      const int64_t* hs = reinterpret_cast<const int64_t*>(sg.csrc + poly * sg.csrc_stride);
      for (int e = threadIdx.x; e < S * kRegWarps; e += blockDim.x) {
        const int r = e / kRegWarps, c = e % kRegWarps;
        tile[tix(r, c)] = signed_mod(__ldg(hs + c0 + c + (size_t)C * r), pc);
      }
    } else if constexpr (CM == 1) {
      // fused centered lift: v = src > q_s/2 ? src - q_s : src, then mod q
      const uint64_t* hs = sg.csrc + poly * sg.csrc_stride;
      const uint64_t qs = sg.csrc_q;
      for (int e = threadIdx.x; e < S * kRegWarps; e += blockDim.x) {
        const int r = e / kRegWarps, c = e % kRegWarps;
        const uint64_t u = __ldg(hs + c0 + c + (size_t)C * r);
        const int64_t v = u > (qs >> 1) ? (int64_t)u - (int64_t)qs : (int64_t)u;
        tile[tix(r, c)] = signed_mod(v, pc);
      }
    } else if constexpr (CM >= 2) {
      // fused fast basis conversion: out_t = REDC(sum_i hat_i * punc_mont[i][t])
      const uint64_t* hs = sg.csrc + poly * sg.csrc_stride;
      const uint64_t q = pc.q;
      if (CM == 2 && nsrc <= kConvMaxSrc && HEGPU_CONV_HYBRID && pc.twf != nullptr &&
          sg.c_fp_src) {
        // hybrid: odd sources as FP64 split products (FP64 pipe), even ones
        // in the 128-bit integer MAC (IMAD / ALU pipes); both exact
        const double2* s_convf = reinterpret_cast<const double2*>(s_conv + 3 * kConvMaxSrc);
        const FpSplitConst fc = fp_split_const(q);
#pragma unroll 2
        for (int e = threadIdx.x; e < S * kRegWarps; e += blockDim.x) {
          const int r = e / kRegWarps, c = e % kRegWarps;
          const size_t x = c0 + c + (size_t)C * r;
          uint64_t h[kConvMaxSrc];
#pragma unroll
          for (int i = 0; i < kConvMaxSrc; ++i) h[i] = i < nsrc ? __ldg(hs + (size_t)i * N + x) : 0;
          Mac128 acc;
          acc.zero();
          FpSplitAcc fa;
          fa.zero();
#pragma unroll
          for (int i = 0; i < kConvMaxSrc; ++i) {
            if (i < nsrc) {
              if (i & 1)
                fa.add(fp_split23(h[i]), s_convf[i]);
              else
                acc.add(h[i], s_conv[i]);
            }
          }
          tile[tix(r, c)] =
              add_mod(acc.redc(pc), fp_to_residue_small(fp_split_fold(fa, fc), fc.q), q);
        }
      } else if (nsrc <= kConvMaxSrc) {
        // unrolled: the nsrc source words of each coefficient load together
#pragma unroll 2
        for (int e = threadIdx.x; e < S * kRegWarps; e += blockDim.x) {
          const int r = e / kRegWarps, c = e % kRegWarps;
          const size_t x = c0 + c + (size_t)C * r;
          uint64_t h[kConvMaxSrc];
#pragma unroll
          for (int i = 0; i < kConvMaxSrc; ++i) h[i] = i < nsrc ? __ldg(hs + (size_t)i * N + x) : 0;
          Mac128 acc;
          acc.zero();
          float f = 0.f;
#pragma unroll
          for (int i = 0; i < kConvMaxSrc; ++i) {
            if (i < nsrc) {
              acc.add(h[i], s_conv[i]);
              if (centered) {
                const uint64_t wbits = s_conv[kConvMaxSrc + i];
                const int sh = (int)s_conv[2 * kConvMaxSrc + i];
                f = fmaf(__uint2float_rn(static_cast<uint32_t>(h[i] >> sh)),
                         __uint_as_float(static_cast<uint32_t>(wbits)), f);
              }
            }
          }
          if (centered) {
            if (nsrc == kConvMaxSrc) acc.fold(q, pc.bar);
            acc.add(static_cast<uint64_t>(__float2int_rn(f)), negd);
          }
          tile[tix(r, c)] = acc.redc(pc);
        }
      } else
      for (int e = threadIdx.x; e < S * kRegWarps; e += blockDim.x) {
        const int r = e / kRegWarps, c = e % kRegWarps;
        const size_t x = c0 + c + (size_t)C * r;
        Mac128 acc;
        acc.zero();
        float f = 0.f;
        for (int i = 0; i < sg.c_nsrc; ++i) {
          const uint64_t h = __ldg(hs + (size_t)i * N + x);
          const uint64_t m = __ldg(sg.cpunc + i * sg.cpunc_ld + limb);
          acc.add(h, m);
          if (centered)
            f = fmaf(__uint2float_rn(static_cast<uint32_t>(h >> __ldg(sg.cfs + 2 * i))),
                     __ldg(sg.cfw + 2 * i), f);
          if (i % kMacFold == kMacFold - 1) acc.fold(q, pc.bar);
        }
        if (centered) {
          if (sg.c_nsrc % kMacFold == 0) acc.fold(q, pc.bar);
          acc.add(static_cast<uint64_t>(__float2int_rn(f)), negd);
        }
        tile[tix(r, c)] = acc.redc(pc);
      }
    } else {
      for (int e = threadIdx.x; e < S * kRegWarps; e += blockDim.x) {
        const int r = e / kRegWarps, c = e % kRegWarps;
        tile[tix(r, c)] = src[c0 + c + (size_t)C * r];
      }
    }
    if (pi == 0) cp_async_wait_all();
    __syncthreads();
    constexpr int LO_S = LOGS - EB;  // strided window: j = lane + 32 e
    uint64_t x[E];
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = tile[tix(reg_j(lane, e, LO_S, EB), warp)];
    if (fpp) {
      // forward: [0, q) in, lazy double intermediate (raw bits) out; inverse:
      // the double intermediate in, fully reduced out
      const double qd = (double)pc.q, qinv = 1.0 / qd;
      double xf[E];
#pragma unroll
      for (int e = 0; e < E; ++e) xf[e] = INV ? __longlong_as_double(x[e]) : fp_from_s64(x[e]);
      const double2* stwf = reinterpret_cast<const double2*>(stw);
      double* wbf = reinterpret_cast<double*>(wbuf);
      if (!INV) {
        fwd_sub_fp<LOGS>(xf, wbf, lane, LO_S, LO_S, stwf, qd);
#pragma unroll
        for (int e = 0; e < E; ++e) x[e] = __double_as_longlong(xf[e]);
      } else {
        const double2 fsf = make_double2((double)fs.x, (double)fs.x / qd);
        const double2 fdf = make_double2((double)fd.x, (double)fd.x / qd);
        inv_sub_fp<LOGS>(xf, wbf, lane, LO_S, LO_S, LOGS - 1, stwf, qd, qinv, fsf, fdf);
#pragma unroll
        for (int e = 0; e < E; ++e) x[e] = fp_to_residue_small(xf[e], qd);
      }
    } else if (!INV)
      fwd_sub<LOGS>(x, wbuf, lane, LO_S, LO_S, stw, pc.q);
    else
      inv_sub<LOGS>(x, wbuf, lane, LO_S, LO_S, LOGS - 1, stw, pc, fs, fd);
#pragma unroll
    for (int e = 0; e < E; ++e) tile[tix(reg_j(lane, e, LO_S, EB), warp)] = x[e];
    __syncthreads();
    for (int e = threadIdx.x; e < S * kRegWarps; e += blockDim.x) {
      const int r = e / kRegWarps, c = e % kRegWarps;
      dst[c0 + c + (size_t)C * r] = tile[tix(r, c)];
    }
    if (pi + 1 < U.np) __syncthreads();  // the tile is reloaded for the next poly
  }
}

template <int LOGS, bool INV>
__global__ void __launch_bounds__(32 * kRegWarps, (LOGS >= 9 ? 2 : HEGPU_BLOCKS_MINB) * kRegMinBlocks) k_ntt_blocks_r(const __grid_constant__ NttParams P) {
  using Sh = RegShape<LOGS>;
  constexpr int S = Sh::S, E = Sh::E, EB = Sh::EB;
  extern __shared__ uint64_t sm[];
  const int log_n = P.log_n, N = 1 << log_n, a = log_n - LOGS;
  const UnitPos U = unit_pos(P, blockIdx.y + P.unit0);
  const Seg& sg = P.S.seg[U.s];
  const int limb = U.limb;
  const int prime = P.S.sel[U.s][limb];
  const PrimeConst pc = P.pc[prime];
  const uint64_t q = pc.q, q2 = q << 1;
  // twiddles are (w, w') Shoup pairs, bit-reversed order, forward then inverse
  const ulonglong2* tw =
      reinterpret_cast<const ulonglong2*>(P.tw + (size_t)prime * 4 * N + (INV ? 2 * (size_t)N : 0));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int blk = blockIdx.x * kRegWarps + warp;
  const size_t off = (size_t)limb * N + (size_t)blk * S;
  uint64_t* wbuf = sm + warp * Sh::PAD_S;
  ulonglong2* stw = reinterpret_cast<ulonglong2*>(sm + kRegWarps * Sh::PAD_S);
  constexpr int LO_S = LOGS - EB;
  const bool fpp = pc.twf != nullptr;  // FP64 path (common.cuh)
  {
    const ulonglong2* tws =
        fpp ? reinterpret_cast<const ulonglong2*>(pc.twf + (INV ? N : 0)) : tw;
    // warp w's sub-transform (block blk0 + w) uses global twiddles
    // (1 << (a + st)) + ((blk0 + w) << st) + local, staged per warp in
    // consumption order (TwLayout): smem run w * (S - 1) + slot
    const int blk0 = blockIdx.x * kRegWarps;
    for (int v = threadIdx.x; v < kRegWarps * (S - 1); v += blockDim.x) {
      const int w = v / (S - 1), i = v - w * (S - 1);
      const int code = g_tw_slot[INV][LOGS - 6][i];
      const int st = code >> 16, local = code & 0xffff;
      cp_async16(stw + v, tws + (1 << (a + st)) + ((blk0 + w) << st) + local);
    }
  }
  const uint64_t cc = P.epi ? P.c[limb] : 0, ccsh = P.epi ? P.csh[limb] : 0;
  auto src_of = [&](int poly) {
    return INV ? (sg.in + poly * sg.in_stride + off) : (sg.out + poly * sg.out_stride + off);
  };
  auto load = [&](uint64_t (&x)[E], int poly) {
    const uint64_t* src = src_of(poly);
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = src[lane + 32 * e];
  };
  // bulk prefetch: this warp's S-word block of the next poly lands in pbuf
  // (mbarrier bar) while the current poly is transformed in registers
  uint64_t* pbuf = reinterpret_cast<uint64_t*>(stw + kRegWarps * (S - 1)) + (size_t)warp * S;
  uint64_t* pbar =
      reinterpret_cast<uint64_t*>(stw + kRegWarps * (S - 1)) + (size_t)kRegWarps * S + warp * 2;
  if (HEGPU_NTT_BULK) {
    if (lane == 0) {
      mbar_init(pbar, 1);
      mbar_init_fence();
      mbar_expect_tx(pbar, S * 8);
      bulk_g2s(pbuf, src_of(U.p0), S * 8, pbar);
    }
    __syncwarp();
  }
  auto finish = [&](uint64_t (&x)[E], int poly) {
    uint64_t* dst = sg.out + poly * sg.out_stride + off;
    if (!INV) {
      if (P.epi) {
        const uint64_t* other = sg.other + poly * sg.other_stride + off;
        uint64_t* eout = sg.eout + poly * sg.eout_stride + off;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          uint64_t y = x[e];
          y = y >= q2 ? y - q2 : y;
          y = y >= q ? y - q : y;
          uint64_t r = shoup(other[lane + 32 * e] + q - y, cc, ccsh, q);
          if (sg.eacc == 1) r = add_mod(r, eout[lane + 32 * e], q);
          if (sg.eacc == 2)
            r = add_mod(r, shoup(sg.ein[poly * sg.ein_stride + off + lane + 32 * e],
                                 P.es[limb], P.essh[limb], q),
                        q);
          eout[lane + 32 * e] = r;
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          uint64_t y = x[e];
          y = y >= q2 ? y - q2 : y;
          dst[lane + 32 * e] = y >= q ? y - q : y;
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) dst[lane + 32 * e] = x[e];
    }
  };
  // re-based twiddle table for the inverse: log_n' = LOGS + log2(warps) (the
  // last-stage scaling is never in this pass)
  const ulonglong2 fs = make_ulonglong2(pc.ninv, pc.ninv_sh);
  const ulonglong2 fd = make_ulonglong2(pc.ilast, pc.ilast_sh);
  const ulonglong2* tab = stw + warp * (S - 1);  // this warp's consumption-order run
  uint64_t x[E];
#pragma unroll 1
  for (int pi = 0; pi < U.np; ++pi) {
    if (HEGPU_NTT_BULK) {
      mbar_wait(pbar, pi & 1);
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = pbuf[lane + 32 * e];
      __syncwarp();
      if (lane == 0 && pi + 1 < U.np) {  // refill the buffer with the next poly's block
        fence_proxy_async_smem();
        mbar_expect_tx(pbar, S * 8);
        bulk_g2s(pbuf, src_of(U.p0 + pi + 1), S * 8, pbar);
      }
    } else {
      load(x, U.p0 + pi);
    }
    if (pi == 0) {
      cp_async_wait_all();
      __syncthreads();
    }
    if (fpp) {
      // forward: double intermediate (raw bits) in, fully reduced out;
      // inverse: [0, q) in, double intermediate (|x| < q) out
      const double qd = (double)q, qinv = 1.0 / qd;
      double xf[E];
#pragma unroll
      for (int e = 0; e < E; ++e) xf[e] = INV ? fp_from_s64(x[e]) : __longlong_as_double(x[e]);
      const double2* tabf = reinterpret_cast<const double2*>(tab);
      double* wbf = reinterpret_cast<double*>(wbuf);
      if (!INV) {
        fwd_sub_fp<LOGS>(xf, wbf, lane, LO_S, LO_S, tabf, qd);
#pragma unroll
        for (int e = 0; e < E; ++e) x[e] = fp_to_residue(xf[e], qd, qinv);
      } else {
        const double2 one = make_double2(1.0, 1.0 / qd);  // never used: no final stage here
        inv_sub_fp<LOGS>(xf, wbf, lane, LO_S, LO_S, -1, tabf, qd, qinv, one, one);
#pragma unroll
        for (int e = 0; e < E; ++e) x[e] = __double_as_longlong(xf[e]);
      }
    } else if (!INV) {
      fwd_sub<LOGS>(x, wbuf, lane, LO_S, LO_S, tab, q);
    } else {
      inv_sub<LOGS>(x, wbuf, lane, LO_S, LO_S, -1, tab, pc, fs, fd);
    }
    finish(x, U.p0 + pi);
  }
}

// ---------------------------------------------------------------------------
// Fused inverse NTT for N = S^2 (2^16): one thread-block CLUSTER of
// kFuseCluster CTAs owns one (poly, limb).  Pass B (row blocks: the GS stages
// with span < S) leaves the intermediate in the cluster's distributed shared
// memory -- CTA c holds rows [c*ROWS, (c+1)*ROWS) -- and after one cluster
// barrier pass A (columns: the last stages, N^-1 / post-scale) fills its
// 8-column tiles over DSMEM.  The intermediate never reaches HBM (one read and
// one write per coefficient instead of two of each).  Same butterflies and
// twiddles as k_ntt_blocks_r / k_ntt_cols_r, so the limbs are identical.
// ---------------------------------------------------------------------------
#ifndef HEGPU_INTT_FUSED
#define HEGPU_INTT_FUSED 0
#endif
#ifndef HEGPU_INTT_CLUSTER
#define HEGPU_INTT_CLUSTER 16  // 16 (non-portable): 86 KiB smem, 2 CTAs per SM
#endif
constexpr int kFuseCluster = HEGPU_INTT_CLUSTER;
constexpr int kFuseTwBufs = kFuseCluster >= 16 ? 1 : 2;  // per-warp twiddle runs in pass B

template <int LOGS>
struct FusedLayout {
  static constexpr int S = 1 << LOGS;
  static constexpr int ROWS = S / kFuseCluster;          // rows (and columns) per CTA
  static constexpr int RPW = ROWS / kRegWarps;           // rows per warp in pass B
  static constexpr int TILES = ROWS / kRegWarps;         // 8-column tiles in pass A
  static constexpr size_t t_words = (size_t)ROWS * S;    // this CTA's rows (DSMEM-shared)
  static constexpr size_t wb_words = (size_t)kRegWarps * RegShape<LOGS>::PAD_S;
  static constexpr size_t stw_words = (size_t)(S - 1) * 2;           // pass-A twiddles
  static constexpr size_t twb_words = (size_t)kRegWarps * kFuseTwBufs * (S - 1) * 2;  // pass B
  static constexpr size_t tile_words = (size_t)S * kRegWarps * TILES;
  static constexpr size_t region_words = twb_words > tile_words ? twb_words : tile_words;
  static constexpr size_t bar_words = kRegWarps;
  static constexpr size_t bytes =
      (t_words + wb_words + stw_words + region_words + bar_words) * 8;
};

template <int LOGS>
__global__ void __cluster_dims__(kFuseCluster, 1, 1) __launch_bounds__(32 * kRegWarps, kFuseCluster >= 16 ? 2 : 1)
    k_intt_fused(const __grid_constant__ NttParams P) {
  namespace cg = cooperative_groups;
  using Sh = RegShape<LOGS>;
  using L = FusedLayout<LOGS>;
  constexpr int S = Sh::S, E = Sh::E, EB = Sh::EB;
  constexpr int LO_S = LOGS - EB;
  constexpr int ROWS = L::ROWS, RPW = L::RPW;
  extern __shared__ __align__(128) uint64_t sm[];
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = (int)cluster.block_rank();
  const int log_n = P.log_n, N = 1 << log_n, a = log_n - LOGS;  // N == S * S
  const UnitPos U = unit_pos(P, blockIdx.y + P.unit0);           // ppb == 1: one poly
  const Seg& sg = P.S.seg[U.s];
  const int limb = U.limb, poly = U.p0;
  const int prime = P.S.sel[U.s][limb];
  const PrimeConst pc = P.pc[prime];
  const uint64_t q = pc.q;
  const ulonglong2* tw =
      reinterpret_cast<const ulonglong2*>(P.tw + (size_t)prime * 4 * N + 2 * (size_t)N);
  const bool fpp = pc.twf != nullptr;
  const ulonglong2* tws = fpp ? reinterpret_cast<const ulonglong2*>(pc.twf + N) : tw;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* T = sm;
  uint64_t* wbuf = T + L::t_words + warp * Sh::PAD_S;
  ulonglong2* stw = reinterpret_cast<ulonglong2*>(T + L::t_words + L::wb_words);
  uint64_t* region = T + L::t_words + L::wb_words + L::stw_words;
  uint64_t* bars = region + L::region_words;
  const uint64_t* src = sg.in + poly * sg.in_stride + (size_t)limb * N;
  uint64_t* dst = sg.out + poly * sg.out_stride + (size_t)limb * N;
  const double qd = (double)q, qinv = 1.0 / qd;
  uint64_t x[E];

  // ---- pass B: warp w transforms rows crank*ROWS + w*RPW + [0, RPW) in T ----
  // the warp's RPW contiguous rows arrive by one bulk copy; per-row twiddle
  // runs are double-buffered with cp.async, so only __syncwarp is needed
  const int row0 = crank * ROWS + warp * RPW;
  uint64_t* trows = T + (size_t)warp * RPW * S;
  uint64_t* bar = bars + warp;
  if (lane == 0) {
    mbar_init(bar, 1);
    mbar_init_fence();
    mbar_expect_tx(bar, RPW * S * 8);
    bulk_g2s(trows, src + (size_t)row0 * S, RPW * S * 8, bar);
  }
  // pass-A twiddles: every column transform uses [1, S) of the table
  for (int i = threadIdx.x; i < S - 1; i += blockDim.x)
    cp_async16(stw + i, tws + tw_slot_index<LOGS, true>(i, 0));
  ulonglong2* twb = reinterpret_cast<ulonglong2*>(region) + (size_t)warp * kFuseTwBufs * (S - 1);
  auto stage = [&](int i) {
    ulonglong2* d = twb + (i % kFuseTwBufs) * (S - 1);
    const int blk = row0 + i;
    for (int v = lane; v < S - 1; v += 32) {
      const int code = g_tw_slot[1][LOGS - 6][v];
      const int st = code >> 16, local = code & 0xffff;
      cp_async16(d + v, tws + (1 << (a + st)) + (blk << st) + local);
    }
    cp_async_commit();
  };
  stage(0);
  if (kFuseTwBufs > 1 && RPW > 1) stage(1);
  __syncwarp();
  mbar_wait(bar, 0);
#pragma unroll 1
  for (int i = 0; i < RPW; ++i) {
    if (kFuseTwBufs > 1 && i + 1 < RPW) cp_async_wait_group<1>(); else cp_async_wait_group<0>();
    __syncwarp();
    const ulonglong2* tab = twb + (i % kFuseTwBufs) * (S - 1);
    uint64_t* trow = trows + (size_t)i * S;
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = trow[lane + 32 * e];
    if (fpp) {
      double xf[E];
#pragma unroll
      for (int e = 0; e < E; ++e) xf[e] = fp_from_s64(x[e]);
      const double2 one = make_double2(1.0, 1.0 / qd);  // no final stage in this pass
      inv_sub_fp<LOGS>(xf, reinterpret_cast<double*>(wbuf), lane, LO_S, LO_S, -1,
                       reinterpret_cast<const double2*>(tab), qd, qinv, one, one);
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = __double_as_longlong(xf[e]);
    } else {
      const ulonglong2 fs = make_ulonglong2(pc.ninv, pc.ninv_sh);
      const ulonglong2 fd = make_ulonglong2(pc.ilast, pc.ilast_sh);
      inv_sub<LOGS>(x, wbuf, lane, LO_S, LO_S, -1, tab, pc, fs, fd);
    }
#pragma unroll
    for (int e = 0; e < E; ++e) trow[lane + 32 * e] = x[e];
    __syncwarp();  // this row's twiddle buffer is consumed
    if (i + kFuseTwBufs < RPW) stage(i + kFuseTwBufs);
  }
  cp_async_wait_all();
  cluster.sync();  // every CTA's rows are in place (and visible cluster-wide)

  // ---- pass A: this CTA's ROWS columns as TILES tiles of 8 -----------------
  // gather the whole 256 x ROWS block over DSMEM (16-byte loads), then each
  // warp runs one column transform per tile
  auto tix = [](int t, int r, int c) {
    return (size_t)t * S * 8 + r * 8 + (c ^ ((r >> 1) & 7));
  };
  uint64_t* tile = region;
  const int cbase = crank * ROWS;
  constexpr int PAIRS = S * ROWS / 2;
#pragma unroll 4
  for (int e = threadIdx.x; e < PAIRS; e += blockDim.x) {
    const int r = e / (ROWS / 2), cp = (e % (ROWS / 2)) * 2;
    const uint64_t* rs = cluster.map_shared_rank(T, r / ROWS);
    const ulonglong2 v =
        *reinterpret_cast<const ulonglong2*>(rs + (size_t)(r % ROWS) * S + cbase + cp);
    const int t = cp >> 3, c = cp & 7;
    tile[tix(t, r, c)] = v.x;
    tile[tix(t, r, c + 1)] = v.y;
  }
  __syncthreads();
  const ulonglong2 fs = P.post ? P.fin_s[limb] : make_ulonglong2(pc.ninv, pc.ninv_sh);
  const ulonglong2 fd = P.post ? P.fin_d[limb] : make_ulonglong2(pc.ilast, pc.ilast_sh);
#pragma unroll 1
  for (int t = 0; t < L::TILES; ++t) {
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = tile[tix(t, reg_j(lane, e, LO_S, EB), warp)];
    if (fpp) {
      double xf[E];
#pragma unroll
      for (int e = 0; e < E; ++e) xf[e] = __longlong_as_double(x[e]);
      const double2 fsf = make_double2((double)fs.x, (double)fs.x / qd);
      const double2 fdf = make_double2((double)fd.x, (double)fd.x / qd);
      inv_sub_fp<LOGS>(xf, reinterpret_cast<double*>(wbuf), lane, LO_S, LO_S, LOGS - 1,
                       reinterpret_cast<const double2*>(stw), qd, qinv, fsf, fdf);
#pragma unroll
      for (int e = 0; e < E; ++e) x[e] = fp_to_residue_small(xf[e], qd);
    } else {
      inv_sub<LOGS>(x, wbuf, lane, LO_S, LO_S, LOGS - 1, stw, pc, fs, fd);
    }
#pragma unroll
    for (int e = 0; e < E; ++e) tile[tix(t, reg_j(lane, e, LO_S, EB), warp)] = x[e];
  }
  __syncthreads();
#pragma unroll 4
  for (int e = threadIdx.x; e < PAIRS; e += blockDim.x) {
    const int r = e / (ROWS / 2), cp = (e % (ROWS / 2)) * 2;
    const int t = cp >> 3, c = cp & 7;
    *reinterpret_cast<ulonglong2*>(dst + (size_t)S * r + cbase + cp) =
        make_ulonglong2(tile[tix(t, r, c)], tile[tix(t, r, c + 1)]);
  }
  cluster.sync();  // no CTA leaves while others still read its rows
}

template <int LOGS, bool INV, int CM>
static void launch_cols_r_cm(const NttParams& P, dim3 grid, cudaStream_t st) {
  const size_t smem = cols_r_smem<LOGS>();
  static bool attr_set = false;  // opt in to > 48 KiB dynamic shared memory once
  if (!attr_set) {
    check_cuda(cudaFuncSetAttribute(k_ntt_cols_r<LOGS, INV, CM>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "smem attr");
    attr_set = true;
  }
  k_ntt_cols_r<LOGS, INV, CM><<<grid, 32 * kRegWarps, smem, st>>>(P);
}

// the first-pass prologue every segment of the launch shares
static int cols_mode(const NttParams& P) {
  int cm = -1;
  for (int g = 0; g < P.S.n_seg; ++g) {
    const Seg& sg = P.S.seg[g];
    const int m = sg.csrc == nullptr ? 0
                  : sg.cmode == 1   ? 1
                  : sg.cmode == 2   ? 3
                  : sg.cmode == 3   ? 4
                                    : 2;
    if (cm >= 0 && m != cm) throw HegpuError{HEGPU_E_ARG, "NTT segments mix prologue modes"};
    cm = m;
  }
  return cm < 0 ? 0 : cm;
}

template <int LOGS>
static void launch_cols_r(bool inverse, const NttParams& P, int n_units, int log_n,
                          cudaStream_t st) {
  const int C = (1 << log_n) >> LOGS;
  dim3 grid(C / kRegWarps, n_units);
  if (inverse) {
    launch_cols_r_cm<LOGS, true, 0>(P, grid, st);
    return;
  }
  switch (cols_mode(P)) {
    case 1: launch_cols_r_cm<LOGS, false, 1>(P, grid, st); break;
    case 2: launch_cols_r_cm<LOGS, false, 2>(P, grid, st); break;
    case 3: launch_cols_r_cm<LOGS, false, 3>(P, grid, st); break;
    case 4: launch_cols_r_cm<LOGS, false, 4>(P, grid, st); break;
    default: launch_cols_r_cm<LOGS, false, 0>(P, grid, st); break;
  }
}

template <int LOGS>
static void launch_blocks_r(bool inverse, const NttParams& P, int n_units, int log_n,
                            cudaStream_t st) {
  const int R = (1 << log_n) >> LOGS;
  dim3 grid(R / kRegWarps, n_units);
  const size_t smem = blocks_r_smem<LOGS>();
  static bool attr_set = false;
  if (!attr_set) {
    check_cuda(cudaFuncSetAttribute(k_ntt_blocks_r<LOGS, true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "smem attr");
    check_cuda(cudaFuncSetAttribute(k_ntt_blocks_r<LOGS, false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "smem attr");
    attr_set = true;
  }
  if (inverse)
    k_ntt_blocks_r<LOGS, true><<<grid, 32 * kRegWarps, smem, st>>>(P);
  else
    k_ntt_blocks_r<LOGS, false><<<grid, 32 * kRegWarps, smem, st>>>(P);
}

static void cols_r(int logs, bool inverse, const NttParams& P, int n_rows, int log_n,
                   cudaStream_t st) {
  switch (logs) {
    case 6: launch_cols_r<6>(inverse, P, n_rows, log_n, st); break;
    case 7: launch_cols_r<7>(inverse, P, n_rows, log_n, st); break;
    case 8: launch_cols_r<8>(inverse, P, n_rows, log_n, st); break;
    case 9: launch_cols_r<9>(inverse, P, n_rows, log_n, st); break;
    default: throw HegpuError{HEGPU_E_ARG, "unsupported NTT column size"};
  }
}

static void blocks_r(int logs, bool inverse, const NttParams& P, int n_rows, int log_n,
                     cudaStream_t st) {
  switch (logs) {
    case 6: launch_blocks_r<6>(inverse, P, n_rows, log_n, st); break;
    case 7: launch_blocks_r<7>(inverse, P, n_rows, log_n, st); break;
    case 8: launch_blocks_r<8>(inverse, P, n_rows, log_n, st); break;
    case 9: launch_blocks_r<9>(inverse, P, n_rows, log_n, st); break;
    default: throw HegpuError{HEGPU_E_ARG, "unsupported NTT block size"};
  }
}

static inline bool P_epi_guard(const NttEpilogue* e) { return e && e->enabled; }

static inline int ilog2(int x) {
  int r = 0;
  while ((1 << r) < x) ++r;
  return r;
}

static bool intt_fused_enabled() {
  static const bool on = [] {
    const char* e = getenv("HEGPU_INTT_FUSED");
    return e ? e[0] == '1' : (HEGPU_INTT_FUSED != 0);
  }();
  return on;
}

template <int LOGS>
static void launch_intt_fused(const NttParams& P, int n_units, cudaStream_t st) {
  const size_t smem = FusedLayout<LOGS>::bytes;
  static bool attr_set = false;
  if (!attr_set) {
    if (kFuseCluster > 8)
      check_cuda(cudaFuncSetAttribute(k_intt_fused<LOGS>,
                                      cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                 "cluster attr");
    check_cuda(cudaFuncSetAttribute(k_intt_fused<LOGS>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "smem attr");
    attr_set = true;
  }
  k_intt_fused<LOGS><<<dim3(kFuseCluster, n_units), 32 * kRegWarps, smem, st>>>(P);
}

void launch_ntt(const PrimeConst* dpc, const uint64_t* dtw, int log_n, bool inverse,
                SegSet& S, const NttEpilogue* epi, cudaStream_t st, const uint64_t* fp_mask) {
  // one kernel per pass serves both arithmetic classes (a per-CTA uniform
  // branch on PrimeConst::twf): measured faster than a launch per class,
  // whose integer-limb launches are too small to fill the GPU
  (void)fp_mask;
  if (S.n_rows == 0) return;
  ensure_tw_slots();
  if (S.n_rows > 65535) throw HegpuError{1, "NTT batch exceeds 65535 limbs"};
  NttParams local;
  local.S = S;
  local.pc = dpc;
  local.tw = dtw;
  local.log_n = log_n;
  local.unit0 = 0;
  const int a = (log_n + 1) / 2;
  local.a = a;
  local.epi = (epi && epi->enabled) ? 1 : 0;
  if (local.epi) {
    for (int i = 0; i < kMaxPrimes; ++i) {
      local.c[i] = epi->c[i];
      local.csh[i] = epi->csh[i];
      local.es[i] = epi->s[i];
      local.essh[i] = epi->ssh[i];
    }
  }
  local.post = (epi && epi->post) ? 1 : 0;
  if (local.post) {
    for (int i = 0; i < kMaxPrimes; ++i) {
      local.fin_s[i] = epi->fin_s[i];
      local.fin_d[i] = epi->fin_d[i];
    }
  }
  bool has_conv = false;
  for (int g = 0; g < S.n_seg; ++g) has_conv |= S.seg[g].csrc != nullptr;
  if ((has_conv || local.post) && log_n < 12)
    throw HegpuError{HEGPU_E_ARG, "fused conversion / post-scale needs N >= 2^12"};
  if (has_conv && inverse) throw HegpuError{HEGPU_E_ARG, "conversion prologue is forward-only"};
  if (local.post && !inverse) throw HegpuError{HEGPU_E_ARG, "post-scale is inverse-only"};
  const int N = 1 << log_n, R = 1 << a, C = N >> a;
  const int kTile = 4096;
  int cpb = kTile / R;
  if (cpb < 1) cpb = 1;
  if (cpb > C) cpb = C;
  int bpc = kTile / C;
  if (bpc < 1) bpc = 1;
  if (bpc > R) bpc = R;
  const int tile_a = R * cpb, tile_b = C * bpc;
  const int thr_a = tile_a / 2 < 256 ? tile_a / 2 : 256;
  const int thr_b = tile_b / 2 < 256 ? tile_b / 2 : 256;
  dim3 grid_a(C / cpb, S.n_rows), grid_b(R / bpc, S.n_rows);
  NttParams pa = local, pb = local;
  const double rows = S.n_rows, nn = N;
  const double bytes_pass = rows * nn * 8.0;  // half of the transform's read+write
  const double mm_a = rows * nn / 2 * a + (inverse ? rows * nn : 0.0);
  const double mm_b = rows * nn / 2 * (log_n - a) + ((P_epi_guard(epi)) ? rows * nn : 0.0);
  pa.tile_log = ilog2(cpb);
  pb.tile_log = ilog2(bpc);
  if (inverse && log_n == 16 && intt_fused_enabled()) {
    // one cluster per (poly, limb): units with one poly each
    int n_units = 0;
    for (int g = 0; g < S.n_seg; ++g) {
      pa.unit_start[g] = n_units;
      n_units += S.seg[g].k * S.seg[g].n_polys;
    }
    pa.unit_start[S.n_seg] = n_units;
    pa.ppb = 1;
    pa.unit0 = 0;
    if (n_units > 65535) throw HegpuError{1, "NTT batch exceeds 65535 units"};
    ProfScope ps(PROF_NTT, st, bytes_pass, rows * nn / 2 * log_n + rows * nn);
    launch_intt_fused<8>(pa, n_units, st);
    check_cuda(cudaGetLastError(), "fused intt launch");
    return;
  }
  if (log_n >= 12) {
    const int logs_b = log_n - a;
    // units: (segment, limb, chunk of ppb polys); a unit's polys share the
    // twiddles and the CTA prologue
    int max_polys = 1;
    for (int g = 0; g < S.n_seg; ++g) max_polys = std::max(max_polys, S.seg[g].n_polys);
    const int ppb = std::max(1, std::min(kNttPolysPerCta, max_polys));
    int n_units = 0;
    for (int g = 0; g < S.n_seg; ++g) {
      pa.unit_start[g] = pb.unit_start[g] = n_units;
      n_units += S.seg[g].k * ((S.seg[g].n_polys + ppb - 1) / ppb);
    }
    pa.unit_start[S.n_seg] = pb.unit_start[S.n_seg] = n_units;
    pa.ppb = pb.ppb = ppb;
    if (n_units > 65535) throw HegpuError{1, "NTT batch exceeds 65535 units"};
    // HEGPU_NTT_CHUNK_MB > 0 runs a large batch in chunks of units whose
    // pass-1 output fits in L2 (the second pass then reads it from L2, not
    // HBM).  Off: measured slower on the training step (97.3 ms unchunked,
    // 102.6 ms at 80 MiB, 111.5 ms at 48 MiB): the smaller launches lose more
    // to tails than the L2 hits save.
    static const long chunk_bytes = [] {
      const char* e = getenv("HEGPU_NTT_CHUNK_MB");
      return (e ? atol(e) : 0L) << 20;
    }();
    const long unit_bytes = (long)ppb * N * 8;
    int chunk = n_units;
    if (chunk_bytes > 0 && (long)n_units * unit_bytes > 2 * chunk_bytes)
      chunk = (int)std::max(1L, chunk_bytes / unit_bytes);
    for (int u0 = 0; u0 < n_units; u0 += chunk) {
      const int nu = std::min(chunk, n_units - u0);
      const double f = (double)nu / n_units;
      pa.unit0 = pb.unit0 = u0;
      if (!inverse) {
        pa.epi = 0;
        {
          ProfScope ps(PROF_NTT, st, bytes_pass * f, mm_a * f);
          cols_r(a, false, pa, nu, log_n, st);
        }
        ProfScope ps(PROF_NTT, st, bytes_pass * (P_epi_guard(epi) ? 1.5 : 1.0) * f, mm_b * f);
        blocks_r(logs_b, false, pb, nu, log_n, st);
      } else {
        {
          ProfScope ps(PROF_NTT, st, bytes_pass * f, rows * nn / 2 * (log_n - a) * f);
          blocks_r(logs_b, true, pb, nu, log_n, st);
        }
        ProfScope ps(PROF_NTT, st, bytes_pass * f, mm_a * f);
        cols_r(a, true, pa, nu, log_n, st);
      }
    }
    check_cuda(cudaGetLastError(), "ntt launch");
    return;
  }
  if (!inverse) {
    pa.epi = 0;
    {
      ProfScope ps(PROF_NTT, st, bytes_pass, mm_a);
      k_ntt_cols<false><<<grid_a, thr_a, tile_a * 8, st>>>(pa);
    }
    // the epilogue reads one more operand per element
    ProfScope ps(PROF_NTT, st, bytes_pass * (P_epi_guard(epi) ? 1.5 : 1.0), mm_b);
    k_ntt_blocks<false><<<grid_b, thr_b, tile_b * 8, st>>>(pb);
  } else {
    {
      ProfScope ps(PROF_NTT, st, bytes_pass, rows * nn / 2 * (log_n - a));
      k_ntt_blocks<true><<<grid_b, thr_b, tile_b * 8, st>>>(pb);
    }
    ProfScope ps(PROF_NTT, st, bytes_pass, mm_a);
    k_ntt_cols<true><<<grid_a, thr_a, tile_a * 8, st>>>(pa);
  }
  check_cuda(cudaGetLastError(), "ntt launch");
}

}  // namespace hegpu
