// numpy-compatible PCG64 uniform residues on the device (sm_100a).
//
// Key generation draws every switching-key digit's `a` part as
// Generator.integers(0, q, size=N, dtype=uint64) per limb (hebert/ckks/keys.py
// 133-151 via ring.sample_poly, ring.py:494-498): 1.8 M bounded 64-bit draws
// per digit at N = 2^16, ~9 s of host time for the trainer's key set.  The
// reference's stream is reproduced exactly:
//   * PCG64 (numpy's pcg64.h): 128-bit LCG state' = state * M + inc, output
//     XSL-RR: rotr64(hi ^ lo, state >> 122), one step per 64-bit draw;
//   * bounded draws (numpy's random_bounded_uint64, Lemire without masking):
//     m = x * q (128-bit); x is rejected iff (m mod 2^64) < (2^64 - q) mod q,
//     else the value is m >> 64.
// Each thread jumps (O(log d) LCG composition) to its first draw and then
// steps sequentially.  Rejections (probability < q / 2^64, well under one per
// key) shift every later draw by one: the host loop re-runs the fill with the
// rejected raw positions known until none is new.  The caller advances its
// numpy generator by the returned number of draws, so later host draws
// (gaussians, other keys) continue the same stream.
#include <algorithm>
#include <vector>

#include "ring.cuh"

namespace hegpu {

typedef unsigned __int128 u128;

constexpr int kPcgPerThread = 16;
constexpr int kPcgMaxRej = 64;  // rejected raw positions per fill (expected: ~0)
constexpr int kPcgMaxBounds = 64;

struct PcgParams {
  u128 state, inc;  // generator state before the fill
  long long n_out;  // k * n outputs
  int n, k;
  int n_rej;
  long long rej[kPcgMaxRej];  // sorted raw indices already known to be rejected
  uint64_t q[kPcgMaxBounds], thr[kPcgMaxBounds];
  uint64_t* out;
  int64_t out_stride;          // between limbs
  unsigned long long* flag;   // min new rejected raw index (ULLONG_MAX: none)
};

__host__ __device__ inline u128 pcg_mult() {
  return ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
}

// state after `delta` LCG steps (pcg_advance_lcg_128)
__device__ inline u128 pcg_advance(u128 state, u128 inc, unsigned long long delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

__device__ inline uint64_t pcg_output(u128 s) {
  const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  const unsigned rot = (unsigned)(s >> 122);
  const uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

__global__ void __launch_bounds__(256) k_pcg_uniform(const __grid_constant__ PcgParams P) {
  const long long i0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * kPcgPerThread;
  if (i0 >= P.n_out) return;
  // raw index of output i0: skip the known rejections at or before it
  long long j = i0;
  int r = 0;
  while (r < P.n_rej && P.rej[r] <= j) {
    ++j;
    ++r;
  }
  u128 s = pcg_advance(P.state, P.inc, (unsigned long long)j + 1);  // draw j uses state_{j+1}
  const u128 M = pcg_mult();
  const long long i1 = min(i0 + kPcgPerThread, P.n_out);
  for (long long i = i0; i < i1; ++i) {
    while (r < P.n_rej && P.rej[r] == j) {  // a known rejection: consume the draw
      s = s * M + P.inc;
      ++j;
      ++r;
    }
    const int l = (int)(i / P.n);
    const uint64_t q = P.q[l];
    const u128 m = (u128)pcg_output(s) * q;
    if ((uint64_t)m < P.thr[l]) atomicMin(P.flag, (unsigned long long)j);
    P.out[(size_t)l * P.out_stride + (i - (long long)l * P.n)] = (uint64_t)(m >> 64);
    s = s * M + P.inc;
    ++j;
  }
}

long long pcg64_uniform_fill(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                             uint64_t inc_lo, const uint64_t* bounds, int k, int n,
                             uint64_t* out, int64_t out_stride, cudaStream_t st) {
  if (k < 1 || k > kPcgMaxBounds || n < 1) throw HegpuError{HEGPU_E_ARG, "pcg64: bad shape"};
  PcgParams P;
  P.state = ((u128)state_hi << 64) | state_lo;
  P.inc = ((u128)inc_hi << 64) | inc_lo;
  P.n = n;
  P.k = k;
  P.n_out = (long long)k * n;
  P.n_rej = 0;
  P.out = out;
  P.out_stride = out_stride;
  for (int l = 0; l < k; ++l) {
    const uint64_t q = bounds[l];
    if (q <= 0xFFFFFFFFull)
      throw HegpuError{HEGPU_E_ARG, "pcg64: bounds <= 2^32 use numpy's 32-bit path"};
    P.q[l] = q;
    P.thr[l] = (uint64_t)(0 - q) % q;  // (2^64 - q) mod q
  }
  unsigned long long* dflag = nullptr;
  check_cuda(cudaMallocAsync(reinterpret_cast<void**>(&dflag), sizeof(unsigned long long), st),
             "pcg flag");
  P.flag = dflag;
  const long long threads = (P.n_out + kPcgPerThread - 1) / kPcgPerThread;
  for (;;) {
    const unsigned long long none = ~0ull;
    check_cuda(cudaMemcpyAsync(dflag, &none, sizeof(none), cudaMemcpyHostToDevice, st),
               "pcg flag reset");
    {
      ProfScope ps(PROF_ENCRYPT, st, (double)P.n_out * 8.0, 0);
      k_pcg_uniform<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(P);
    }
    check_cuda(cudaGetLastError(), "pcg launch");
    unsigned long long flag = 0;
    check_cuda(cudaMemcpyAsync(&flag, dflag, sizeof(flag), cudaMemcpyDeviceToHost, st),
               "pcg flag read");
    check_cuda(cudaStreamSynchronize(st), "pcg sync");
    if (flag == ~0ull) break;
    // the earliest new rejection is certain; later ones are re-evaluated
    if (P.n_rej == kPcgMaxRej) throw HegpuError{HEGPU_E_ARG, "pcg64: too many rejections"};
    P.rej[P.n_rej++] = (long long)flag;
    std::sort(P.rej, P.rej + P.n_rej);
  }
  cudaFreeAsync(dflag, st);
  return P.n_out + P.n_rej;
}


// ---------------------------------------------------------------------------
// Encryption randomness for UNSEEDED encryptions (the reference draws v, e0,
// e1 from numpy's Generator seeded by OS entropy there: ops.py:87-100,
// logreg.py:151-156, bootstrap.py:367 -- never reproducible, so there is no
// stream to match).  The host supplies 64 bits of OS entropy; the device
// expands them with the counter-based Philox4x32-10 generator:
//   v  = ternary, uniform on {-1, 0, 1}   (ring.py:499-501)
//   e0, e1 = rint(N(0, sigma^2))          (ring.py:507-509), Box-Muller
// Seeded encryptions keep numpy on the host (bit-exact with the reference).
// ---------------------------------------------------------------------------
struct Philox {
  uint32_t c[4];
};

__device__ __forceinline__ Philox philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                uint32_t k0, uint32_t k1) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
    const uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
    k0 += W0;
    k1 += W1;
  }
  Philox o;
  o.c[0] = c0;
  o.c[1] = c1;
  o.c[2] = c2;
  o.c[3] = c3;
  return o;
}

__device__ __forceinline__ double u01_53(uint32_t a, uint32_t b) {  // (0, 1]
  const uint64_t x = ((uint64_t)a << 21) ^ (uint64_t)b;  // 53 bits
  return ((double)(x & ((1ull << 53) - 1)) + 1.0) * 0x1.0p-53;
}

__global__ void __launch_bounds__(256) k_sample_encrypt(int64_t* out, int n, uint64_t seed,
                                                        double sigma) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  // one Philox block per (coefficient, draw): counters never repeat
  const Philox t = philox4x32_10((uint32_t)x, 0u, 0x7e3a11u, 0u, k0, k1);
  const Philox g = philox4x32_10((uint32_t)x, 1u, 0x7e3a11u, 0u, k0, k1);
  // ternary: floor(3 u / 2^32) - 1 (bias 2^-32)
  out[x] = (int64_t)((((uint64_t)t.c[0]) * 3u) >> 32) - 1;
  // Box-Muller: two independent N(0, 1) from two 53-bit uniforms
  const double u1 = u01_53(g.c[0], g.c[1]), u2 = u01_53(g.c[2], g.c[3]);
  const double r = sqrt(-2.0 * log(u1)) * sigma;
  double sn, cs;
  sincospi(2.0 * u2, &sn, &cs);
  out[n + x] = (int64_t)rint(r * cs);
  out[2 * n + x] = (int64_t)rint(r * sn);
}

void sample_encrypt(int64_t* out, int n, uint64_t seed, double sigma, cudaStream_t st) {
  if (n <= 0 || sigma <= 0.0) throw HegpuError{HEGPU_E_ARG, "sample_encrypt: n > 0, sigma > 0"};
  k_sample_encrypt<<<(n + 255) / 256, 256, 0, st>>>(out, n, seed, sigma);
  check_cuda(cudaGetLastError(), "sample_encrypt launch");
}

}  // namespace hegpu
