// Elementwise / gather / basis-conversion / key-switch inner-product kernels.
//
// All kernels are HBM-bound streaming kernels over limb-major uint64 data:
// each thread owns 2 consecutive coefficients (128-bit loads/stores) of one
// limb; grid.y enumerates (poly, limb) rows.  Reference semantics are cited
// per kernel.
#include "ring.cuh"

namespace hegpu {

constexpr int kEwThreads = 256;

struct EwParams {
  const uint64_t* a;
  const uint64_t* b;
  uint64_t* o;
  int64_t as, bs, os;
  int k;
  int log_n;
  int rows;  // n_polys * k: the last grid.z slice may overhang
  const PrimeConst* pc;
  uint8_t sel[kMaxPrimes];
  uint64_t c[kMaxPrimes];
  uint64_t csh[kMaxPrimes];
};

// One row = one limb of one poly; 2 coefficients per thread.
template <int OP>
__global__ void __launch_bounds__(kEwThreads) k_elementwise(const __grid_constant__ EwParams P) {
  const int N = 1 << P.log_n;
  const int row = blockIdx.y + blockIdx.z * 65535;
  if (row >= P.rows) return;
  const int poly = row / P.k, limb = row - poly * P.k;
  const int x = (blockIdx.x * kEwThreads + threadIdx.x) * 2;
  if (x >= N) return;
  const PrimeConst pc = P.pc[P.sel[limb]];
  const uint64_t q = pc.q;
  const size_t la = (size_t)limb * N + x;
  const ulonglong2 va = *reinterpret_cast<const ulonglong2*>(P.a + poly * P.as + la);
  ulonglong2 vb = make_ulonglong2(0, 0);
  if (OP == HEGPU_OP_ADD || OP == HEGPU_OP_SUB || OP == HEGPU_OP_MUL || OP == HEGPU_OP_MONT ||
      OP == HEGPU_OP_FMA || OP == HEGPU_OP_AXPYC)
    vb = *reinterpret_cast<const ulonglong2*>(P.b + poly * P.bs + la);
  uint64_t* op = P.o + poly * P.os + la;
  ulonglong2 r;
  if (OP == HEGPU_OP_ADD) {
    r.x = add_mod(va.x, vb.x, q);
    r.y = add_mod(va.y, vb.y, q);
  } else if (OP == HEGPU_OP_SUB) {
    r.x = sub_mod(va.x, vb.x, q);
    r.y = sub_mod(va.y, vb.y, q);
  } else if (OP == HEGPU_OP_MUL) {
    r.x = mul_mod(va.x, vb.x, pc);
    r.y = mul_mod(va.y, vb.y, pc);
  } else if (OP == HEGPU_OP_MONT) {
    r.x = mont_mul(va.x, vb.x, q, pc.qinv_neg);
    r.y = mont_mul(va.y, vb.y, q, pc.qinv_neg);
  } else if (OP == HEGPU_OP_NEG) {
    r.x = va.x ? q - va.x : 0;
    r.y = va.y ? q - va.y : 0;
  } else if (OP == HEGPU_OP_SCALAR) {
    r.x = shoup(va.x, P.c[limb], P.csh[limb], q);
    r.y = shoup(va.y, P.c[limb], P.csh[limb], q);
  } else if (OP == HEGPU_OP_ROWMONT) {
    r.x = mont_mul(va.x, P.c[limb], q, pc.qinv_neg);
    r.y = mont_mul(va.y, P.c[limb], q, pc.qinv_neg);
  } else if (OP == HEGPU_OP_REDUCE) {
    r.x = reduce64(va.x, pc);
    r.y = reduce64(va.y, pc);
  } else if (OP == HEGPU_OP_ADDC) {
    r.x = add_mod(va.x, P.c[limb], q);
    r.y = add_mod(va.y, P.c[limb], q);
  } else if (OP == HEGPU_OP_AXPYC) {
    r.x = add_mod(vb.x, shoup(va.x, P.c[limb], P.csh[limb], q), q);
    r.y = add_mod(vb.y, shoup(va.y, P.c[limb], P.csh[limb], q), q);
  } else if (OP == HEGPU_OP_FMA) {
    const ulonglong2 acc = *reinterpret_cast<const ulonglong2*>(op);
    r.x = add_mod(acc.x, mul_mod(va.x, vb.x, pc), q);
    r.y = add_mod(acc.y, mul_mod(va.y, vb.y, pc), q);
  } else {  // COPY
    r = va;
  }
  *reinterpret_cast<ulonglong2*>(op) = r;
}

static dim3 rows_grid(int n, int rows, int per_thread) {
  int gx = (n / per_thread + kEwThreads - 1) / kEwThreads;
  if (gx < 1) gx = 1;
  int gy = rows < 65535 ? rows : 65535;
  int gz = (rows + 65534) / 65535;
  return dim3(gx, gy, gz);
}

void launch_elementwise(const PrimeConst* dpc, const std::vector<uint64_t>& hq, int log_n,
                        const EwArgs& A, cudaStream_t st) {
  const int rows = A.n_polys * A.k;
  if (rows == 0) return;
  if (A.k > kMaxPrimes) throw HegpuError{HEGPU_E_ARG, "too many limbs"};
  EwParams P;
  P.a = A.a;
  P.b = A.b;
  P.o = A.o;
  P.as = A.as;
  P.bs = A.bs;
  P.os = A.os;
  P.k = A.k;
  P.log_n = log_n;
  P.rows = rows;
  P.pc = dpc;
  for (int l = 0; l < A.k; ++l) {
    const int p = A.primes[l];
    if (p < 0 || p >= (int)hq.size()) throw HegpuError{HEGPU_E_ARG, "prime index out of range"};
    P.sel[l] = (uint8_t)p;
    if (A.consts) {
      const uint64_t q = hq[p];
      P.c[l] = A.consts[l];
      if (A.op == HEGPU_OP_SCALAR || A.op == HEGPU_OP_ADDC || A.op == HEGPU_OP_AXPYC) {
        if (A.consts[l] >= q) throw HegpuError{HEGPU_E_ARG, "scalar not reduced"};
        P.csh[l] = h_shoup(A.consts[l], q);
      }
    }
  }
  if ((A.op == HEGPU_OP_SCALAR || A.op == HEGPU_OP_ROWMONT || A.op == HEGPU_OP_ADDC ||
       A.op == HEGPU_OP_AXPYC) &&
      !A.consts)
    throw HegpuError{HEGPU_E_ARG, "scalar op needs consts"};
  const int n = 1 << log_n;
  if (n < 2) throw HegpuError{HEGPU_E_ARG, "N too small"};
  const dim3 grid = rows_grid(n, rows, 2);
  const bool two_in = A.op == HEGPU_OP_ADD || A.op == HEGPU_OP_SUB || A.op == HEGPU_OP_MUL ||
                      A.op == HEGPU_OP_MONT || A.op == HEGPU_OP_FMA || A.op == HEGPU_OP_AXPYC;
  const double ew_elems = (double)rows * n;
  const double ew_mm = (A.op == HEGPU_OP_MUL || A.op == HEGPU_OP_FMA) ? 2 * ew_elems
                       : (A.op == HEGPU_OP_MONT || A.op == HEGPU_OP_SCALAR ||
                          A.op == HEGPU_OP_ROWMONT) ? ew_elems : 0.0;
  ProfScope ps(PROF_ELEMENTWISE, st,
               ew_elems * 8.0 * ((two_in ? 2 : 1) + (A.op == HEGPU_OP_FMA ? 2 : 1)), ew_mm);
  switch (A.op) {
    case HEGPU_OP_ADD: k_elementwise<HEGPU_OP_ADD><<<grid, kEwThreads, 0, st>>>(P); break;
    case HEGPU_OP_SUB: k_elementwise<HEGPU_OP_SUB><<<grid, kEwThreads, 0, st>>>(P); break;
    case HEGPU_OP_MUL: k_elementwise<HEGPU_OP_MUL><<<grid, kEwThreads, 0, st>>>(P); break;
    case HEGPU_OP_MONT: k_elementwise<HEGPU_OP_MONT><<<grid, kEwThreads, 0, st>>>(P); break;
    case HEGPU_OP_NEG: k_elementwise<HEGPU_OP_NEG><<<grid, kEwThreads, 0, st>>>(P); break;
    case HEGPU_OP_SCALAR: k_elementwise<HEGPU_OP_SCALAR><<<grid, kEwThreads, 0, st>>>(P); break;
    case HEGPU_OP_ROWMONT: k_elementwise<HEGPU_OP_ROWMONT><<<grid, kEwThreads, 0, st>>>(P); break;
    case HEGPU_OP_FMA: k_elementwise<HEGPU_OP_FMA><<<grid, kEwThreads, 0, st>>>(P); break;
    case HEGPU_OP_COPY: k_elementwise<HEGPU_OP_COPY><<<grid, kEwThreads, 0, st>>>(P); break;
    case HEGPU_OP_ADDC: k_elementwise<HEGPU_OP_ADDC><<<grid, kEwThreads, 0, st>>>(P); break;
    case HEGPU_OP_REDUCE: k_elementwise<HEGPU_OP_REDUCE><<<grid, kEwThreads, 0, st>>>(P); break;
    case HEGPU_OP_AXPYC: k_elementwise<HEGPU_OP_AXPYC><<<grid, kEwThreads, 0, st>>>(P); break;
    default: throw HegpuError{HEGPU_E_ARG, "unknown elementwise op"};
  }
  check_cuda(cudaGetLastError(), "elementwise launch");
}

// ---------------------------------------------------------------------------
// lifts (limbs_from_signed, ring.py:381-387; centered lifts ops.py:170-173)
// ---------------------------------------------------------------------------

struct LiftParams {
  const void* src;
  int64_t ss;
  uint64_t* out;
  int64_t os;
  int k;
  int log_n;
  uint64_t src_q;  // centered mode: modulus of the source limb
  const PrimeConst* pc;
  uint8_t sel[kMaxPrimes];
};

template <bool CENTERED>
__global__ void __launch_bounds__(kEwThreads) k_lift(const __grid_constant__ LiftParams P) {
  const int N = 1 << P.log_n;
  const int poly = blockIdx.y;
  const int x = blockIdx.x * kEwThreads + threadIdx.x;
  if (x >= N) return;
  int64_t v;
  if (CENTERED) {
    const uint64_t u = reinterpret_cast<const uint64_t*>(P.src)[poly * P.ss + x];
    v = u > (P.src_q >> 1) ? (int64_t)u - (int64_t)P.src_q : (int64_t)u;
  } else {
    v = reinterpret_cast<const int64_t*>(P.src)[poly * P.ss + x];
  }
  uint64_t* o = P.out + poly * P.os + x;
  for (int l = 0; l < P.k; ++l) o[(size_t)l * N] = signed_mod(v, P.pc[P.sel[l]]);
}

static void fill_sel(uint8_t* sel, const int32_t* primes, int k) {
  if (k > kMaxPrimes) throw HegpuError{HEGPU_E_ARG, "too many limbs"};
  for (int l = 0; l < k; ++l) {
    if (primes[l] < 0 || primes[l] >= kMaxPrimes) throw HegpuError{HEGPU_E_ARG, "bad prime index"};
    sel[l] = (uint8_t)primes[l];
  }
}

void launch_lift_signed(const PrimeConst* dpc, int log_n, const int64_t* src, int64_t ss,
                        uint64_t* out, int64_t os, int n_polys, int k, const int32_t* primes,
                        cudaStream_t st) {
  if (n_polys == 0 || k == 0) return;
  if (n_polys > 65535) throw HegpuError{HEGPU_E_ARG, "lift batch exceeds 65535 polys"};
  LiftParams P;
  P.src = src;
  P.ss = ss;
  P.out = out;
  P.os = os;
  P.k = k;
  P.log_n = log_n;
  P.src_q = 0;
  P.pc = dpc;
  fill_sel(P.sel, primes, k);
  const int n = 1 << log_n;
  dim3 grid((n + kEwThreads - 1) / kEwThreads, n_polys);
  ProfScope ps(PROF_LIFT, st, (double)n_polys * n * 8.0 * (1 + k), (double)n_polys * n * k);
  k_lift<false><<<grid, kEwThreads, 0, st>>>(P);
  check_cuda(cudaGetLastError(), "lift launch");
}

void launch_lift_centered(const PrimeConst* dpc, int log_n, const uint64_t* src, int64_t ss,
                          uint64_t src_q, uint64_t* out, int64_t os, int n_polys, int k,
                          const int32_t* primes, cudaStream_t st) {
  if (n_polys == 0 || k == 0) return;
  if (n_polys > 65535) throw HegpuError{HEGPU_E_ARG, "lift batch exceeds 65535 polys"};
  LiftParams P;
  P.src = src;
  P.ss = ss;
  P.out = out;
  P.os = os;
  P.k = k;
  P.log_n = log_n;
  P.src_q = src_q;
  P.pc = dpc;
  fill_sel(P.sel, primes, k);
  const int n = 1 << log_n;
  dim3 grid((n + kEwThreads - 1) / kEwThreads, n_polys);
  ProfScope ps(PROF_LIFT, st, (double)n_polys * n * 8.0 * (1 + k), (double)n_polys * n * k);
  k_lift<true><<<grid, kEwThreads, 0, st>>>(P);
  check_cuda(cudaGetLastError(), "lift launch");
}

// ---------------------------------------------------------------------------
// automorphisms (ring.py:416-482)
// ---------------------------------------------------------------------------

struct AutoParams {
  const uint64_t* in;
  uint64_t* out;
  int64_t is, os;
  int k;
  int log_n;
  int rows;  // n_polys * k: the last grid.z slice may overhang
  uint64_t g;  // odd, reduced mod 2N
  const PrimeConst* pc;
  uint8_t sel[kMaxPrimes];
};

// Eval form: slot i holds p(psi^(2 brev(i) + 1)); X -> X^g moves the value at
// exponent e*g into slot i: out[i] = in[pos((2 brev(i) + 1) g mod 2N)] with
// pos(e) = brev((e - 1) / 2) -- the closed form of _eval_exponent_map
// (ring.py:440-468) for this NTT ordering.
__global__ void __launch_bounds__(kEwThreads) k_auto_eval(const __grid_constant__ AutoParams P) {
  const int log_n = P.log_n, N = 1 << log_n;
  const int row = blockIdx.y + blockIdx.z * 65535;
  if (row >= P.rows) return;
  const int i = blockIdx.x * kEwThreads + threadIdx.x;
  if (i >= N) return;
  const uint32_t mask2n = (2u << log_n) - 1u;
  const uint32_t bi = __brev((uint32_t)i) >> (32 - log_n);
  const uint32_t e = (uint32_t)(((uint64_t)(2u * bi + 1u) * P.g) & mask2n);
  const uint32_t src = __brev((e - 1u) >> 1) >> (32 - log_n);
  const int poly = row / P.k, limb = row - poly * P.k;
  P.out[poly * P.os + (size_t)limb * N + i] = P.in[poly * P.is + (size_t)limb * N + src];
}

// Coefficient form: coefficient j moves to (j g mod 2N) with a sign flip when
// the exponent wraps past N (X^N = -1).
__global__ void __launch_bounds__(kEwThreads) k_auto_coeff(const __grid_constant__ AutoParams P) {
  const int log_n = P.log_n, N = 1 << log_n;
  const int row = blockIdx.y + blockIdx.z * 65535;
  if (row >= P.rows) return;
  const int j = blockIdx.x * kEwThreads + threadIdx.x;
  if (j >= N) return;
  const int poly = row / P.k, limb = row - poly * P.k;
  const uint64_t mask2n = (2ull << log_n) - 1ull;
  const uint64_t e = ((uint64_t)j * P.g) & mask2n;
  const uint64_t q = P.pc[P.sel[limb]].q;
  const uint64_t v = P.in[poly * P.is + (size_t)limb * N + j];
  const uint64_t tgt = e & (uint64_t)(N - 1);
  P.out[poly * P.os + (size_t)limb * N + tgt] = (e >= (uint64_t)N) ? (v ? q - v : 0) : v;
}

void launch_automorphism(const PrimeConst* dpc, int log_n, bool eval_form, uint64_t g,
                         const uint64_t* in, int64_t is, uint64_t* out, int64_t os, int n_polys,
                         int k, const int32_t* primes, cudaStream_t st) {
  const int rows = n_polys * k;
  if (rows == 0) return;
  AutoParams P;
  P.in = in;
  P.out = out;
  P.is = is;
  P.os = os;
  P.k = k;
  P.log_n = log_n;
  P.rows = rows;
  P.g = g & ((2ull << log_n) - 1ull);
  if ((P.g & 1ull) == 0) throw HegpuError{HEGPU_E_ARG, "automorphism exponent must be odd"};
  P.pc = dpc;
  fill_sel(P.sel, primes, k);
  const dim3 grid = rows_grid(1 << log_n, rows, 1);
  ProfScope ps(PROF_AUTOMORPHISM, st, (double)rows * (1 << log_n) * 16.0, 0.0);
  if (eval_form)
    k_auto_eval<<<grid, kEwThreads, 0, st>>>(P);
  else
    k_auto_coeff<<<grid, kEwThreads, 0, st>>>(P);
  check_cuda(cudaGetLastError(), "automorphism launch");
}

// ---------------------------------------------------------------------------
// tensor product (ops.py:355-357) and encryption combine (ops.py:102-116)
// ---------------------------------------------------------------------------



// d1 = a0 b1 + a1 b0 is accumulated in 128 bits and reduced once.
__global__ void __launch_bounds__(kEwThreads) k_tensor(const __grid_constant__ TensorParams P) {
  const int N = 1 << P.log_n;
  const int row = blockIdx.y + blockIdx.z * 65535;
  if (row >= P.rows) return;
  const int poly = row / P.k, limb = row - poly * P.k;
  // two adjacent coefficients per thread: 16-byte loads and stores
  const int x = (blockIdx.x * kEwThreads + threadIdx.x) * 2;
  if (x >= N) return;
  const PrimeConst pc = P.pc[limb];
  const size_t l = (size_t)limb * N + x;
  const int64_t ap = (int64_t)(poly % P.amod) * P.as;
  auto ld2 = [](const uint64_t* p) { return *reinterpret_cast<const ulonglong2*>(p); };
  const ulonglong2 a0 = ld2(P.a0 + ap + l), a1 = ld2(P.a1 + ap + l);
  const ulonglong2 b0 = ld2(P.b0 + poly * P.bs + l), b1 = ld2(P.b1 + poly * P.bs + l);
  uint64_t d1[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    Mac128 acc;
    acc.zero();
    acc.add(h ? a0.y : a0.x, h ? b1.y : b1.x);
    acc.add(h ? a1.y : a1.x, h ? b0.y : b0.x);
    d1[h] = mont_mul(acc.redc(pc), pc.r2, pc.q, pc.qinv_neg);
  }
  *reinterpret_cast<ulonglong2*>(P.d0 + poly * P.ds + l) =
      make_ulonglong2(mul_mod(a0.x, b0.x, pc), mul_mod(a0.y, b0.y, pc));
  *reinterpret_cast<ulonglong2*>(P.d1 + poly * P.ds + l) = make_ulonglong2(d1[0], d1[1]);
  *reinterpret_cast<ulonglong2*>(P.d2 + poly * P.ds + l) =
      make_ulonglong2(mul_mod(a1.x, b1.x, pc), mul_mod(a1.y, b1.y, pc));
}

void launch_tensor(const PrimeConst* dpc, int log_n, const TensorParams& T0, int n_polys,
                   cudaStream_t st) {
  const int rows = n_polys * T0.k;
  if (rows == 0) return;
  TensorParams T = T0;
  T.rows = rows;
  T.pc = dpc;
  T.log_n = log_n;
  if (log_n < 1) throw HegpuError{HEGPU_E_ARG, "tensor: N >= 2"};
  const dim3 grid = rows_grid(1 << log_n, rows, 2);
  ProfScope ps(PROF_TENSOR, st, (double)rows * (1 << log_n) * 56.0,
               (double)rows * (1 << log_n) * 8.0);
  k_tensor<<<grid, kEwThreads, 0, st>>>(T);
  check_cuda(cudaGetLastError(), "tensor launch");
}



__global__ void __launch_bounds__(kEwThreads) k_encrypt(const __grid_constant__ EncParams P) {
  const int N = 1 << P.log_n;
  const int limb = blockIdx.y;
  const int x = blockIdx.x * kEwThreads + threadIdx.x;
  if (x >= N) return;
  const PrimeConst pc = P.pc[limb];
  const size_t l = (size_t)limb * N + x;
  const uint64_t v = P.v[l];
  uint64_t c0 = add_mod(mul_mod(v, P.pb[l], pc), P.e0[l], pc.q);
  if (P.m) c0 = add_mod(c0, P.m[l], pc.q);
  P.c0[l] = c0;
  P.c1[l] = add_mod(mul_mod(v, P.pa[l], pc), P.e1[l], pc.q);
}

void launch_encrypt(const PrimeConst* dpc, int log_n, const EncParams& E0, int k,
                    cudaStream_t st) {
  if (k == 0) return;
  EncParams E = E0;
  E.pc = dpc;
  E.log_n = log_n;
  dim3 grid(((1 << log_n) + kEwThreads - 1) / kEwThreads, k);
  ProfScope ps(PROF_ENCRYPT, st, (double)k * (1 << log_n) * 8.0 * (E.m ? 9 : 8),
               (double)k * (1 << log_n) * 4.0);
  k_encrypt<<<grid, kEwThreads, 0, st>>>(E);
  check_cuda(cudaGetLastError(), "encrypt launch");
}

// ---------------------------------------------------------------------------
// plaintext-diagonal multiply-accumulate (bootstrap.py:222-241)
// ---------------------------------------------------------------------------

constexpr int kMaxDiagTerms = 64;
constexpr int kDiagMaxB = 4;
struct DiagParams {
  const uint64_t* ct[kMaxDiagTerms];
  const uint64_t* pt[kMaxDiagTerms];
  int n_terms;
  int n_batch;        // ciphertexts per term (<= kDiagMaxB per launch)
  int64_t ct_c1_off;
  int64_t ct_bstride;  // batch stride of the term ciphertexts
  uint64_t* out;
  int64_t out_c1_off;
  int64_t out_bstride;
  int k, log_n;
  int accumulate;
  const PrimeConst* pc;
};

// out_b.c{0,1} (+)= sum_t pt[t] * ct[t]_b.c{0,1}.  Each thread owns two
// adjacent coefficients (128-bit loads) of one limb; the plaintext diagonal
// is loaded once and applied to every ciphertext of the batch; products are
// accumulated in 128 bits and reduced once per output (one REDC + R^2 fix).
template <int NB>
__global__ void __launch_bounds__(kEwThreads) k_diag_mac(const __grid_constant__ DiagParams P) {
  const int N = 1 << P.log_n;
  const int limb = blockIdx.y;
  const int x = (blockIdx.x * kEwThreads + threadIdx.x) * 2;
  if (x >= N) return;
  const PrimeConst pc = P.pc[limb];
  const size_t l = (size_t)limb * N + x;
  Mac128 a[NB][4];
#pragma unroll
  for (int b = 0; b < NB; ++b)
#pragma unroll
    for (int c = 0; c < 4; ++c) a[b][c].zero();
#pragma unroll 2
  for (int t = 0; t < P.n_terms; ++t) {
    if (t % kMacFold == kMacFold - 1) {
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int c = 0; c < 4; ++c) a[b][c].fold(pc.q, pc.bar);
    }
    const ulonglong2 p = __ldg(reinterpret_cast<const ulonglong2*>(P.pt[t] + l));
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const uint64_t* base = P.ct[t] + b * P.ct_bstride + l;
      const ulonglong2 v0 = __ldg(reinterpret_cast<const ulonglong2*>(base));
      const ulonglong2 v1 = __ldg(reinterpret_cast<const ulonglong2*>(base + P.ct_c1_off));
      a[b][0].add(v0.x, p.x);
      a[b][1].add(v0.y, p.y);
      a[b][2].add(v1.x, p.x);
      a[b][3].add(v1.y, p.y);
    }
  }
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    uint64_t r[4];
#pragma unroll
    for (int c = 0; c < 4; ++c)
      r[c] = mont_mul(a[b][c].redc(pc), pc.r2, pc.q, pc.qinv_neg);
    uint64_t* o0 = P.out + b * P.out_bstride + l;
    uint64_t* o1 = o0 + P.out_c1_off;
    if (P.accumulate) {
      const ulonglong2 p0 = *reinterpret_cast<const ulonglong2*>(o0);
      const ulonglong2 p1 = *reinterpret_cast<const ulonglong2*>(o1);
      r[0] = add_mod(r[0], p0.x, pc.q);
      r[1] = add_mod(r[1], p0.y, pc.q);
      r[2] = add_mod(r[2], p1.x, pc.q);
      r[3] = add_mod(r[3], p1.y, pc.q);
    }
    *reinterpret_cast<ulonglong2*>(o0) = make_ulonglong2(r[0], r[1]);
    *reinterpret_cast<ulonglong2*>(o1) = make_ulonglong2(r[2], r[3]);
  }
}

void launch_diag_mac(const PrimeConst* dpc, int log_n, const uint64_t* const* ct,
                     int64_t ct_c1_off, int64_t ct_bstride, const uint64_t* const* pt,
                     int n_terms, int n_batch, uint64_t* out, int64_t out_c1_off,
                     int64_t out_bstride, int k, int accumulate, cudaStream_t st) {
  if (n_terms == 0 && !accumulate) throw HegpuError{HEGPU_E_ARG, "diag_mac with no terms"};
  if (n_batch < 1) throw HegpuError{HEGPU_E_ARG, "diag_mac needs n_batch >= 1"};
  for (int b0 = 0; b0 < n_batch; b0 += kDiagMaxB) {
    const int nb = n_batch - b0 < kDiagMaxB ? n_batch - b0 : kDiagMaxB;
    int done = 0;
    bool acc = accumulate != 0;
    while (done < n_terms) {
      DiagParams P;
      P.n_terms = n_terms - done < kMaxDiagTerms ? n_terms - done : kMaxDiagTerms;
      for (int t = 0; t < P.n_terms; ++t) {
        P.ct[t] = ct[done + t] + b0 * ct_bstride;
        P.pt[t] = pt[done + t];
      }
      P.n_batch = nb;
      P.ct_c1_off = ct_c1_off;
      P.ct_bstride = ct_bstride;
      P.out = out + b0 * out_bstride;
      P.out_c1_off = out_c1_off;
      P.out_bstride = out_bstride;
      P.k = k;
      P.log_n = log_n;
      P.accumulate = acc ? 1 : 0;
      P.pc = dpc;
      dim3 grid(((1 << log_n) / 2 + kEwThreads - 1) / kEwThreads, k);
      ProfScope ps(PROF_DIAG_MAC, st,
                   (double)k * (1 << log_n) * 8.0 * (P.n_terms * (1.0 + 2.0 * nb) + (acc ? 4 : 2) * nb),
                   (double)k * (1 << log_n) * nb * (2.0 * P.n_terms + 4));
      switch (nb) {
        case 1: k_diag_mac<1><<<grid, kEwThreads, 0, st>>>(P); break;
        case 2: k_diag_mac<2><<<grid, kEwThreads, 0, st>>>(P); break;
        case 3: k_diag_mac<3><<<grid, kEwThreads, 0, st>>>(P); break;
        default: k_diag_mac<4><<<grid, kEwThreads, 0, st>>>(P); break;
      }
      check_cuda(cudaGetLastError(), "diag_mac launch");
      done += P.n_terms;
      acc = true;
    }
  }
}

// ---------------------------------------------------------------------------
// fast basis conversion (BaseConverter.convert, keys.py:43-49;
// base_convert, _kernels.py:300-317), one or several jobs per launch.
// hat_i = x_i * (Q/q_i)^-1 mod q_i; out_t = REDC(sum_i hat_i * punc_mont[i][t]).
// ---------------------------------------------------------------------------

constexpr int kMaxConvSrc = 32;

// 128-bit accumulation without reduction; fold() keeps T < q 2^64 (call it
// at least every second product of two < 2^62 x < q factors).
struct Acc2 {
  uint64_t hi, lo;
  __device__ __forceinline__ void zero() { hi = lo = 0; }
  __device__ __forceinline__ void add(uint64_t a, uint64_t b) {
    const uint64_t plo = a * b;
    const uint64_t phi = __umul64hi(a, b);
    const uint64_t nlo = lo + plo;
    hi = hi + phi + (nlo < lo);
    lo = nlo;
  }
  __device__ __forceinline__ void fold(uint64_t q) { hi = hi >= q ? hi - q : hi; }
};

// Two adjacent coefficients per thread; the job's conversion matrix and the
// destination moduli are staged in shared memory; NS = compile-time bound on
// the job's source-limb count (loops fully unrolled, predicated on n_src).
template <int NS>
__global__ void __launch_bounds__(kEwThreads) k_conv(const __grid_constant__ ConvParams P) {
  __shared__ uint64_t s_punc[NS * kMaxPrimes];
  __shared__ uint64_t s_q[kMaxPrimes], s_qi[kMaxPrimes], s_bar[kMaxPrimes];
  const int N = 1 << P.log_n;
  const int j = blockIdx.y;
  const int poly = blockIdx.z;
  const ConvJob& J = P.job[j];
  const int ns = J.n_src, nd = J.n_dst;
  for (int e = threadIdx.x; e < ns * nd; e += blockDim.x) {
    const int i = e / nd, t = e - i * nd;
    s_punc[i * kMaxPrimes + t] = J.punc[(size_t)i * J.punc_ld + t];
  }
  for (int t = threadIdx.x; t < nd; t += blockDim.x) {
    const PrimeConst pc = P.pc[P.dst_sel[j][t]];
    s_q[t] = pc.q;
    s_qi[t] = pc.qinv_neg;
    s_bar[t] = pc.bar;
  }
  __syncthreads();
  const int x = (blockIdx.x * kEwThreads + threadIdx.x) * 2;
  if (x >= N) return;
  uint64_t h0[NS], h1[NS];
  const uint64_t* src = J.src + poly * J.src_stride + x;
#pragma unroll
  for (int i = 0; i < NS; ++i) {
    if (i < ns) {
      const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(src + (size_t)i * N);
      if (J.inv) {
        const uint64_t q = P.pc[P.src_sel[j][i]].q;
        const uint64_t w = J.inv[i], wsh = J.inv_sh[i];
        h0[i] = shoup(v.x, w, wsh, q);
        h1[i] = shoup(v.y, w, wsh, q);
      } else {
        h0[i] = v.x;
        h1[i] = v.y;
      }
    } else {
      h0[i] = h1[i] = 0;
    }
  }
  uint64_t* dst = J.dst + poly * J.dst_stride + x;
  for (int t = 0; t < nd; ++t) {
    PrimeConst pt;
    pt.q = s_q[t];
    pt.qinv_neg = s_qi[t];
    pt.bar = s_bar[t];
    Mac128 a0, a1;
    a0.zero();
    a1.zero();
#pragma unroll
    for (int i = 0; i < NS; ++i) {
      if (i < ns) {
        const uint64_t c = s_punc[i * kMaxPrimes + t];
        a0.add(h0[i], c);
        a1.add(h1[i], c);
        if (i % kMacFold == kMacFold - 1) {
          a0.fold(pt.q, pt.bar);
          a1.fold(pt.q, pt.bar);
        }
      }
    }
    *reinterpret_cast<ulonglong2*>(dst + (size_t)t * N) = make_ulonglong2(a0.redc(pt), a1.redc(pt));
  }
}

void launch_conv(ConvParams& P, cudaStream_t st) {
  if (P.n_jobs == 0 || P.n_polys == 0) return;
  for (int j = 0; j < P.n_jobs; ++j)
    if (P.job[j].n_src > kMaxConvSrc) throw HegpuError{HEGPU_E_ARG, "too many source limbs"};
  dim3 grid(((1 << P.log_n) + kEwThreads - 1) / kEwThreads, P.n_jobs, P.n_polys);
  double cb = 0, cm = 0;
  for (int j = 0; j < P.n_jobs; ++j) {
    cb += (double)P.n_polys * (1 << P.log_n) * 8.0 * (P.job[j].n_src + P.job[j].n_dst);
    cm += (double)P.n_polys * (1 << P.log_n) *
          ((double)P.job[j].n_src * P.job[j].n_dst + P.job[j].n_src);
  }
  int ns = 1;
  for (int j = 0; j < P.n_jobs; ++j) ns = P.job[j].n_src > ns ? P.job[j].n_src : ns;
  grid.x = ((1 << P.log_n) / 2 + kEwThreads - 1) / kEwThreads;
  ProfScope ps(PROF_CONV, st, cb, cm);
  if (ns <= 2) k_conv<2><<<grid, kEwThreads, 0, st>>>(P);
  else if (ns <= 4) k_conv<4><<<grid, kEwThreads, 0, st>>>(P);
  else if (ns <= 6) k_conv<6><<<grid, kEwThreads, 0, st>>>(P);
  else if (ns <= 8) k_conv<8><<<grid, kEwThreads, 0, st>>>(P);
  else if (ns <= 12) k_conv<12><<<grid, kEwThreads, 0, st>>>(P);
  else k_conv<kMaxConvSrc><<<grid, kEwThreads, 0, st>>>(P);
  check_cuda(cudaGetLastError(), "conv launch");
}

// ---------------------------------------------------------------------------
// key-switch inner product (keys.py:299-323 / fma_gather_inplace,
// _kernels.py:271-286), batched: the (digit x row) key values of a coefficient
// are loaded once and applied to every ciphertext of the batch.
// ---------------------------------------------------------------------------



// Two adjacent coefficients per thread (128-bit loads); BETA = compile-time
// bound on the digit count, predicated on P.beta.
template <int BETA>
__global__ void __launch_bounds__(kEwThreads) k_ks_ip(const __grid_constant__ IpParams P) {
  const int N = 1 << P.log_n;
  const int r = blockIdx.y;
  const int x = (blockIdx.x * kEwThreads + threadIdx.x) * 2;
  if (x >= N) return;
  const int prime = r <= P.level ? r : P.n_chain + (r - P.level - 1);
  const int krow = r <= P.level ? r : P.key_sp_row0 + (r - P.level - 1);
  const PrimeConst pc = P.pc[prime];
  ulonglong2 kb[BETA], ka[BETA];
#pragma unroll
  for (int j = 0; j < BETA; ++j) {
    if (j < P.beta) {
      kb[j] = __ldg(reinterpret_cast<const ulonglong2*>(P.kb[j] + (size_t)krow * N + x));
      ka[j] = __ldg(reinterpret_cast<const ulonglong2*>(P.ka[j] + (size_t)krow * N + x));
    }
  }
  for (int b = 0; b < P.n_batch; ++b) {
    Mac128 b0, b1, a0, a1;
    b0.zero();
    b1.zero();
    a0.zero();
    a1.zero();
#pragma unroll
    for (int j = 0; j < BETA; ++j) {
      if (j < P.beta) {
        const int g0 = j * P.alpha;
        const int g1 = min(g0 + P.alpha, P.level + 1);
        const uint64_t* src;
        if (r >= g0 && r < g1)
          src = P.d + b * P.ds + (size_t)r * N + x;
        else
          src = P.ext + b * P.ext_sb + j * P.ext_sj + (size_t)(r < g0 ? r : r - (g1 - g0)) * N + x;
        const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(src));
        b0.add(v.x, kb[j].x);
        b1.add(v.y, kb[j].y);
        a0.add(v.x, ka[j].x);
        a1.add(v.y, ka[j].y);
        if (j % kMacFold == kMacFold - 1) {
          b0.fold(pc.q, pc.bar);
          b1.fold(pc.q, pc.bar);
          a0.fold(pc.q, pc.bar);
          a1.fold(pc.q, pc.bar);
        }
      }
    }
    uint64_t* o = P.acc + b * P.acc_sb + (size_t)r * N + x;
    const uint64_t q = pc.q, qn = pc.qinv_neg, r2 = pc.r2;
    ulonglong2 vb = make_ulonglong2(mont_mul(b0.redc(pc), r2, q, qn), mont_mul(b1.redc(pc), r2, q, qn));
    ulonglong2 va = make_ulonglong2(mont_mul(a0.redc(pc), r2, q, qn), mont_mul(a1.redc(pc), r2, q, qn));
    if (P.accumulate) {
      const ulonglong2 pb = *reinterpret_cast<const ulonglong2*>(o);
      const ulonglong2 pa = *reinterpret_cast<const ulonglong2*>(o + (size_t)P.n_ext * N);
      vb = make_ulonglong2(add_mod(vb.x, pb.x, q), add_mod(vb.y, pb.y, q));
      va = make_ulonglong2(add_mod(va.x, pa.x, q), add_mod(va.y, pa.y, q));
    }
    *reinterpret_cast<ulonglong2*>(o) = vb;
    *reinterpret_cast<ulonglong2*>(o + (size_t)P.n_ext * N) = va;
  }
}

// Source index of output slot i under X -> X^g (eval form, see k_auto_eval).
// The map keeps aligned blocks of 2^b slots together for every b, so a warp's
// 32 consecutive outputs gather from one aligned 32-slot source block.
__device__ __forceinline__ uint32_t auto_src(uint32_t i, uint32_t g, int log_n) {
  const uint32_t mask2n = (2u << log_n) - 1u;
  const uint32_t bi = __brev(i) >> (32 - log_n);
  const uint32_t e = (uint32_t)(((uint64_t)(2u * bi + 1u) * g) & mask2n);
  return __brev((e - 1u) >> 1) >> (32 - log_n);
}

// One coefficient per thread, BG batch elements per CTA (grid.z groups),
// BETA = compile-time bound on the digit count.  Per rotation all digits'
// key words and gathered digit words are loaded first (2*BETA + BG*BETA
// independent loads in flight), then multiplied: the kernel is bound by
// load latency, not arithmetic.
template <int BG, int BETA>
__global__ void __launch_bounds__(kEwThreads) k_ks_ip_rot(const __grid_constant__ IpRotParams P) {
  const int N = 1 << P.log_n;
  // grid (batch groups, coefficient blocks, rows): the groups sharing a key
  // slice are scheduled back to back, so the key words hit L2 after the first
  const int r = blockIdx.z;
  const int x = blockIdx.y * kEwThreads + threadIdx.x;
  if (x >= N) return;
  const int b0 = blockIdx.x * BG;
  const int nb = P.n_batch - b0 < BG ? P.n_batch - b0 : BG;
  const int prime = r <= P.level ? r : P.n_chain + (r - P.level - 1);
  const int krow = r <= P.level ? r : P.key_sp_row0 + (r - P.level - 1);
  const PrimeConst pc = P.pc[prime];
  // digit j's source row (own rows come from d, the others from ext)
  const uint64_t* base[BETA];
  int64_t bstr[BETA], rstr[BETA];
#pragma unroll
  for (int j = 0; j < BETA; ++j) {
    const int g0 = j * P.alpha;
    const int g1 = min(g0 + P.alpha, P.level + 1);
    if (r >= g0 && r < g1) {
      base[j] = P.d + (size_t)r * N + (size_t)b0 * P.ds;
      bstr[j] = P.ds;
      rstr[j] = P.d_sr;
    } else {
      base[j] = P.ext + j * P.ext_sj + (size_t)(r < g0 ? r : r - (g1 - g0)) * N +
                (size_t)b0 * P.ext_sb;
      bstr[j] = P.ext_sb;
      rstr[j] = P.ext_sr;
    }
  }
  const size_t koff = (size_t)krow * N + x;
  Mac128 ab[BG], aa[BG];
#pragma unroll
  for (int b = 0; b < BG; ++b) {
    ab[b].zero();
    aa[b].zero();
  }
  int since = 0;
  for (int rot = 0; rot < P.n_rot; ++rot) {
    const uint32_t src = auto_src((uint32_t)x, P.gal[rot], P.log_n);
    uint64_t kb[BETA], ka[BETA], v[BETA][BG];
#pragma unroll
    for (int j = 0; j < BETA; ++j) {
      if (j < P.beta) {
        kb[j] = __ldg(P.kb[rot][j] + koff);
        ka[j] = __ldg(P.ka[rot][j] + koff);
        const uint64_t* bp = base[j] + rot * rstr[j] + src;
#pragma unroll
        for (int b = 0; b < BG; ++b) v[j][b] = b < nb ? __ldg(bp + (size_t)b * bstr[j]) : 0;
      }
    }
#pragma unroll
    for (int j = 0; j < BETA; ++j) {
      if (j < P.beta) {
#pragma unroll
        for (int b = 0; b < BG; ++b) {
          ab[b].add(v[j][b], kb[j]);
          aa[b].add(v[j][b], ka[j]);
        }
        if (++since == kMacFold) {
          since = 0;
#pragma unroll
          for (int b = 0; b < BG; ++b) {
            ab[b].fold(pc.q, pc.bar);
            aa[b].fold(pc.q, pc.bar);
          }
        }
      }
    }
    if (!P.sum_mode || rot == P.n_rot - 1) {
      uint64_t* o = P.acc + (P.sum_mode ? 0 : rot * P.acc_sr) + (size_t)r * N + x;
#pragma unroll
      for (int b = 0; b < BG; ++b) {
        if (b < nb) {
          uint64_t* ob = o + (size_t)(b0 + b) * P.acc_sb;
          uint64_t vb = mont_mul(ab[b].redc(pc), pc.r2, pc.q, pc.qinv_neg);
          uint64_t va = mont_mul(aa[b].redc(pc), pc.r2, pc.q, pc.qinv_neg);
          if (P.c0 && r <= P.level)
            vb = add_mod(vb, shoup(__ldg(P.c0 + (size_t)(b0 + b) * P.c0s + (size_t)r * N + src),
                                   P.pm[r], P.pm_sh[r], pc.q),
                         pc.q);
          if (P.accumulate) {
            vb = add_mod(vb, ob[0], pc.q);
            va = add_mod(va, ob[(size_t)P.n_ext * N], pc.q);
          }
          ob[0] = vb;
          ob[(size_t)P.n_ext * N] = va;
        }
        ab[b].zero();
        aa[b].zero();
      }
      since = 0;
    }
  }
}

// n_batch == 1 (the bootstrap's hoisted babies): two adjacent coefficients
// per thread -- the key words load as one 16-byte pair, the digit words are
// gathered per coefficient -- so each thread keeps 4 independent accumulators
// and half as many key-load instructions are issued per byte.
#ifndef HEGPU_IPROT_1X2
#define HEGPU_IPROT_1X2 1
#endif
constexpr bool kIpRot1x2 = HEGPU_IPROT_1X2;
template <int BETA>
__global__ void __launch_bounds__(kEwThreads) k_ks_ip_rot1x2(const __grid_constant__ IpRotParams P) {
  const int N = 1 << P.log_n;
  const int r = blockIdx.z;
  const int x = (blockIdx.y * kEwThreads + threadIdx.x) * 2;
  if (x >= N) return;
  const int prime = r <= P.level ? r : P.n_chain + (r - P.level - 1);
  const int krow = r <= P.level ? r : P.key_sp_row0 + (r - P.level - 1);
  const PrimeConst pc = P.pc[prime];
  const uint64_t* base[BETA];
  int64_t rstr[BETA];
#pragma unroll
  for (int j = 0; j < BETA; ++j) {
    const int g0 = j * P.alpha;
    const int g1 = min(g0 + P.alpha, P.level + 1);
    if (r >= g0 && r < g1) {
      base[j] = P.d + (size_t)r * N;
      rstr[j] = P.d_sr;
    } else {
      base[j] = P.ext + j * P.ext_sj + (size_t)(r < g0 ? r : r - (g1 - g0)) * N;
      rstr[j] = P.ext_sr;
    }
  }
  const size_t koff = (size_t)krow * N + x;
  Mac128 ab[2], aa[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    ab[h].zero();
    aa[h].zero();
  }
  int since = 0;
  for (int rot = 0; rot < P.n_rot; ++rot) {
    const uint32_t s0 = auto_src((uint32_t)x, P.gal[rot], P.log_n);
    const uint32_t s1 = auto_src((uint32_t)x + 1, P.gal[rot], P.log_n);
    ulonglong2 kb[BETA], ka[BETA];
    uint64_t v0[BETA], v1[BETA];
#pragma unroll
    for (int j = 0; j < BETA; ++j) {
      if (j < P.beta) {
        kb[j] = __ldg(reinterpret_cast<const ulonglong2*>(P.kb[rot][j] + koff));
        ka[j] = __ldg(reinterpret_cast<const ulonglong2*>(P.ka[rot][j] + koff));
        const uint64_t* bp = base[j] + rot * rstr[j];
        v0[j] = __ldg(bp + s0);
        v1[j] = __ldg(bp + s1);
      }
    }
#pragma unroll
    for (int j = 0; j < BETA; ++j) {
      if (j < P.beta) {
        ab[0].add(v0[j], kb[j].x);
        ab[1].add(v1[j], kb[j].y);
        aa[0].add(v0[j], ka[j].x);
        aa[1].add(v1[j], ka[j].y);
        if (++since == kMacFold) {
          since = 0;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            ab[h].fold(pc.q, pc.bar);
            aa[h].fold(pc.q, pc.bar);
          }
        }
      }
    }
    if (!P.sum_mode || rot == P.n_rot - 1) {
      uint64_t* o = P.acc + (P.sum_mode ? 0 : rot * P.acc_sr) + (size_t)r * N + x;
      uint64_t vb[2], va[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        vb[h] = mont_mul(ab[h].redc(pc), pc.r2, pc.q, pc.qinv_neg);
        va[h] = mont_mul(aa[h].redc(pc), pc.r2, pc.q, pc.qinv_neg);
      }
      if (P.c0 && r <= P.level) {
        const uint64_t* c0 = P.c0 + (size_t)r * N;
        vb[0] = add_mod(vb[0], shoup(__ldg(c0 + s0), P.pm[r], P.pm_sh[r], pc.q), pc.q);
        vb[1] = add_mod(vb[1], shoup(__ldg(c0 + s1), P.pm[r], P.pm_sh[r], pc.q), pc.q);
      }
      if (P.accumulate) {
        const ulonglong2 pb = *reinterpret_cast<const ulonglong2*>(o);
        const ulonglong2 pa = *reinterpret_cast<const ulonglong2*>(o + (size_t)P.n_ext * N);
        vb[0] = add_mod(vb[0], pb.x, pc.q);
        vb[1] = add_mod(vb[1], pb.y, pc.q);
        va[0] = add_mod(va[0], pa.x, pc.q);
        va[1] = add_mod(va[1], pa.y, pc.q);
      }
      *reinterpret_cast<ulonglong2*>(o) = make_ulonglong2(vb[0], vb[1]);
      *reinterpret_cast<ulonglong2*>(o + (size_t)P.n_ext * N) = make_ulonglong2(va[0], va[1]);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        ab[h].zero();
        aa[h].zero();
      }
      since = 0;
    }
  }
}

template <int BG>
static void launch_ip_rot_bg(IpRotParams& P, dim3 grid, cudaStream_t st) {
  if (P.beta <= 2)
    k_ks_ip_rot<BG, 2><<<grid, kEwThreads, 0, st>>>(P);
  else if (P.beta <= 4)
    k_ks_ip_rot<BG, 4><<<grid, kEwThreads, 0, st>>>(P);
  else
    k_ks_ip_rot<BG, kMaxRotDigits><<<grid, kEwThreads, 0, st>>>(P);
}

void launch_ks_ip_rot(IpRotParams& P, cudaStream_t st) {
  if (P.beta > kMaxRotDigits) throw HegpuError{HEGPU_E_ARG, "too many key-switch digits"};
  if (P.n_rot < 1 || P.n_rot > kMaxRot) throw HegpuError{HEGPU_E_ARG, "1..16 rotations"};
  const int bg = P.n_batch >= 4 ? 4 : P.n_batch >= 2 ? 2 : 1;
  dim3 grid((P.n_batch + bg - 1) / bg, ((1 << P.log_n) + kEwThreads - 1) / kEwThreads, P.n_ext);
  const double ipn = (double)(1 << P.log_n) * P.n_ext;
  ProfScope ps(PROF_KS_IP, st,
               ipn * 8.0 * P.n_rot * (2.0 * P.beta + P.n_batch * P.beta) +
                   ipn * 8.0 * 2.0 * P.n_batch * (P.sum_mode ? 1 : P.n_rot),
               ipn * P.n_batch * P.n_rot * 2.0 * P.beta);
  if (launch_ks_ip_rot_tma(P, st)) return;
  if (P.n_batch == 1 && (1 << P.log_n) >= 2 * kEwThreads && kIpRot1x2) {
    dim3 g2(1, ((1 << P.log_n) / 2 + kEwThreads - 1) / kEwThreads, P.n_ext);
    if (P.beta <= 2)
      k_ks_ip_rot1x2<2><<<g2, kEwThreads, 0, st>>>(P);
    else if (P.beta <= 4)
      k_ks_ip_rot1x2<4><<<g2, kEwThreads, 0, st>>>(P);
    else
      k_ks_ip_rot1x2<kMaxRotDigits><<<g2, kEwThreads, 0, st>>>(P);
    check_cuda(cudaGetLastError(), "ks rotation inner product launch");
    return;
  }
  if (bg == 4)
    launch_ip_rot_bg<4>(P, grid, st);
  else if (bg == 2)
    launch_ip_rot_bg<2>(P, grid, st);
  else
    launch_ip_rot_bg<1>(P, grid, st);
  check_cuda(cudaGetLastError(), "ks rotation inner product launch");
}

struct AutoSumParams {
  int kq, n_chain;  // limbs >= kq: special primes
  const uint64_t* in;
  int64_t is, in_sr;  // rotation r permutes in + r*in_sr
  const uint64_t* base;  // out = base + sum_r sigma_r(in); base == in when null
  int64_t bs;
  uint64_t* out;
  int64_t os;
  uint32_t gal[kMaxRot];
  int n_rot, k, log_n;
  int rows;  // n_polys * k: the last grid.z slice may overhang
  const PrimeConst* pc;
};

__global__ void __launch_bounds__(kEwThreads) k_auto_sum(const __grid_constant__ AutoSumParams P) {
  const int N = 1 << P.log_n;
  const int row = blockIdx.y + blockIdx.z * 65535;
  if (row >= P.rows) return;
  const int x = blockIdx.x * kEwThreads + threadIdx.x;
  if (x >= N) return;
  const int poly = row / P.k, limb = row - poly * P.k;
  const uint64_t q = P.pc[limb < P.kq ? limb : P.n_chain + (limb - P.kq)].q;
  const uint64_t* in = P.in + poly * P.is + (size_t)limb * N;
  uint64_t s = P.base ? P.base[poly * P.bs + (size_t)limb * N + x] : in[x];
  for (int r = 0; r < P.n_rot; ++r)
    s = add_mod(s, __ldg(in + r * P.in_sr + auto_src((uint32_t)x, P.gal[r], P.log_n)), q);
  P.out[poly * P.os + (size_t)limb * N + x] = s;
}

void launch_auto_sum(const PrimeConst* dpc, int log_n, const uint32_t* gal, int n_rot,
                     const uint64_t* in, int64_t is, const uint64_t* base, int64_t bs,
                     uint64_t* out, int64_t os, int n_polys, int k, cudaStream_t st,
                     int64_t in_sr, int kq, int n_chain) {
  if (n_rot > kMaxRot) throw HegpuError{HEGPU_E_ARG, "1..16 rotations"};
  AutoSumParams P;
  P.kq = kq < 0 ? k : kq;
  P.n_chain = n_chain;
  P.in = in;
  P.is = is;
  P.in_sr = in_sr;
  P.base = base;
  P.bs = bs;
  P.out = out;
  P.os = os;
  for (int r = 0; r < n_rot; ++r) P.gal[r] = gal[r];
  P.n_rot = n_rot;
  P.k = k;
  P.log_n = log_n;
  P.pc = dpc;
  const int rows = n_polys * k;
  if (rows == 0) return;
  P.rows = rows;
  const dim3 grid = rows_grid(1 << log_n, rows, 1);
  ProfScope ps(PROF_AUTOMORPHISM, st, (double)rows * (1 << log_n) * 8.0 * (n_rot + 2), 0.0);
  k_auto_sum<<<grid, kEwThreads, 0, st>>>(P);
  check_cuda(cudaGetLastError(), "automorphism sum launch");
}

void launch_ks_ip(IpParams& P, cudaStream_t st) {
  if (P.beta > kMaxDigits) throw HegpuError{HEGPU_E_ARG, "too many key-switch digits"};
  dim3 grid(((1 << P.log_n) / 2 + kEwThreads - 1) / kEwThreads, P.n_ext);
  const double ipn = (double)(1 << P.log_n) * P.n_ext;
  ProfScope ps(PROF_KS_IP, st, ipn * 8.0 * (2.0 * P.beta + P.n_batch * (P.beta + 2.0)),
               ipn * P.n_batch * (2.0 * P.beta + 4));
  {  // TMA-staged key streaming: the same inner product as one "rotation" by g = 1
    IpRotParams R{};
    R.d = P.d;
    R.ds = P.ds;
    R.ext = P.ext;
    R.ext_sb = P.ext_sb;
    R.ext_sj = P.ext_sj;
    for (int j = 0; j < P.beta && j < kMaxRotDigits; ++j) {
      R.kb[0][j] = P.kb[j];
      R.ka[0][j] = P.ka[j];
    }
    R.gal[0] = 1;
    R.n_rot = 1;
    R.accumulate = P.accumulate;
    R.acc = P.acc;
    R.acc_sb = P.acc_sb;
    R.level = P.level;
    R.alpha = P.alpha;
    R.beta = P.beta;
    R.n_ext = P.n_ext;
    R.n_chain = P.n_chain;
    R.key_sp_row0 = P.key_sp_row0;
    R.n_batch = P.n_batch;
    R.log_n = P.log_n;
    R.pc = P.pc;
    if (P.beta <= kMaxRotDigits && launch_ks_ip_rot_tma(R, st)) return;
  }
  if (P.beta <= 2) k_ks_ip<2><<<grid, kEwThreads, 0, st>>>(P);
  else if (P.beta <= 4) k_ks_ip<4><<<grid, kEwThreads, 0, st>>>(P);
  else if (P.beta <= 8) k_ks_ip<8><<<grid, kEwThreads, 0, st>>>(P);
  else k_ks_ip<kMaxDigits><<<grid, kEwThreads, 0, st>>>(P);
  check_cuda(cudaGetLastError(), "ks inner product launch");
}

}  // namespace hegpu

namespace hegpu {

// ---------------------------------------------------------------------------
// INT64 modular-multiplication peak microbenchmark (the roofline denominator
// for the NTT / key-switch INT bound; MEASURED_PEAKS.json has no INT peak).
// Each thread runs 8 independent chains of Shoup (w, w') multiplications --
// the NTT butterfly's product -- so the FMA/ALU pipes, not latency, bound it.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_modmul_peak(uint64_t* sink, uint64_t q, uint64_t w,
                                                     uint64_t wsh, int iters) {
  uint64_t x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = (threadIdx.x * 8 + c + blockIdx.x) % q;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = shoup_lazy(x[c], w, wsh, q);
  }
  uint64_t acc = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) acc ^= x[c];
  if (acc == 0x123456789ull) sink[0] = acc;  // keep the chains alive
}

// FP64-pipe modmul (common.cuh fp_mulmod) on a 40-bit chain prime
__global__ void __launch_bounds__(256) k_fp_modmul_peak(double* sink, double q, double w,
                                                        double wq, int iters) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = (double)((threadIdx.x * 8 + c + blockIdx.x) % 100000);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fp_mulmod(x[c], w, wq, q);
  }
  double acc = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) acc += x[c];
  if (acc == 0.5) sink[0] = acc;  // keep the chains alive
}

double bench_fp_modmul_peak(int iters) {
  const uint64_t qi = 0xffffe80001ull;  // 40-bit prime of the P16 chain
  const double q = (double)qi, w = (double)(0x123456789ull % qi), wq = w / q;
  int dev = 0, sms = 0;
  check_cuda(cudaGetDevice(&dev), "device");
  check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sm count");
  double* sink = nullptr;
  check_cuda(cudaMalloc(&sink, 8), "alloc");
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_fp_modmul_peak<<<blocks, threads>>>(sink, q, w, wq, 64);
  cudaEventRecord(a);
  k_fp_modmul_peak<<<blocks, threads>>>(sink, q, w, wq, iters);
  cudaEventRecord(b);
  check_cuda(cudaEventSynchronize(b), "fp modmul bench");
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  return (double)blocks * threads * 8.0 * iters / (ms * 1e-3);
}

double bench_modmul_peak(int iters) {
  const uint64_t q = 0xffffffffffc0001ull;  // 60-bit prime of the P16 chain
  const uint64_t w = 0x123456789abcdull % q;
  const uint64_t wsh = h_shoup(w, q);
  int dev = 0, sms = 0;
  check_cuda(cudaGetDevice(&dev), "device");
  check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sm count");
  uint64_t* sink = nullptr;
  check_cuda(cudaMalloc(&sink, 8), "alloc");
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k_modmul_peak<<<blocks, threads>>>(sink, q, w, wsh, 64);  // warm-up
  cudaEventRecord(a);
  k_modmul_peak<<<blocks, threads>>>(sink, q, w, wsh, iters);
  cudaEventRecord(b);
  check_cuda(cudaEventSynchronize(b), "modmul bench");
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  return (double)blocks * threads * 8.0 * iters / (ms * 1e-3);
}

}  // namespace hegpu

namespace hegpu {

// ---------------------------------------------------------------------------
// All-giants BSGS multiply-accumulate (the linear transforms of bootstrapping,
// bootstrap.py:200-247): for every giant g and batch element b
//   out[g]_b.c{0,1} = sum_t pt[idx[g][t]] * baby[t]_b.c{0,1}.
// A CTA owns 32 coefficients of one limb: it stages those coefficients of
// every baby ciphertext in shared memory once, then each thread accumulates
// GPT giants for one coefficient.  HBM traffic is the minimum: every plaintext
// diagonal, every baby and every output is touched exactly once (the per-giant
// formulation re-reads all babies once per giant).
// ---------------------------------------------------------------------------
constexpr int kBsgsMaxTerms = 256;

struct BsgsParams {
  const uint64_t* baby[kBsgsMaxTerms];
  int n_terms, n_giants, n_batch, log_n;
  int64_t c1_off, bstride;          // baby / output component and batch strides
  const uint64_t* pt_base;
  int64_t pt_stride;                // elements between diagonals
  int pt_log_run;                   // diagonals stored run-compressed (see launch_bsgs)
  const int32_t* pt_idx;            // device [n_giants][n_terms], -1 = zero diagonal
  uint64_t* out;
  int64_t out_gstride;              // elements between giants' outputs
  const PrimeConst* pc;
  int kq, n_chain;                  // limbs >= kq are special primes n_chain + (limb - kq)
};

// CTA = 32 warps over a 64-coefficient tile of one limb; warp w accumulates
// giant w for 2 coefficients per lane (128-bit loads).  The babies' tile is
// staged in shared memory in chunks of kBsgsChunk terms; the term loop is
// unrolled by 4 so every lane keeps 4 independent 16-byte diagonal loads in
// flight (64 KiB per SM) while it multiplies the previous ones.
constexpr int kBsgsTile = 64;
constexpr int kBsgsChunk = 16;

// WARPS giants per CTA (one per warp); grid.z enumerates giant groups.
template <int NB, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) k_bsgs(const __grid_constant__ BsgsParams P) {
  __shared__ __align__(16) uint64_t sm[kBsgsChunk * NB * 2 * kBsgsTile];
  __shared__ int32_t s_idx[WARPS * kBsgsMaxTerms];
  const int N = 1 << P.log_n;
  const int limb = blockIdx.y;
  const int x0 = blockIdx.x * kBsgsTile;
  const PrimeConst pc = P.pc[limb < P.kq ? limb : P.n_chain + (limb - P.kq)];
  constexpr int per_term = NB * 2 * kBsgsTile;
  const int nthr = WARPS * 32;
  const int g0 = blockIdx.z * WARPS;  // first giant of this CTA
  const int ng = P.n_giants - g0 < WARPS ? P.n_giants - g0 : WARPS;
  for (int e = threadIdx.x; e < ng * P.n_terms; e += nthr)
    s_idx[e] = __ldg(P.pt_idx + (size_t)g0 * P.n_terms + e);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int xi = lane * 2;
  const size_t coef = (size_t)limb * N + x0 + xi;
  // run-compressed diagonal: one stored word per 2^lr consecutive coefficients
  const int lr = P.pt_log_run;
  const size_t pcoef = ((size_t)limb * N + x0 + xi) >> lr;
  const int g = warp;  // local giant
  Mac128 acc[NB][2][2];
#pragma unroll
  for (int b = 0; b < NB; ++b)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      acc[b][c][0].zero();
      acc[b][c][1].zero();
    }
  for (int tc = 0; tc < P.n_terms; tc += kBsgsChunk) {
    const int nt = P.n_terms - tc < kBsgsChunk ? P.n_terms - tc : kBsgsChunk;
    __syncthreads();  // previous chunk fully consumed (and s_idx visible)
    for (int e = threadIdx.x; e < nt * per_term / 2; e += nthr) {
      const int e2 = e * 2;
      const int t = e2 / per_term;
      const int rem = e2 - t * per_term;
      const int b = rem / (2 * kBsgsTile);
      const int c = (rem / kBsgsTile) & 1;
      const int xx = rem % kBsgsTile;
      *reinterpret_cast<ulonglong2*>(sm + e2) = __ldg(reinterpret_cast<const ulonglong2*>(
          P.baby[tc + t] + b * P.bstride + c * P.c1_off + (size_t)limb * N + x0 + xx));
    }
    __syncthreads();
    if (g < ng) {
      for (int t0 = 0; t0 < nt; t0 += 4) {
        ulonglong2 pv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int t = t0 + u;
          const int idx = t < nt ? s_idx[g * P.n_terms + tc + t] : -1;
          if (idx < 0) {
            pv[u] = make_ulonglong2(0, 0);
          } else if (lr == 0) {
            pv[u] = __ldg(reinterpret_cast<const ulonglong2*>(
                P.pt_base + (size_t)idx * P.pt_stride + coef));
          } else {
            const uint64_t v = __ldg(P.pt_base + (size_t)idx * P.pt_stride + pcoef);
            pv[u] = make_ulonglong2(v, v);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int t = t0 + u;
          if (t >= nt) break;
#pragma unroll
          for (int b = 0; b < NB; ++b) {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const ulonglong2 bv = *reinterpret_cast<const ulonglong2*>(
                  sm + t * per_term + b * 2 * kBsgsTile + c * kBsgsTile + xi);
              acc[b][c][0].add(bv.x, pv[u].x);
              acc[b][c][1].add(bv.y, pv[u].y);
            }
          }
        }
        if ((t0 + 4) % kMacFold == 0) {  // 4 products per accumulator per t0 step
#pragma unroll
          for (int b = 0; b < NB; ++b)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              acc[b][c][0].fold(pc.q, pc.bar);
              acc[b][c][1].fold(pc.q, pc.bar);
            }
        }
      }
    }
  }
  if (g >= ng) return;
#pragma unroll
  for (int b = 0; b < NB; ++b) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      uint64_t r[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) r[h] = mont_mul(acc[b][c][h].redc(pc), pc.r2, pc.q, pc.qinv_neg);
      *reinterpret_cast<ulonglong2*>(P.out + (g0 + g) * P.out_gstride + b * P.bstride +
                                     c * P.c1_off + coef) = make_ulonglong2(r[0], r[1]);
    }
  }
}

// Run-compressed diagonals (pt_log_run >= 4): the problem per 32-coefficient
// tile of one limb is a small GEMM, out[g][col] = sum_t P[g][t] * B[t][col],
// with P (giants x terms, one word per run) and B (terms x NB*2*32 columns).
// The CTA stages B and its P slice in shared memory, then each thread
// accumulates GPT giants x 2 adjacent columns (2*GPT independent accumulators)
// reading one 16-byte baby word and GPT/2 broadcast 16-byte P words (P is
// stored [term][run][giant]) per term.
constexpr int kRunTile = 32;   // coefficients per CTA
constexpr int kRunGiants = 32; // giants per CTA (grid.z covers more)
#ifndef HEGPU_RUN_CHUNK
#define HEGPU_RUN_CHUNK 16  // measured: 16 -> 15.2 ms BSGS MAC per step, 32 -> 15.5, 64 -> 24.7
#endif
#ifndef HEGPU_RUN_GPT
#define HEGPU_RUN_GPT 4
#endif
constexpr int kRunChunk = HEGPU_RUN_CHUNK;  // terms per shared-memory stage (double-buffered)

// a run's row of giants is padded by one 16-byte slot so the (up to 4) runs a
// warp reads in one step sit in different banks
constexpr int run_row(int ng) { return ng + 2; }
constexpr size_t bsgs_run_smem(int ng, int rt) {
  return (size_t)2 * kRunChunk * (2 * kRunTile + run_row(ng) * rt) * 8;  // two stage buffers
}

// RT = runs per tile (2 for pt_log_run 4, 1 for 5); one batch element per CTA.
template <int RT, int GPT, int NG>
__global__ void __launch_bounds__(32 * (NG / GPT), GPT == 8 ? 3 : 2)
    k_bsgs_run(const __grid_constant__ BsgsParams P) {
  constexpr int kRunGpt = GPT;
  constexpr int kRunGiants = NG;  // giants per CTA
  extern __shared__ __align__(16) uint64_t sm[];
  constexpr int COLS = 2 * kRunTile;  // (c0, c1) x 32 coefficients
  constexpr int LR = RT == 4 ? 3 : RT == 2 ? 4 : 5;
  constexpr int RROW = run_row(NG);
  constexpr int BUF = kRunChunk * (COLS + RROW * RT);  // words per stage buffer
  const int N = 1 << P.log_n;
  // grid (giant groups, tiles, limbs): the groups staging the same baby tile
  // run back to back, so all but the first read it from L2
  const int limb = blockIdx.z;
  const int x0 = blockIdx.y * kRunTile;
  const int g0 = blockIdx.x * kRunGiants;
  const int T = P.n_terms;
  const int nch = (T + kRunChunk - 1) / kRunChunk;
  // terms are staged kRunChunk at a time into one of two buffers (babies
  // [t][2][32], diagonals [t][RT][32 giants]), all by cp.async: chunk c + 1
  // loads while chunk c is multiplied; accumulators carry across chunks
  constexpr int PAIRS = kRunTile;  // (c, x pair)
  const int p = threadIdx.x % PAIRS, gg = threadIdx.x / PAIRS;
  const int c = p / (kRunTile / 2), xl = (p % (kRunTile / 2)) * 2;
  const int run = xl >> LR;
  const PrimeConst pc = P.pc[limb < P.kq ? limb : P.n_chain + (limb - P.kq)];
  // products < q^2; fold often enough to stay below 2^128 (see Mac128)
  const int fold_every = pc.q < (1ull << 61) ? 32 : kMacFold;
  Mac128 acc[kRunGpt][2];
#pragma unroll
  for (int g = 0; g < kRunGpt; ++g) {
    acc[g][0].zero();
    acc[g][1].zero();
  }
  const size_t pcol = ((size_t)limb * N + x0) >> LR;
  auto stage = [&](int ch) {
    uint64_t* bab = sm + (size_t)(ch & 1) * BUF;
    uint64_t* pts = bab + (size_t)kRunChunk * COLS;
    const int tc = ch * kRunChunk;
    const int nt = T - tc < kRunChunk ? T - tc : kRunChunk;
    for (int e = threadIdx.x; e < nt * COLS / 2; e += blockDim.x) {
      const int t = e / (COLS / 2), rem = e - t * (COLS / 2);
      const int cc = rem / (kRunTile / 2), xx = (rem - cc * (kRunTile / 2)) * 2;
      cp_async16(bab + (size_t)t * COLS + cc * kRunTile + xx,
                 P.baby[tc + t] + cc * P.c1_off + (size_t)limb * N + x0 + xx);
    }
    // giant-major within a term: consecutive threads fill consecutive words
    // of the [t][run][giant] layout (conflict-free shared-memory writes)
    for (int e = threadIdx.x; e < kRunGiants * nt; e += blockDim.x) {
      const int t = e / kRunGiants, g = e - t * kRunGiants;
      const int idx =
          g0 + g < P.n_giants ? __ldg(P.pt_idx + (size_t)(g0 + g) * T + tc + t) : -1;
      uint64_t* d = pts + (size_t)t * RT * RROW + g;
      const uint64_t* srcp = P.pt_base + (size_t)(idx < 0 ? 0 : idx) * P.pt_stride + pcol;
#pragma unroll
      for (int r = 0; r < RT; ++r) {
        if (idx < 0)
          d[r * RROW] = 0;
        else
          cp_async8(d + r * RROW, srcp + r);
      }
    }
    cp_async_commit();
  };
  stage(0);
  int since = 0;
#pragma unroll 1
  for (int ch = 0; ch < nch; ++ch) {
    if (ch + 1 < nch) {
      stage(ch + 1);
      cp_async_wait_group<1>();  // chunk ch has landed, ch + 1 in flight
    } else {
      cp_async_wait_group<0>();
    }
    __syncthreads();
    const uint64_t* bab = sm + (size_t)(ch & 1) * BUF;
    const uint64_t* pts = bab + (size_t)kRunChunk * COLS;
    const uint64_t* pt_g = pts + run * RROW + gg * kRunGpt;
    const uint64_t* bab_c = bab + c * kRunTile + xl;
    const int nt = T - ch * kRunChunk < kRunChunk ? T - ch * kRunChunk : kRunChunk;
#pragma unroll 2
    for (int t = 0; t < nt; ++t) {
      const ulonglong2 bv = *reinterpret_cast<const ulonglong2*>(bab_c + (size_t)t * COLS);
      const ulonglong2* pp =
          reinterpret_cast<const ulonglong2*>(pt_g + (size_t)t * RT * RROW);
#pragma unroll
      for (int h = 0; h < kRunGpt / 2; ++h) {
        const ulonglong2 pv = pp[h];
        acc[2 * h][0].add(bv.x, pv.x);
        acc[2 * h][1].add(bv.y, pv.x);
        acc[2 * h + 1][0].add(bv.x, pv.y);
        acc[2 * h + 1][1].add(bv.y, pv.y);
      }
      if (++since == fold_every) {
        since = 0;
#pragma unroll
        for (int g = 0; g < kRunGpt; ++g) {
          acc[g][0].fold(pc.q, pc.bar);
          acc[g][1].fold(pc.q, pc.bar);
        }
      }
    }
    __syncthreads();  // buffer ch & 1 is restaged for chunk ch + 2
  }
#pragma unroll
  for (int g = 0; g < kRunGpt; ++g) {
    const int gi = g0 + gg * kRunGpt + g;
    if (gi >= P.n_giants) break;
    const uint64_t r0 = mont_mul(acc[g][0].redc(pc), pc.r2, pc.q, pc.qinv_neg);
    const uint64_t r1 = mont_mul(acc[g][1].redc(pc), pc.r2, pc.q, pc.qinv_neg);
    *reinterpret_cast<ulonglong2*>(P.out + (size_t)gi * P.out_gstride + c * P.c1_off +
                                   (size_t)limb * N + x0 + xl) = make_ulonglong2(r0, r1);
  }
}
template <int RT, int GPT, int NG>
static void launch_bsgs_run_g(const BsgsParams& P, int k, cudaStream_t st) {
  const size_t smem = bsgs_run_smem(NG, RT);
  static bool attr_set = false;
  if (!attr_set) {
    check_cuda(cudaFuncSetAttribute(k_bsgs_run<RT, GPT, NG>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "bsgs smem attr");
    attr_set = true;
  }
  dim3 grid((P.n_giants + NG - 1) / NG, (1 << P.log_n) / kRunTile, k);
  k_bsgs_run<RT, GPT, NG><<<grid, 32 * (NG / GPT), smem, st>>>(P);
}

// 4 giants x 2 columns per thread (8 accumulators, 256 threads): measured
// 1.38 T products/s vs 1.19 (8 giants, 128 threads) and 1.00 (2 giants) on
// the CtS shape; the register-only ceiling of Mac128 is 2.16 T/s.
// a CTA covers 32 giants, or 16 when the transform has no more (its thread
// groups would otherwise idle)
template <int RT>
static void launch_bsgs_run(const BsgsParams& P, int k, cudaStream_t st) {
  if (P.n_giants <= 16)
    launch_bsgs_run_g<RT, HEGPU_RUN_GPT, 16>(P, k, st);
  else
    launch_bsgs_run_g<RT, HEGPU_RUN_GPT, kRunGiants>(P, k, st);
}

// ---------------------------------------------------------------------------
// Run-compressed BSGS MAC on the tensor cores (pt_log_run >= 3).  Within one
// run of 2^LR coefficients the product is a small exact GEMM,
//   out[g][col] = sum_t P[g][t] * B[t][col]   (mod q),
// with 16 giants x 8 columns x 32 terms per IMMA m16n8k32 tile.  Both operands
// (< 2^64) are split into byte planes a = sum_i a_i 2^(8i); the u8 x u8 -> s32
// products of plane pair (i, j) accumulate into sum_{i+j=s} of shift s (at most
// 8 pairs x 255^2 x 256 terms < 2^31), and the epilogue recombines the
// 15 shifts into the exact 128-bit sum (< 256 q^2 < 2^128) before one Barrett /
// Montgomery reduction: the limbs are identical to k_bsgs_run's.
// CTA = 8 warps over 32 coefficients x 16 giants of one limb; warp w owns the
// 8-column tile w (component w / 4, coefficients 8 (w % 4) ..).  32-term
// chunks of raw words arrive by cp.async (double-buffered); the diagonals'
// byte planes are built once per CTA in shared memory, each lane builds its
// own B fragments from its column's raw words (PRMT transposes).
// ---------------------------------------------------------------------------
#ifndef HEGPU_BSGS_MMA
#define HEGPU_BSGS_MMA 1
#endif
#ifndef HEGPU_MMA_BDIRECT
#define HEGPU_MMA_BDIRECT 1  // B fragments built in registers from the raw chunk
#endif
constexpr int kMmaNbuf = 2;  // raw chunk buffers (1 buffer at 3 CTAs/SM measured 17% slower)
constexpr bool kMmaBDirect = HEGPU_MMA_BDIRECT != 0;
constexpr int kMmaGiants = 16;
constexpr int kMmaTile = 32;  // coefficients per CTA

// 4 x u64 -> 8 byte planes: plane p = bytes p of (v0, v1, v2, v3), v0 lowest
__device__ __forceinline__ void byte_planes4(const uint64_t (&v)[4], uint32_t (&pl)[8]) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint32_t w0 = static_cast<uint32_t>(v[0] >> (32 * h));
    const uint32_t w1 = static_cast<uint32_t>(v[1] >> (32 * h));
    const uint32_t w2 = static_cast<uint32_t>(v[2] >> (32 * h));
    const uint32_t w3 = static_cast<uint32_t>(v[3] >> (32 * h));
    const uint32_t t0 = __byte_perm(w0, w1, 0x5140), t1 = __byte_perm(w0, w1, 0x7362);
    const uint32_t u0 = __byte_perm(w2, w3, 0x5140), u1 = __byte_perm(w2, w3, 0x7362);
    pl[4 * h + 0] = __byte_perm(t0, u0, 0x5410);
    pl[4 * h + 1] = __byte_perm(t0, u0, 0x7632);
    pl[4 * h + 2] = __byte_perm(t1, u1, 0x5410);
    pl[4 * h + 3] = __byte_perm(t1, u1, 0x7632);
  }
}

// word swizzle of an 8-word (32-term) row: conflict-free fragment loads
// (8 consecutive rows x 4 words) and staging stores (32 consecutive rows)
__device__ __forceinline__ int mma_sw(int row) {
  return (((row >> 2) & 1) << 2) | ((row >> 3) & 3);
}

__device__ __forceinline__ void imma_u8(int (&d)[4], const uint32_t (&a)[4], uint32_t b0,
                                        uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// shared-memory plan of k_bsgs_mma: raw u64 chunks (double-buffered, cp.async),
// byte planes of the current chunk, and the CTA's diagonal-index table
template <int RT, int MG>
struct MmaSmem {
  static constexpr int NGC = kMmaGiants * MG;             // giants per CTA
  static constexpr int COLS = 2 * kMmaTile;
  // raw babies [t][col], rows padded by 16 B when the B fragments are read
  // straight from them (4 term rows of one fragment fall in 2 wavefronts)
  static constexpr int BSTR = COLS + (kMmaBDirect ? 2 : 0);
  static constexpr int RAW_B = 32 * BSTR;
  static constexpr int RAW_A = 32 * NGC * RT;      // u64 words [t][giant][run]
  static constexpr int PL_B = kMmaBDirect ? 0 : 8 * COLS * 8;  // u32 [plane][col][8]
  static constexpr int PL_A = 8 * RT * NGC * 8;    // u32 words [plane][run][giant][8]
  static size_t bytes(int T) {
    return (size_t)kMmaNbuf * (RAW_B + RAW_A) * 8 + (size_t)(PL_B + PL_A) * 4 +
           (size_t)NGC * T * 4;
  }
};

// MG = 16-giant m-tiles per CTA (8 warps each): MG = 2 stages and converts the
// babies' planes once for 32 giants
template <int RT, int MG>
__global__ void __launch_bounds__(256 * MG, MG == 2 ? 1 : 2)
    k_bsgs_mma(const __grid_constant__ BsgsParams P) {
  using L = MmaSmem<RT, MG>;
  constexpr int NGC = L::NGC, NT = 256 * MG;
  constexpr int LR = RT == 4 ? 3 : RT == 2 ? 4 : 5;
  constexpr int COLS = L::COLS;
  extern __shared__ __align__(16) uint64_t smem_mma[];
  uint64_t* raw_b = smem_mma;                       // 2 buffers
  uint64_t* raw_a = raw_b + kMmaNbuf * L::RAW_B;
  uint32_t* Bs = reinterpret_cast<uint32_t*>(raw_a + kMmaNbuf * L::RAW_A);
  uint32_t* As = Bs + L::PL_B;
  int* s_idx = reinterpret_cast<int*>(As + L::PL_A);
  const int N = 1 << P.log_n;
  const int limb = blockIdx.z;
  const int x0 = blockIdx.y * kMmaTile;
  const int g0 = blockIdx.x * NGC;
  const int T = P.n_terms;
  const int nch = (T + 31) >> 5;
  const PrimeConst pc = P.pc[limb < P.kq ? limb : P.n_chain + (limb - P.kq)];
  const int nby = (64 - __clzll(pc.q) + 7) >> 3;  // byte planes in use
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = warp >> 3;                          // this warp's 16-giant m-tile
  const int comp = (warp & 7) >> 2, xo = (warp & 3) * 8;  // and 8-column tile
  const int run = xo >> LR;
  const size_t pcol = ((size_t)limb * N + x0) >> LR;
  for (int e = threadIdx.x; e < NGC * T; e += NT) {
    const int g = e / T, t = e - g * T;
    s_idx[e] = g0 + g < P.n_giants ? __ldg(P.pt_idx + (size_t)(g0 + g) * T + t) : -1;
  }
  __syncthreads();
  // raw chunk ch -> buffer ch & 1 (terms past T and absent diagonals are
  // zero-filled by plain stores)
  auto stage = [&](int ch) {
    uint64_t* rb = raw_b + (ch % kMmaNbuf) * L::RAW_B;
    uint64_t* ra = raw_a + (ch % kMmaNbuf) * L::RAW_A;
    const int tc = ch * 32;
    for (int e = threadIdx.x; e < 32 * COLS / 2; e += NT) {
      const int t = e / (COLS / 2), j = (e % (COLS / 2)) * 2;
      const int c = j / kMmaTile, xl = j % kMmaTile;
      uint64_t* d = rb + t * L::BSTR + j;
      if (tc + t < T)
        cp_async16(d, P.baby[tc + t] + c * P.c1_off + (size_t)limb * N + x0 + xl);
      else
        *reinterpret_cast<ulonglong2*>(d) = make_ulonglong2(0, 0);
    }
    for (int e = threadIdx.x; e < 32 * NGC; e += NT) {
      const int t = e / NGC, g = e % NGC;
      const int idx = tc + t < T ? s_idx[g * T + tc + t] : -1;
      uint64_t* d = ra + (t * NGC + g) * RT;
      const uint64_t* src = P.pt_base + (size_t)(idx < 0 ? 0 : idx) * P.pt_stride + pcol;
#pragma unroll
      for (int r = 0; r < RT; r += (RT >= 2 ? 2 : 1)) {
        if (RT >= 2) {
          if (idx < 0)
            *reinterpret_cast<ulonglong2*>(d + r) = make_ulonglong2(0, 0);
          else
            cp_async16(d + r, src + r);
        } else {
          if (idx < 0)
            d[r] = 0;
          else
            cp_async8(d + r, src + r);
        }
      }
    }
    cp_async_commit();
  };
  int acc[15][4];
#pragma unroll
  for (int s = 0; s < 15; ++s)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[s][i] = 0;
  const int fr = lane >> 2, fq = lane & 3;  // fragment row / word
  stage(0);
#pragma unroll 1
  for (int ch = 0; ch < nch; ++ch) {
    cp_async_wait_group<0>();
    __syncthreads();  // raw chunk ch landed; planes of ch - 1 consumed
    if (ch + 1 < nch) stage(ch + 1);
    const uint64_t* rb = raw_b + (ch % kMmaNbuf) * L::RAW_B;
    const uint64_t* ra = raw_a + (ch % kMmaNbuf) * L::RAW_A;
    // ---- byte planes: babies (64 cols x 8 term quads) ------------------------
    for (int e = threadIdx.x; e < (kMmaBDirect ? 0 : COLS * 8); e += NT) {
      const int j = e % COLS, q = e / COLS;
      uint64_t v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) v[i] = rb[(4 * q + i) * L::BSTR + j];
      uint32_t pl[8];
      byte_planes4(v, pl);
      const int w = j * 8 + (q ^ mma_sw(j));
#pragma unroll
      for (int p = 0; p < 8; ++p)
        if (p < nby) Bs[p * COLS * 8 + w] = pl[p];
    }
    // ---- diagonals: 16 giants x 8 quads x RT runs -----------------------------
    for (int e = threadIdx.x; e < NGC * 8 * RT; e += NT) {
      const int g = e % NGC, q = (e / NGC) % 8, r = e / (NGC * 8);
      uint64_t v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) v[i] = ra[((4 * q + i) * NGC + g) * RT + r];
      uint32_t pl[8];
      byte_planes4(v, pl);
      const int w = (r * NGC + g) * 8 + (q ^ mma_sw(g));
#pragma unroll
      for (int p = 0; p < 8; ++p)
        if (p < nby) As[p * RT * NGC * 8 + w] = pl[p];
    }
    __syncthreads();
    // ---- MMAs: plane pairs (i, j) into shift i + j ----------------------------
    const int jb = comp * kMmaTile + xo + fr;  // this lane's B column
    uint32_t bf[8][2];
    if constexpr (kMmaBDirect) {
      // the lane's fragment words are byte planes of its own column's terms
      // 4 fq .. 4 fq + 3 and 4 fq + 16 .. 4 fq + 19: no shared-memory planes
      uint64_t v0[4], v1[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        v0[i] = rb[(4 * fq + i) * L::BSTR + jb];
        v1[i] = rb[(4 * fq + 16 + i) * L::BSTR + jb];
      }
      uint32_t p0[8], p1[8];
      byte_planes4(v0, p0);
      byte_planes4(v1, p1);
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        bf[p][0] = p0[p];
        bf[p][1] = p1[p];
      }
    } else {
      const uint32_t* bcol = Bs + jb * 8;
      const int bw0 = fq ^ mma_sw(jb), bw1 = (fq + 4) ^ mma_sw(jb);
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        bf[p][0] = bcol[p * COLS * 8 + bw0];
        bf[p][1] = bcol[p * COLS * 8 + bw1];
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i >= nby) break;
      const uint32_t* ap = As + i * RT * NGC * 8 + run * NGC * 8;
      const int ga = mt * 16 + fr, gb = ga + 8;
      uint32_t af[4];
      af[0] = ap[ga * 8 + (fq ^ mma_sw(ga))];
      af[1] = ap[gb * 8 + (fq ^ mma_sw(gb))];
      af[2] = ap[ga * 8 + ((fq + 4) ^ mma_sw(ga))];
      af[3] = ap[gb * 8 + ((fq + 4) ^ mma_sw(gb))];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j < nby) imma_u8(acc[i + j], af, bf[j][0], bf[j][1]);
      }
    }
  }
  // ---- epilogue: C rows fr / fr + 8 (giants), columns 2 fq, 2 fq + 1 ----------
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int gi = g0 + mt * 16 + fr + 8 * h;
    if (gi >= P.n_giants) continue;
    uint64_t r[2];
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      unsigned __int128 v = 0;
#pragma unroll
      for (int s = 0; s < 15; ++s)
        v += static_cast<unsigned __int128>(static_cast<uint32_t>(acc[s][2 * h + cc])) << (8 * s);
      Mac128 m;
      m.L = static_cast<uint64_t>(v);
      m.H = static_cast<uint64_t>(v >> 64);
      m.M = 0;
      m.c = 0;
      r[cc] = mont_mul(m.redc(pc), pc.r2, pc.q, pc.qinv_neg);
    }
    *reinterpret_cast<ulonglong2*>(P.out + (size_t)gi * P.out_gstride + comp * P.c1_off +
                                   (size_t)limb * N + x0 + xo + 2 * fq) =
        make_ulonglong2(r[0], r[1]);
  }
}

static bool bsgs_mma_enabled() {
  static const bool on = [] {
    const char* e = getenv("HEGPU_BSGS_MMA");
    return e ? e[0] == '1' : (HEGPU_BSGS_MMA != 0);
  }();
  return on;
}

#ifndef HEGPU_MMA_MG2
#define HEGPU_MMA_MG2 0  // 32-giant CTAs (512 threads, 1 CTA/SM): measured 37% slower
#endif
template <int RT, int MG>
static void launch_bsgs_mma_g(const BsgsParams& P, int k, cudaStream_t st) {
  using L = MmaSmem<RT, MG>;
  const size_t smem = L::bytes(P.n_terms);
  static bool attr_set = false;
  if (!attr_set) {
    check_cuda(cudaFuncSetAttribute(k_bsgs_mma<RT, MG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)L::bytes(kBsgsMaxTerms)),
               "bsgs mma smem attr");
    attr_set = true;
  }
  dim3 grid((P.n_giants + L::NGC - 1) / L::NGC, (1 << P.log_n) / kMmaTile, k);
  k_bsgs_mma<RT, MG><<<grid, 256 * MG, smem, st>>>(P);
}
template <int RT>
static void launch_bsgs_mma(const BsgsParams& P, int k, cudaStream_t st) {
  if (HEGPU_MMA_MG2 && P.n_giants > kMmaGiants)
    launch_bsgs_mma_g<RT, 2>(P, k, st);
  else
    launch_bsgs_mma_g<RT, 1>(P, k, st);
}

template <int NB>
static void launch_bsgs_nb(const BsgsParams& P, int k, cudaStream_t st) {
  constexpr int W = 16;  // <= 128 registers per thread (7-word accumulators)
  dim3 grid((1 << P.log_n) / kBsgsTile, k, (P.n_giants + W - 1) / W);
  k_bsgs<NB, W><<<grid, W * 32, 0, st>>>(P);
}

void launch_bsgs(const PrimeConst* dpc, int log_n, const uint64_t* const* babies, int n_terms,
                 int64_t c1_off, int64_t bstride, int n_batch, const uint64_t* pt_base,
                 int64_t pt_stride, int pt_log_run, const int32_t* pt_idx, int n_giants,
                 uint64_t* out, int64_t out_gstride, int k, cudaStream_t st, int kq,
                 int n_chain) {
  if (n_terms < 1 || n_terms > kBsgsMaxTerms) throw HegpuError{HEGPU_E_ARG, "bsgs: 1..256 terms"};
  if (pt_log_run < 0 || pt_log_run > 5 || pt_log_run >= log_n)
    throw HegpuError{HEGPU_E_ARG, "bsgs: pt_log_run must be in [0, 5]"};
  if ((1 << log_n) % kBsgsTile) throw HegpuError{HEGPU_E_ARG, "bsgs: N too small"};
  const int max_giants = 1 << 20;  // giant groups are a grid dimension
  for (int b0 = 0; b0 < n_batch; b0 += 2) {
    const int nb = n_batch - b0 < 2 ? n_batch - b0 : 2;
    for (int g0 = 0; g0 < n_giants; g0 += max_giants) {
      BsgsParams P;
      for (int t = 0; t < n_terms; ++t) P.baby[t] = babies[t] + b0 * bstride;
      P.n_terms = n_terms;
      P.n_giants = n_giants - g0 < max_giants ? n_giants - g0 : max_giants;
      P.n_batch = nb;
      P.log_n = log_n;
      P.c1_off = c1_off;
      P.bstride = bstride;
      P.pt_base = pt_base;
      P.pt_stride = pt_stride;
      P.pt_log_run = pt_log_run;
      P.pt_idx = pt_idx + (size_t)g0 * n_terms;
      P.out = out + (size_t)g0 * out_gstride + b0 * bstride;
      P.out_gstride = out_gstride;
      P.pc = dpc;
      P.kq = kq;
      P.n_chain = n_chain;
      const double el = (double)k * (1 << log_n);
      ProfScope ps(PROF_DIAG_MAC, st,
                   el * 8.0 * ((double)P.n_giants * n_terms / (1 << pt_log_run) +
                               2.0 * nb * (n_terms + P.n_giants)),
                   el * 2.0 * nb * ((double)P.n_giants * n_terms + P.n_giants));
      if (pt_log_run >= 3 && (1 << log_n) % kRunTile == 0) {
        // one batch element per launch: 16 accumulators per thread at 3 CTAs/SM
        // (the compressed diagonals are re-read per element, 1/16 of a baby)
        for (int bi = 0; bi < nb; ++bi) {
          BsgsParams Q = P;
          for (int t = 0; t < n_terms; ++t) Q.baby[t] = P.baby[t] + bi * bstride;
          Q.out = P.out + bi * bstride;
          Q.n_batch = 1;
          if (bsgs_mma_enabled()) {
            if (pt_log_run == 3)
              launch_bsgs_mma<4>(Q, k, st);
            else if (pt_log_run == 4)
              launch_bsgs_mma<2>(Q, k, st);
            else
              launch_bsgs_mma<1>(Q, k, st);
          } else if (pt_log_run == 3)
            launch_bsgs_run<4>(Q, k, st);
          else if (pt_log_run == 4)
            launch_bsgs_run<2>(Q, k, st);
          else
            launch_bsgs_run<1>(Q, k, st);
        }
      } else if (nb == 1) {
        launch_bsgs_nb<1>(P, k, st);
      } else {
        launch_bsgs_nb<2>(P, k, st);
      }
      check_cuda(cudaGetLastError(), "bsgs launch");
    }
  }
}

}  // namespace hegpu
