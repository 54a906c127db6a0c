// GPU canonical-embedding encode of the full-slot bootstrap diagonals
// (sm_100a, FP64).
//
// The reference re-encodes every linear-transform diagonal on the host for
// every bootstrap (hebert/bootstrap.py:200-247): numpy FFT of a 2^16-point
// spectrum per diagonal, 196,609 of them per full-slot bootstrap at N = 2^16.
// Sparse contexts cache their diagonals in HBM (bootstrap.py here); full-slot
// contexts cannot (1.8 TiB), so their diagonals are generated and encoded on
// the device, one giant step at a time:
//
//   value    closed forms of bootstrap.py:_cts_diag_full / _stc_diag_full
//            (hebert/bootstrap.py:174-197), rolled by the giant step and
//            optionally conjugated (bootstrap.py:219-236);
//   spectrum spec[slot_idx[j]] = v_j * scale, spec[conj_idx[j]] = conj(.)
//            (hebert/ckks/encoding.py:17-30, 62-97), generated on the fly
//            through a discrete-log table of 5 mod 2N;
//   FFT      numpy's forward transform sum_m spec[m] e^{-2 pi i m k / N},
//            four-step N = N1 * N2 in two shared-memory passes;
//   round    c_k = rint(Re(X_k * conj(zeta^k)) / N) -> int64.
//
// The integer coefficients then go through the usual signed lift + NTT.  The
// float rounding differs from numpy's in the last bits, so an encoded
// diagonal may differ by +-1 in a coefficient: bootstrapping is
// tolerance-gated (hebert tests bootstrap to 1e-2, T/test_bootstrap.py:23).
#include <cmath>
#include <vector>

#include "ring.cuh"

namespace hegpu {

constexpr int kEncCols = 8;  // transform columns per CTA

struct DiagEncParams {
  int kind, half, log_n, n_diags;
  double fold, scale;
  const int32_t* dlog;  // spectrum index m -> slot j | (conj << 30)
  const int32_t* pow5;  // j -> 5^j mod 2N, j < N/2
  const double2* eroot; // e -> exp(i pi e / N), e < 2N (every root the encoder needs)
  double2* y;           // pass A -> pass B scratch [diag][N]
  int64_t* out;         // [diag][N] rounded coefficients
  int* overflow;
  int32_t d[kEncMaxDiags];
  int32_t g0c[kEncMaxDiags];  // giant step | (conjugate << 30)
};

// Slot value R[j] of diagonal i (rolled by its giant step, maybe conjugated).
__device__ __forceinline__ double2 diag_value(const DiagEncParams& P, int i, int j) {
  const int n = 1 << P.log_n, s = n >> 1;
  const int g0 = P.g0c[i] & ((1 << 30) - 1);
  const bool conj = (P.g0c[i] >> 30) & 1;
  const int d = P.d[i];
  const int src = (j - g0) & (s - 1);  // np.roll(vals, g0)[j] = vals[(j - g0) mod s]
  const long long two_n2 = 2LL * n;
  long long e;
  if (P.kind == 0) {  // CoeffToSlot: e = -(row) * 5^((src + d) mod s) mod 2N
    const long long row = src + (long long)P.half * s;
    e = (-(row * P.pow5[(src + d) & (s - 1)])) % two_n2;
  } else {  // SlotToCoeff: e = 5^src * (((src + d) mod s) + half s) mod 2N
    const long long col = ((src + d) & (s - 1)) + (long long)P.half * s;
    e = ((long long)P.pow5[src] * col) % two_n2;
  }
  if (e < 0) e += two_n2;
  const double2 r = P.eroot[e];  // exp(i pi e / N)
  return make_double2(r.x * P.fold, (conj ? -r.y : r.y) * P.fold);
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// kEncCols independent L-point forward DFTs (e^{-2 pi i / L}) on buf[c][L],
// input in bit-reversed order; tw[t] = e^{-2 pi i t / L}, t < L/2.
__device__ void smem_dft(double2* buf, const double2* tw, int log_l) {
  const int L = 1 << log_l;
  const int nb = (L >> 1) * kEncCols;
  for (int ls = 1; ls <= log_l; ++ls) {
    const int half = 1 << (ls - 1);
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
      const int c = b >> (log_l - 1), r = b & ((L >> 1) - 1);
      const int pos = r & (half - 1), grp = r >> (ls - 1);
      const int i0 = c * L + (grp << ls) + pos, i1 = i0 + half;
      const double2 w = tw[pos << (log_l - ls)];
      const double2 u = buf[i0], v = cmul(buf[i1], w);
      buf[i0] = make_double2(u.x + v.x, u.y + v.y);
      buf[i1] = make_double2(u.x - v.x, u.y - v.y);
    }
    __syncthreads();
  }
}

__device__ __forceinline__ int bitrev(int x, int bits) { return __brev(x) >> (32 - bits); }

// tw[t] = e^{-2 pi i t / L} = eroot[-2 t N / L mod 2N]
__device__ void fill_twiddles(double2* tw, int log_l, const double2* eroot, int log_n) {
  const int L = 1 << log_l, two_n = 2 << log_n;
  for (int t = threadIdx.x; t < L / 2; t += blockDim.x)
    tw[t] = eroot[(two_n - ((2 * t) << (log_n - log_l))) & (two_n - 1)];
}

// pass A: columns m2 of x[N2 m1 + m2], DFT over m1, twiddle e^{-2 pi i m2 k1 / N},
// store y[k1 N2 + m2]
__global__ void __launch_bounds__(256) k_enc_pass_a(const __grid_constant__ DiagEncParams P) {
  extern __shared__ double2 esm[];
  const int n = 1 << P.log_n, a = (P.log_n + 1) / 2, n1 = 1 << a, n2 = n >> a;
  double2* buf = esm;
  double2* tw = esm + kEncCols * n1;
  const int i = blockIdx.y;
  const int m2_0 = blockIdx.x * kEncCols;
  fill_twiddles(tw, a, P.eroot, P.log_n);
  for (int e = threadIdx.x; e < kEncCols * n1; e += blockDim.x) {
    const int c = e / n1, m1 = e - c * n1;
    const int m = n2 * m1 + m2_0 + c;
    const int code = P.dlog[m];
    double2 v = diag_value(P, i, code & ((1 << 30) - 1));
    v.x *= P.scale;
    v.y *= P.scale;
    if (code >> 30) v.y = -v.y;  // conjugate spectrum index
    buf[c * n1 + bitrev(m1, a)] = v;
  }
  __syncthreads();
  smem_dft(buf, tw, a);
  double2* y = P.y + (size_t)i * n;
  for (int e = threadIdx.x; e < kEncCols * n1; e += blockDim.x) {
    const int k1 = e / kEncCols, c = e - k1 * kEncCols;
    const int m2 = m2_0 + c;
    // e^{-2 pi i m2 k1 / N} = eroot[-2 (m2 k1 mod N) mod 2N]
    const double2 w = P.eroot[(2 * n - 2 * ((m2 * k1) & (n - 1))) & (2 * n - 1)];
    y[(size_t)k1 * n2 + m2] = cmul(buf[c * n1 + k1], w);
  }
}

// pass B: rows k1 of y, DFT over m2 -> X[k1 + N1 k2], untwist by conj(zeta^k),
// scale 1/N, rint -> int64
__global__ void __launch_bounds__(256) k_enc_pass_b(const __grid_constant__ DiagEncParams P) {
  extern __shared__ double2 esm[];
  const int n = 1 << P.log_n, a = (P.log_n + 1) / 2, n1 = 1 << a, b = P.log_n - a,
            n2 = 1 << b;
  double2* buf = esm;
  double2* tw = esm + kEncCols * n2;
  const int i = blockIdx.y;
  const int k1_0 = blockIdx.x * kEncCols;
  fill_twiddles(tw, b, P.eroot, P.log_n);
  const double2* y = P.y + (size_t)i * n;
  for (int e = threadIdx.x; e < kEncCols * n2; e += blockDim.x) {
    const int c = e / n2, m2 = e - c * n2;
    buf[c * n2 + bitrev(m2, b)] = y[(size_t)(k1_0 + c) * n2 + m2];
  }
  __syncthreads();
  smem_dft(buf, tw, b);
  int64_t* out = P.out + (size_t)i * n;
  const double inv_n = 1.0 / n;
  for (int e = threadIdx.x; e < kEncCols * n2; e += blockDim.x) {
    const int k2 = e / kEncCols, c = e - k2 * kEncCols;
    const int k = k1_0 + c + n1 * k2;
    const double2 z = P.eroot[k];  // zeta^k = exp(i pi k / N)
    const double2 x = buf[c * n2 + k2];
    const double v = rint((x.x * z.x + x.y * z.y) * inv_n);
    if (!(fabs(v) < 4611686018427387904.0)) atomicExch(P.overflow, 1);  // 2^62
    out[k] = (int64_t)v;
  }
}

const EncTables& Ring::enc_tables() {
  std::lock_guard<std::mutex> lk(mu);
  if (enc.dlog) return enc;
  const int s = n / 2;
  const uint64_t two_n = 2ull * n;
  std::vector<int32_t> pw(s), dl(n, -1);
  std::vector<double2> er(2 * (size_t)n);
  for (int e = 0; e < 2 * n; ++e) {  // exp(i pi e / N) in long double
    const long double ang = 3.141592653589793238462643383279503L * e / n;
    er[e] = make_double2((double)cosl(ang), (double)sinl(ang));
  }
  uint64_t g = 1;
  for (int j = 0; j < s; ++j) {
    pw[j] = (int32_t)g;
    dl[(g - 1) / 2] = j;                          // slot_idx[j] = (5^j - 1) / 2
    dl[n - 1 - (g - 1) / 2] = j | (1 << 30);      // conj_idx[j] = N - 1 - slot_idx[j]
    g = g * 5 % two_n;
  }
  check_cuda(cudaMalloc(&enc.dlog, n * sizeof(int32_t)), "alloc dlog");
  check_cuda(cudaMalloc(&enc.pow5, s * sizeof(int32_t)), "alloc pow5");
  check_cuda(cudaMalloc(&enc.overflow, sizeof(int)), "alloc flag");
  check_cuda(cudaMalloc(&enc.eroot, er.size() * sizeof(double2)), "alloc roots");
  check_cuda(cudaMemcpy(enc.eroot, er.data(), er.size() * sizeof(double2),
                        cudaMemcpyHostToDevice), "roots");
  check_cuda(cudaMemcpy(enc.dlog, dl.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice), "dlog");
  check_cuda(cudaMemcpy(enc.pow5, pw.data(), s * sizeof(int32_t), cudaMemcpyHostToDevice), "pow5");
  check_cuda(cudaMemset(enc.overflow, 0, sizeof(int)), "flag");
  return enc;
}

void launch_encode_diags(Ring& R, int kind, int half, double fold, double scale, int n_diags,
                         const int32_t* d, const int32_t* g0, const uint8_t* conj,
                         double2* scratch, int64_t* out, cudaStream_t st) {
  if (R.log_n < 6) throw HegpuError{HEGPU_E_ARG, "diagonal encode needs N >= 2^6"};
  if (kind != 0 && kind != 1) throw HegpuError{HEGPU_E_ARG, "diagonal kind must be 0 or 1"};
  if (half != 0 && half != 1) throw HegpuError{HEGPU_E_ARG, "half must be 0 or 1"};
  const EncTables& T = R.enc_tables();
  static bool attr_set = false;  // up to (8 + 1) * 512 * 16 B = 72 KiB at N = 2^17
  if (!attr_set) {
    const int mx = (kEncCols + 1) * 512 * (int)sizeof(double2);
    check_cuda(cudaFuncSetAttribute(k_enc_pass_a, cudaFuncAttributeMaxDynamicSharedMemorySize, mx),
               "enc smem");
    check_cuda(cudaFuncSetAttribute(k_enc_pass_b, cudaFuncAttributeMaxDynamicSharedMemorySize, mx),
               "enc smem");
    attr_set = true;
  }
  const int n = R.n, s = n / 2;
  const int a = (R.log_n + 1) / 2, b = R.log_n - a;
  for (int c0 = 0; c0 < n_diags; c0 += kEncMaxDiags) {
    const int m = std::min(kEncMaxDiags, n_diags - c0);
    DiagEncParams P;
    P.kind = kind;
    P.half = half;
    P.log_n = R.log_n;
    P.n_diags = m;
    P.fold = fold;
    P.scale = scale;
    P.dlog = T.dlog;
    P.pow5 = T.pow5;
    P.eroot = T.eroot;
    P.y = scratch;
    P.out = out + (size_t)c0 * n;
    P.overflow = T.overflow;
    for (int i = 0; i < m; ++i) {
      if (d[c0 + i] < 0 || d[c0 + i] >= s || g0[c0 + i] < 0 || g0[c0 + i] >= s)
        throw HegpuError{HEGPU_E_ARG, "diagonal / giant index out of range"};
      P.d[i] = d[c0 + i];
      P.g0c[i] = g0[c0 + i] | (conj[c0 + i] ? (1 << 30) : 0);
    }
    const double bytes = (double)m * n * (16.0 * 2 + 8.0);
    {
      ProfScope ps(PROF_ENCODE, st, bytes, 0);
      const size_t smem = (size_t)(kEncCols + 1) * (1 << a) * sizeof(double2);
      k_enc_pass_a<<<dim3((1 << b) / kEncCols, m), 256, smem, st>>>(P);
    }
    {
      ProfScope ps(PROF_ENCODE, st, bytes, 0);
      const size_t smem = (size_t)(kEncCols + 1) * (1 << b) * sizeof(double2);
      k_enc_pass_b<<<dim3((1 << a) / kEncCols, m), 256, smem, st>>>(P);
    }
    check_cuda(cudaGetLastError(), "encode launch");
  }
}

bool encode_overflow_check(Ring& R) {
  const EncTables& T = R.enc_tables();
  int flag = 0;
  check_cuda(cudaMemcpy(&flag, T.overflow, sizeof(int), cudaMemcpyDeviceToHost), "flag read");
  if (flag) check_cuda(cudaMemset(T.overflow, 0, sizeof(int)), "flag reset");
  return flag != 0;
}

}  // namespace hegpu
