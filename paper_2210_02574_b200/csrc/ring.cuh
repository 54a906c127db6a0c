// Host-side ring context and internal launch API of libhegpu.
#pragma once
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "hegpu.h"

namespace hegpu {

// Device constants for hybrid key switching at one (level, alpha), derived
// from BaseConverter (keys.py:19-49) and _p_inv_consts (keys.py:264-275).
struct KsLevel {
  int level = 0, alpha = 0, beta = 0, n_ext = 0, K = 0;
  uint64_t* dmem = nullptr;
  // ModUp: for chain limb i <= level (digit j = i / alpha)
  const uint64_t* mu_inv = nullptr;     // (Q_j/q_i)^-1 mod q_i, natural   [level+1]
  const uint64_t* mu_inv_sh = nullptr;  // Shoup companions                 [level+1]
  const uint64_t* mu_punc = nullptr;    // (Q_j/q_i mod p_t) R mod p_t      [level+1][n_ext]
  // ModDown: specials -> chain 0..level
  const uint64_t* md_inv = nullptr;     // [K]
  const uint64_t* md_inv_sh = nullptr;  // [K]
  const uint64_t* md_punc = nullptr;    // [K][level+1]
  std::vector<uint64_t> pinv, pinv_sh;  // P^-1 mod q_t, t <= level (host, kernel params)
  // final-stage constants of the post-scaled inverse NTTs that produce the
  // conversion inputs hat_i = x_i * inv_i directly (fused ModUp / ModDown)
  std::vector<ulonglong2> mu_fin_s, mu_fin_d;  // [level+1]
  std::vector<ulonglong2> md_fin_s, md_fin_d;  // [K]
  std::vector<int> dst_prime_of_digit;  // flattened [beta][n_ext] compact dst -> global prime
  // ModDown fused with the rescale (level >= 1): divide by D = q_level * P.
  // Sources are the acc rows level, level+1 .. level+K (q_level, specials).
  const uint64_t* mdr_punc = nullptr;          // (D/d_i mod q_t) R mod q_t  [K+1][level]
  const uint64_t* mdr_negd = nullptr;          // (-D mod q_t) R mod q_t      [level]
  // centered-conversion estimate (Seg::cmode 2): fp32 2^s_i / d_i and s_i,
  // one per 64-bit word (low 32 bits) [K+1]
  const uint64_t* mdr_fw_words = nullptr;
  const uint64_t* mdr_fs_words = nullptr;
  std::vector<ulonglong2> mdr_fin_s, mdr_fin_d;  // post-scaled INTT, [K+1]
  std::vector<uint64_t> dinv, dinv_sh;    // D^-1 mod q_t, t < level
  std::vector<uint64_t> qlinv, qlinv_sh;  // q_level^-1 mod q_t, t < level
  uint64_t p_mod_ql = 0;                  // P mod q_level
};

// device tables of the diagonal encoder (encode.cu), built on first use
struct EncTables {
  int32_t* dlog = nullptr;  // spectrum index -> slot | (conj << 30)
  int32_t* pow5 = nullptr;  // 5^j mod 2N
  int* overflow = nullptr;  // sticky |coefficient| >= 2^62 flag
  double2* eroot = nullptr; // exp(i pi e / N), e < 2N
};
constexpr int kEncMaxDiags = 256;  // diagonals per encode launch (kernel parameter space)

struct Ring {
  int log_n = 0, n = 0, n_chain = 0, n_special = 0, n_primes = 0;
  int device = 0;
  std::vector<uint64_t> primes;  // chain then special
  std::vector<PrimeConst> hpc;
  PrimeConst* dpc = nullptr;
  uint64_t* dtw = nullptr;  // [n_primes][4][N]: psi, psi_sh, ipsi, ipsi_sh
  void* dtwf = nullptr;     // FP64 twiddles of the primes < 2^kFpMaxBits (PrimeConst::twf)
  uint64_t fp_mask = 0;     // bit p: prime p has FP64 twiddles
  std::mutex mu;
  std::map<std::pair<int, int>, std::unique_ptr<KsLevel>> ks;
  // rescale constants: level -> (q_level^-1 mod q_i, shoup) for i < level
  std::map<int, std::pair<std::vector<uint64_t>, std::vector<uint64_t>>> rescale;

  EncTables enc;

  ~Ring();
  const EncTables& enc_tables();
  const KsLevel& ks_level(int level, int alpha);
  const std::pair<std::vector<uint64_t>, std::vector<uint64_t>>& rescale_consts(int level);
  int special_prime(int i) const { return n_chain + i; }
};

// --- host 128-bit helpers -------------------------------------------------
inline uint64_t h_mulmod(uint64_t a, uint64_t b, uint64_t q) {
  return static_cast<uint64_t>((static_cast<unsigned __int128>(a) * b) % q);
}
inline uint64_t h_powmod(uint64_t b, uint64_t e, uint64_t q) {
  uint64_t r = 1 % q;
  b %= q;
  while (e) {
    if (e & 1) r = h_mulmod(r, b, q);
    b = h_mulmod(b, b, q);
    e >>= 1;
  }
  return r;
}
inline uint64_t h_inv(uint64_t a, uint64_t q) { return h_powmod(a, q - 2, q); }  // q prime
inline uint64_t h_shoup(uint64_t w, uint64_t q) {
  return static_cast<uint64_t>((static_cast<unsigned __int128>(w) << 64) / q);
}
inline uint64_t h_rmod(uint64_t q) {  // 2^64 mod q
  return static_cast<uint64_t>((static_cast<unsigned __int128>(1) << 64) % q);
}
PrimeConst make_prime_const(uint64_t q, int log_n, uint64_t ipsi1);

// --- error state ------------------------------------------------------------
void set_error(const std::string& msg);
struct HegpuError {
  int code;
  std::string msg;
};
void check_cuda(cudaError_t e, const char* what);  // throws HegpuError

// --- launch accounting / profiling ------------------------------------------
// Every kernel launch bumps a global counter; when profiling is enabled the
// launch is bracketed by CUDA events on its stream and the device time is
// accumulated per kernel class (read back by hegpu_profile_read).
enum ProfClass {
  PROF_NTT = 0,
  PROF_ELEMENTWISE,
  PROF_LIFT,
  PROF_AUTOMORPHISM,
  PROF_TENSOR,
  PROF_CONV,
  PROF_KS_IP,
  PROF_DIAG_MAC,
  PROF_ENCRYPT,
  PROF_ENCODE,
  PROF_NUM_CLASSES
};
// bytes / modmuls: ALGORITHMIC traffic and modular multiplications of the
// launch (each input read once, each output written once).
// NTT launches are additionally attributed to the step that issued them
// (profile classes after PROF_NUM_CLASSES: ntt_modup, ntt_moddown, ntt_rescale).
enum NttTag { NTT_TAG_OTHER = 0, NTT_TAG_MODUP, NTT_TAG_MODDOWN, NTT_TAG_RESCALE, NTT_TAG_N };
struct NttTagScope {
  int prev;
  explicit NttTagScope(int tag);
  ~NttTagScope();
};
struct ProfScope {
  int slot = -1;
  cudaStream_t st;
  ProfScope(int cls, cudaStream_t s, double bytes = 0, double modmuls = 0);
  ~ProfScope();
};

// --- launchers (stream-ordered; throw HegpuError on failure) ----------------
struct NttEpilogue {
  bool enabled = false;  // forward: eout = (other - y) * c[limb]
  uint64_t c[kMaxPrimes];
  uint64_t csh[kMaxPrimes];
  // seg.eacc == 2: eout = ein * s[limb] + (other - y) * c[limb]
  uint64_t s[kMaxPrimes];
  uint64_t ssh[kMaxPrimes];
  bool post = false;     // inverse: final stage scales by fin_s / fin_d (Shoup pairs)
  ulonglong2 fin_s[kMaxPrimes];
  ulonglong2 fin_d[kMaxPrimes];
};

// NTT over a set of segments.  For the forward transform with an epilogue,
// seg.eout receives (seg.other - NTT(x)) * c[limb] and seg.out is scratch.
// device tables of the NTT kernels (idempotent; called at ring creation so it
// never runs inside a stream capture)
void ensure_tw_slots();
// fp_mask: bit p set when prime p takes the FP64 path (PrimeConst::twf);
// nullptr launches both arithmetic variants
void launch_ntt(const PrimeConst* dpc, const uint64_t* dtw, int log_n, bool inverse,
                SegSet& S, const NttEpilogue* epi, cudaStream_t st,
                const uint64_t* fp_mask = nullptr);

struct EwArgs {
  int op;
  const uint64_t* a;
  int64_t as;
  const uint64_t* b;
  int64_t bs;
  uint64_t* o;
  int64_t os;
  int n_polys, k;
  const int32_t* primes;
  const uint64_t* consts;  // host, k entries
};
void launch_elementwise(const PrimeConst* dpc, const std::vector<uint64_t>& hq, int log_n,
                        const EwArgs& A, cudaStream_t st);

void launch_lift_signed(const PrimeConst* dpc, int log_n, const int64_t* src, int64_t ss,
                        uint64_t* out, int64_t os, int n_polys, int k, const int32_t* primes,
                        cudaStream_t st);
void launch_lift_centered(const PrimeConst* dpc, int log_n, const uint64_t* src, int64_t ss,
                          uint64_t src_q, uint64_t* out, int64_t os, int n_polys, int k,
                          const int32_t* primes, cudaStream_t st);

struct ConvJob {
  const uint64_t* src;
  int64_t src_stride;
  uint64_t* dst;
  int64_t dst_stride;
  int n_src, n_dst;
  const uint64_t* inv;     // [n_src] natural
  const uint64_t* inv_sh;  // [n_src]
  const uint64_t* punc;    // [n_src] rows, row stride punc_ld, Montgomery form
  int punc_ld;
};
struct ConvParams {
  int n_jobs;
  int n_polys;
  int log_n;
  const PrimeConst* pc;
  ConvJob job[kMaxSeg];
  uint8_t src_sel[kMaxSeg][kMaxPrimes];
  uint8_t dst_sel[kMaxSeg][kMaxPrimes];
};
void launch_conv(ConvParams& P, cudaStream_t st);

struct TensorParams {
  const uint64_t *a0, *a1, *b0, *b1;
  uint64_t *d0, *d1, *d2;
  int64_t as, bs, ds;
  int amod;  // operand a of poly p is a[(p % amod) * as] (periodic broadcast)
  int k, log_n;
  int rows;  // n_polys * k (set by launch_tensor): the last grid.z slice may overhang
  const PrimeConst* pc;
};

struct EncParams {
  const uint64_t *v, *e0, *e1, *m, *pb, *pa;
  uint64_t *c0, *c1;
  int log_n;
  const PrimeConst* pc;
};

constexpr int kMaxDigits = 16;
struct IpParams {
  const uint64_t* d;  // eval-form input, (level+1) limbs per poly
  int64_t ds;
  const uint64_t* ext;  // [b][j][row][N] converted rows (compact per digit)
  int64_t ext_sb, ext_sj;
  const uint64_t* kb[kMaxDigits];
  const uint64_t* ka[kMaxDigits];
  uint64_t* acc;  // [b][2][n_ext][N]
  int64_t acc_sb;
  int accumulate;  // add into acc instead of overwriting (lazy ModDown)
  int level, alpha, beta, n_ext, n_chain, key_sp_row0, n_batch, log_n;
  const PrimeConst* pc;
};

// Key inner products of several rotations of hoisted digits in ONE launch:
// for rotation r, the digits are read through X -> X^gal[r] (eval-form
// gather, fused: no permuted copy is written).  Sources of rotation r:
// d + r*d_sr (own-digit rows, level+1 limbs per batch element, stride ds)
// and ext + r*ext_sr (converted rows).  sum_mode: all rotations accumulate
// into acc; otherwise rotation r writes acc + r*acc_sr.
constexpr int kMaxRot = 16;
constexpr int kMaxRotDigits = 8;
struct IpRotParams {
  const uint64_t* d;
  int64_t ds, d_sr;
  const uint64_t* ext;
  int64_t ext_sb, ext_sj, ext_sr;
  const uint64_t* kb[kMaxRot][kMaxRotDigits];
  const uint64_t* ka[kMaxRot][kMaxRotDigits];
  uint32_t gal[kMaxRot];
  int n_rot, sum_mode, accumulate;
  uint64_t* acc;
  int64_t acc_sb, acc_sr;
  int level, alpha, beta, n_ext, n_chain, key_sp_row0, n_batch, log_n;
  const PrimeConst* pc;
  // optional (separate mode): the b part of rows <= level also gets
  // P * sigma_r(c0) (double-hoisted rotations output P-scaled extended-basis
  // ciphertexts); c0 of batch element b at c0 + b*c0s
  const uint64_t* c0;
  int64_t c0s;
  uint64_t pm[kMaxPrimes], pm_sh[kMaxPrimes];  // P mod q_r, Shoup
};
void launch_ks_ip_rot(IpRotParams& P, cudaStream_t st);
// TMA-staged variant (ks_tma.cu); false when it does not apply
bool launch_ks_ip_rot_tma(const IpRotParams& P, cudaStream_t st);
// out[b] = base[b] + sum_r sigma_r(in[b] + r*in_sr) (eval form, k limbs;
// base = the unpermuted in when null).  Limbs >= kq are special primes
// n_chain + (limb - kq) (extended-basis operands); kq < 0: all chain.
void launch_auto_sum(const PrimeConst* dpc, int log_n, const uint32_t* gal, int n_rot,
                     const uint64_t* in, int64_t is, const uint64_t* base, int64_t bs,
                     uint64_t* out, int64_t os, int n_polys, int k, cudaStream_t st,
                     int64_t in_sr = 0, int kq = -1, int n_chain = 0);

void launch_automorphism(const PrimeConst* dpc, int log_n, bool eval_form, uint64_t g,
                         const uint64_t* in, int64_t is, uint64_t* out, int64_t os, int n_polys,
                         int k, const int32_t* primes, cudaStream_t st);
void launch_tensor(const PrimeConst* dpc, int log_n, const TensorParams& T0, int n_polys,
                   cudaStream_t st);
void launch_encrypt(const PrimeConst* dpc, int log_n, const EncParams& E0, int k,
                    cudaStream_t st);
void launch_diag_mac(const PrimeConst* dpc, int log_n, const uint64_t* const* ct,
                     int64_t ct_c1_off, int64_t ct_bstride, const uint64_t* const* pt,
                     int n_terms, int n_batch, uint64_t* out, int64_t out_c1_off,
                     int64_t out_bstride, int k, int accumulate, cudaStream_t st);
void launch_ks_ip(IpParams& P, cudaStream_t st);
double bench_modmul_peak(int iters);
double bench_fp_modmul_peak(int iters);
void launch_bsgs(const PrimeConst* dpc, int log_n, const uint64_t* const* babies, int n_terms,
                 int64_t c1_off, int64_t bstride, int n_batch, const uint64_t* pt_base,
                 int64_t pt_stride, int pt_log_run, const int32_t* pt_idx, int n_giants,
                 uint64_t* out, int64_t out_gstride, int k, cudaStream_t st, int kq,
                 int n_chain);

// encode.cu: full-slot bootstrap diagonals -> rounded integer coefficients
void launch_encode_diags(Ring& R, int kind, int half, double fold, double scale, int n_diags,
                         const int32_t* d, const int32_t* g0, const uint8_t* conj,
                         double2* scratch, int64_t* out, cudaStream_t st);
bool encode_overflow_check(Ring& R);

// rng.cu: numpy-compatible PCG64 bounded uniform draws; returns draws consumed
void sample_encrypt(int64_t* out, int n, uint64_t seed, double sigma, cudaStream_t st);
long long pcg64_uniform_fill(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                             uint64_t inc_lo, const uint64_t* bounds, int k, int n,
                             uint64_t* out, int64_t out_stride, cudaStream_t st);

}  // namespace hegpu
