// Ring context, fused CKKS operations (key switch, rescale, ModRaise,
// encryption) and the C ABI of libhegpu.
#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "ring.cuh"

namespace hegpu {

thread_local std::string g_last_error;
void set_error(const std::string& m) { g_last_error = m; }

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    throw HegpuError{HEGPU_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e)};
  }
}

// --- launch accounting / profiling ------------------------------------------
static std::atomic<long long> g_launches{0};
static std::atomic<bool> g_prof_on{false};
static std::mutex g_prof_mu;
static thread_local int g_ntt_tag = NTT_TAG_OTHER;
NttTagScope::NttTagScope(int tag) : prev(g_ntt_tag) { g_ntt_tag = tag; }
NttTagScope::~NttTagScope() { g_ntt_tag = prev; }

struct ProfRec {
  int cls, sub;
  double bytes, modmuls;
  cudaEvent_t a, b;
};
static std::vector<ProfRec> g_prof;

ProfScope::ProfScope(int cls, cudaStream_t s, double bytes, double modmuls) : st(s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (!g_prof_on.load(std::memory_order_relaxed)) return;
  ProfRec r;
  r.cls = cls;
  r.sub = cls == PROF_NTT ? g_ntt_tag : 0;
  r.bytes = bytes;
  r.modmuls = modmuls;
  cudaEventCreate(&r.a);
  cudaEventCreate(&r.b);
  cudaEventRecord(r.a, st);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  slot = (int)g_prof.size();
  g_prof.push_back(r);
}
ProfScope::~ProfScope() {
  if (slot < 0) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  cudaEventRecord(g_prof[slot].b, st);
}

// Stream-ordered scratch from the device's default memory pool (cached: the
// pool's release threshold is raised at ring creation).
// Scratch memory: stream-ordered, from the host's allocator when one is
// registered (hegpu_set_allocator: the Python layer registers torch's caching
// allocator, so tensors and scratch share ONE pool and neither strands memory
// the other needs), else the driver's stream-ordered pool (cudaMallocAsync).
static hegpu_alloc_fn g_alloc = nullptr;
static hegpu_free_fn g_free = nullptr;

struct Scratch {
  void* p = nullptr;
  size_t n = 0;
  cudaStream_t st;
  Scratch(size_t bytes, cudaStream_t s) : n(bytes), st(s) {
    if (!bytes) return;
    if (g_alloc) {
      p = g_alloc(bytes, static_cast<void*>(s));
      if (!p) throw HegpuError{HEGPU_E_NOMEM, "scratch alloc: out of memory (host allocator)"};
    } else {
      check_cuda(cudaMallocAsync(&p, bytes, s), "scratch alloc");
    }
  }
  ~Scratch() {
    if (!p) return;
    if (g_alloc && g_free)
      g_free(p, n, static_cast<void*>(st));
    else if (!g_alloc)
      cudaFreeAsync(p, st);
  }
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  uint64_t* u64() const { return static_cast<uint64_t*>(p); }
};

// --- host number theory (ring.py:60-128, 217-238) ---------------------------

static bool is_prime_u64(uint64_t n) {
  if (n < 2) return false;
  static const uint64_t small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  for (uint64_t p : small)
    if (n % p == 0) return n == p;
  uint64_t d = n - 1;
  int s = 0;
  while ((d & 1) == 0) {
    d >>= 1;
    ++s;
  }
  for (uint64_t a : small) {
    uint64_t x = h_powmod(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int r = 1; r < s; ++r) {
      x = h_mulmod(x, x, n);
      if (x == n - 1) {
        comp = false;
        break;
      }
    }
    if (comp) return false;
  }
  return true;
}

// First base in [2, 10^4) whose (q-1)/2N power has order exactly 2N
// (find_primitive_2n_root, ring.py:69-78).
static uint64_t find_psi(uint64_t q, uint64_t two_n) {
  if ((q - 1) % two_n != 0) throw HegpuError{HEGPU_E_ARG, "modulus is not NTT-friendly"};
  const uint64_t e = (q - 1) / two_n;
  for (uint64_t base = 2; base < 10000; ++base) {
    const uint64_t cand = h_powmod(base, e, q);
    if (h_powmod(cand, two_n / 2, q) == q - 1) return cand;
  }
  throw HegpuError{HEGPU_E_ARG, "no primitive root found"};
}

static uint64_t neg_inv_2_64(uint64_t q) {
  uint64_t x = q;  // correct to 3 bits for odd q
  for (int i = 0; i < 5; ++i) x *= 2 - q * x;
  return 0 - x;
}

static inline uint32_t brev(uint32_t x, int bits) {
  uint32_t r = 0;
  for (int b = 0; b < bits; ++b) r |= ((x >> b) & 1u) << (bits - 1 - b);
  return r;
}

PrimeConst make_prime_const(uint64_t q, int log_n, uint64_t ipsi1) {
  PrimeConst c;
  c.q = q;
  c.qinv_neg = neg_inv_2_64(q);
  const uint64_t r = h_rmod(q);
  c.r2 = h_mulmod(r, r, q);
  c.bar = h_shoup(1, q);
  c.ninv = h_inv((uint64_t)1 << log_n, q);
  c.ninv_sh = h_shoup(c.ninv, q);
  c.ilast = h_mulmod(ipsi1, c.ninv, q);
  c.ilast_sh = h_shoup(c.ilast, q);
  c.twf = nullptr;
  c.pad_ = 0;
  return c;
}

// FP64 twiddles (w, w/q) of every prime below 2^kFpMaxBits, built from the
// integer Shoup tables (layout [prime][4N]: forward pairs, inverse pairs).
// Sets pc[i].twf to the prime's device table; returns the allocation (or
// nullptr when no prime qualifies or HEGPU_NTT_FP=0).
static void* attach_fp_twiddles(std::vector<PrimeConst>& pc, const uint64_t* tw, int n) {
  const char* env = getenv("HEGPU_NTT_FP");
  if (env && atoi(env) == 0) return nullptr;
  std::vector<int> fp;
  for (int i = 0; i < (int)pc.size(); ++i)
    if (pc[i].q < (1ull << kFpMaxBits)) fp.push_back(i);
  if (fp.empty()) return nullptr;
  std::vector<double> h((size_t)fp.size() * 4 * n);
  for (size_t f = 0; f < fp.size(); ++f) {
    const int i = fp[f];
    const double qd = (double)pc[i].q;
    const uint64_t* t = tw + (size_t)i * 4 * n;
    double* o = h.data() + f * 4 * n;
    for (int j = 0; j < 2 * n; ++j) {  // forward then inverse
      const double w = (double)t[2 * j];
      o[2 * j] = w;
      o[2 * j + 1] = w / qd;
    }
  }
  void* d = nullptr;
  check_cuda(cudaMalloc(&d, h.size() * 8), "alloc fp twiddles");
  check_cuda(cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice), "copy fp twiddles");
  for (size_t f = 0; f < fp.size(); ++f)
    pc[fp[f]].twf = reinterpret_cast<const double2*>(static_cast<double*>(d) + f * 4 * n);
  return d;
}

// Twiddles of one prime, natural form, bit-reversed order, as interleaved
// Shoup pairs: [psi_rev[i], shoup(psi_rev[i])] for i < N, then the same for
// ipsi_rev -- one 16-byte load per butterfly.
static void make_twiddles(uint64_t q, int log_n, uint64_t* out4n) {
  const uint64_t n = 1ull << log_n;
  const uint64_t psi = find_psi(q, 2 * n);
  const uint64_t ipsi = h_inv(psi, q);
  std::vector<uint64_t> pw(n), ipw(n);
  uint64_t x = 1, ix = 1;
  for (uint64_t i = 0; i < n; ++i) {
    pw[i] = x;
    ipw[i] = ix;
    x = h_mulmod(x, psi, q);
    ix = h_mulmod(ix, ipsi, q);
  }
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t rv = brev((uint32_t)i, log_n);
    out4n[2 * i] = pw[rv];
    out4n[2 * i + 1] = h_shoup(pw[rv], q);
    out4n[2 * n + 2 * i] = ipw[rv];
    out4n[2 * n + 2 * i + 1] = h_shoup(ipw[rv], q);
  }
}

Ring::~Ring() {
  for (auto& kv : ks)
    if (kv.second->dmem) cudaFree(kv.second->dmem);
  if (dpc) cudaFree(dpc);
  if (dtw) cudaFree(dtw);
  if (dtwf) cudaFree(dtwf);
  if (enc.dlog) cudaFree(enc.dlog);
  if (enc.pow5) cudaFree(enc.pow5);
  if (enc.overflow) cudaFree(enc.overflow);
  if (enc.eroot) cudaFree(enc.eroot);
}

static uint64_t prod_mod(const std::vector<uint64_t>& ps, int skip, uint64_t m) {
  uint64_t r = 1 % m;
  for (int i = 0; i < (int)ps.size(); ++i)
    if (i != skip) r = h_mulmod(r, ps[i] % m, m);
  return r;
}

const KsLevel& Ring::ks_level(int level, int alpha) {
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(level, alpha);
  auto it = ks.find(key);
  if (it != ks.end()) return *it->second;
  if (level < 0 || level >= n_chain) throw HegpuError{HEGPU_E_ARG, "level out of range"};
  if (alpha < 1) throw HegpuError{HEGPU_E_ARG, "digit size must be >= 1"};
  auto L = std::make_unique<KsLevel>();
  const int k = level + 1, K = n_special, n_ext = k + K;
  const int beta = (k + alpha - 1) / alpha;
  L->level = level;
  L->alpha = alpha;
  L->beta = beta;
  L->n_ext = n_ext;
  L->K = K;
  std::vector<uint64_t> mu_inv(k), mu_inv_sh(k), mu_punc((size_t)k * n_ext, 0);
  L->dst_prime_of_digit.assign((size_t)beta * n_ext, -1);
  for (int j = 0; j < beta; ++j) {
    const int g0 = j * alpha, g1 = std::min(g0 + alpha, k);
    std::vector<uint64_t> grp(primes.begin() + g0, primes.begin() + g1);
    std::vector<int> dst;
    for (int r = 0; r < n_ext; ++r) {
      if (r >= g0 && r < g1) continue;
      dst.push_back(r <= level ? r : n_chain + (r - level - 1));
    }
    for (int t = 0; t < (int)dst.size(); ++t) L->dst_prime_of_digit[(size_t)j * n_ext + t] = dst[t];
    for (int i = 0; i < (int)grp.size(); ++i) {
      const uint64_t qi = grp[i];
      const uint64_t inv = h_inv(prod_mod(grp, i, qi), qi);
      mu_inv[g0 + i] = inv;
      mu_inv_sh[g0 + i] = h_shoup(inv, qi);
      for (int t = 0; t < (int)dst.size(); ++t) {
        const uint64_t p = primes[dst[t]];
        mu_punc[(size_t)(g0 + i) * n_ext + t] = h_mulmod(prod_mod(grp, i, p), h_rmod(p), p);
      }
    }
  }
  std::vector<uint64_t> sp(primes.begin() + n_chain, primes.end());
  std::vector<uint64_t> md_inv(K), md_inv_sh(K), md_punc((size_t)K * k);
  for (int i = 0; i < K; ++i) {
    const uint64_t si = sp[i];
    md_inv[i] = h_inv(prod_mod(sp, i, si), si);
    md_inv_sh[i] = h_shoup(md_inv[i], si);
    for (int t = 0; t < k; ++t) {
      const uint64_t q = primes[t];
      md_punc[(size_t)i * k + t] = h_mulmod(prod_mod(sp, i, q), h_rmod(q), q);
    }
  }
  auto fin = [&](int p, uint64_t sc, std::vector<ulonglong2>& fs, std::vector<ulonglong2>& fd) {
    const uint64_t q = primes[p];
    const uint64_t a = h_mulmod(hpc[p].ninv, sc, q), b = h_mulmod(hpc[p].ilast, sc, q);
    fs.push_back(make_ulonglong2(a, h_shoup(a, q)));
    fd.push_back(make_ulonglong2(b, h_shoup(b, q)));
  };
  for (int i = 0; i < k; ++i) fin(i, mu_inv[i], L->mu_fin_s, L->mu_fin_d);
  for (int i = 0; i < K; ++i) fin(n_chain + i, md_inv[i], L->md_fin_s, L->md_fin_d);
  L->pinv.resize(k);
  L->pinv_sh.resize(k);
  for (int t = 0; t < k; ++t) {
    const uint64_t q = primes[t];
    L->pinv[t] = h_inv(prod_mod(sp, -1, q), q);
    L->pinv_sh[t] = h_shoup(L->pinv[t], q);
  }
  // ModDown fused with the rescale: D = q_level * P, sources (q_level, specials)
  std::vector<uint64_t> mdr_punc, mdr_negd;
  std::vector<float> mdr_fw;
  std::vector<int32_t> mdr_fs;
  if (level >= 1) {
    std::vector<uint64_t> D{primes[level]};
    std::vector<int> dp{level};
    for (int i = 0; i < K; ++i) {
      D.push_back(sp[i]);
      dp.push_back(n_chain + i);
    }
    mdr_punc.resize((size_t)(K + 1) * level);
    for (int i = 0; i <= K; ++i) {
      fin(dp[i], h_inv(prod_mod(D, i, D[i]), D[i]), L->mdr_fin_s, L->mdr_fin_d);
      for (int t = 0; t < level; ++t) {
        const uint64_t q = primes[t];
        mdr_punc[(size_t)i * level + t] = h_mulmod(prod_mod(D, i, q), h_rmod(q), q);
      }
    }
    for (int t = 0; t < level; ++t) {
      const uint64_t q = primes[t];
      L->dinv.push_back(h_inv(prod_mod(D, -1, q), q));
      L->dinv_sh.push_back(h_shoup(L->dinv.back(), q));
      L->qlinv.push_back(h_inv(primes[level] % q, q));
      L->qlinv_sh.push_back(h_shoup(L->qlinv.back(), q));
    }
    L->p_mod_ql = prod_mod(sp, -1, primes[level]);
    for (int i = 0; i <= K; ++i) {
      int bits = 0;
      while (bits < 64 && (D[i] >> bits)) ++bits;
      const int sh = bits > 32 ? bits - 32 : 0;
      mdr_fs.push_back(sh);
      mdr_fw.push_back(static_cast<float>(std::ldexp(1.0, sh) / static_cast<double>(D[i])));
    }
    for (int t = 0; t < level; ++t) {
      const uint64_t q = primes[t];
      mdr_negd.push_back(h_mulmod((q - prod_mod(D, -1, q)) % q, h_rmod(q), q));
    }
  }
  const size_t total = mu_inv.size() * 2 + mu_punc.size() + md_inv.size() * 2 + md_punc.size() +
                       mdr_punc.size() + mdr_negd.size() + mdr_fw.size() + mdr_fs.size();
  std::vector<uint64_t> host;
  host.reserve(total);
  auto append = [&](const std::vector<uint64_t>& v) {
    const size_t off = host.size();
    host.insert(host.end(), v.begin(), v.end());
    return off;
  };
  const size_t o1 = append(mu_inv), o2 = append(mu_inv_sh), o3 = append(mu_punc);
  const size_t o4 = append(md_inv), o5 = append(md_inv_sh), o6 = append(md_punc);
  const size_t o7 = append(mdr_punc), o8 = append(mdr_negd);
  // fp32 weights and int32 shifts, one 64-bit word each
  std::vector<uint64_t> fw64(mdr_fw.size()), fs64(mdr_fs.size());
  for (size_t i = 0; i < mdr_fw.size(); ++i) {
    uint32_t bits;
    std::memcpy(&bits, &mdr_fw[i], 4);
    fw64[i] = bits;
    fs64[i] = static_cast<uint32_t>(mdr_fs[i]);
  }
  const size_t o9 = append(fw64), o10 = append(fs64);
  check_cuda(cudaMalloc(&L->dmem, std::max<size_t>(total, 1) * 8), "ks const alloc");
  check_cuda(cudaMemcpy(L->dmem, host.data(), total * 8, cudaMemcpyHostToDevice), "ks const copy");
  L->mu_inv = L->dmem + o1;
  L->mu_inv_sh = L->dmem + o2;
  L->mu_punc = L->dmem + o3;
  L->md_inv = L->dmem + o4;
  L->md_inv_sh = L->dmem + o5;
  L->md_punc = L->dmem + o6;
  L->mdr_punc = L->dmem + o7;
  L->mdr_negd = L->dmem + o8;
  L->mdr_fw_words = L->dmem + o9;
  L->mdr_fs_words = L->dmem + o10;
  const KsLevel& ref = *L;
  ks[key] = std::move(L);
  return ref;
}

const std::pair<std::vector<uint64_t>, std::vector<uint64_t>>& Ring::rescale_consts(int level) {
  std::lock_guard<std::mutex> lk(mu);
  auto it = rescale.find(level);
  if (it != rescale.end()) return it->second;
  std::vector<uint64_t> c(level), csh(level);
  const uint64_t ql = primes[level];
  for (int i = 0; i < level; ++i) {
    c[i] = h_inv(ql % primes[i], primes[i]);
    csh[i] = h_shoup(c[i], primes[i]);
  }
  return rescale[level] = std::make_pair(c, csh);
}

static Ring* create_ring(int log_n, const uint64_t* chain, int n_chain, const uint64_t* special,
                         int n_special) {
  if (log_n < 4 || log_n > 17) throw HegpuError{HEGPU_E_ARG, "ring degree must be 2^4..2^17"};
  if (n_chain < 1 || n_special < 0 || n_chain + n_special > kMaxPrimes)
    throw HegpuError{HEGPU_E_ARG, "bad prime counts"};
  auto R = std::make_unique<Ring>();
  R->log_n = log_n;
  R->n = 1 << log_n;
  R->n_chain = n_chain;
  R->n_special = n_special;
  R->n_primes = n_chain + n_special;
  R->primes.assign(chain, chain + n_chain);
  R->primes.insert(R->primes.end(), special, special + n_special);
  for (size_t i = 0; i < R->primes.size(); ++i) {
    const uint64_t q = R->primes[i];
    if (q >= (1ull << 62)) throw HegpuError{HEGPU_E_ARG, "modulus >= 2^62"};
    if (q % (2ull * R->n) != 1) throw HegpuError{HEGPU_E_ARG, "modulus != 1 mod 2N"};
    if (!is_prime_u64(q)) throw HegpuError{HEGPU_E_ARG, "modulus is not prime"};
    for (size_t j = 0; j < i; ++j)
      if (R->primes[j] == q) throw HegpuError{HEGPU_E_ARG, "duplicate modulus"};
  }
  check_cuda(cudaGetDevice(&R->device), "get device");
  ensure_tw_slots();
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, R->device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  const size_t n = R->n;
  std::vector<uint64_t> tw(R->primes.size() * 4 * n);
  R->hpc.resize(R->primes.size());
  for (size_t i = 0; i < R->primes.size(); ++i) {
    uint64_t* t = tw.data() + i * 4 * n;
    make_twiddles(R->primes[i], log_n, t);
    R->hpc[i] = make_prime_const(R->primes[i], log_n, t[2 * n + 2]);  // ipsi_rev[1]
  }
  R->dtwf = attach_fp_twiddles(R->hpc, tw.data(), (int)n);
  for (size_t i = 0; i < R->hpc.size(); ++i)
    if (R->hpc[i].twf) R->fp_mask |= 1ull << i;
  check_cuda(cudaMalloc(&R->dpc, R->hpc.size() * sizeof(PrimeConst)), "alloc consts");
  check_cuda(cudaMemcpy(R->dpc, R->hpc.data(), R->hpc.size() * sizeof(PrimeConst),
                        cudaMemcpyHostToDevice),
             "copy consts");
  check_cuda(cudaMalloc(&R->dtw, tw.size() * 8), "alloc twiddles");
  check_cuda(cudaMemcpy(R->dtw, tw.data(), tw.size() * 8, cudaMemcpyHostToDevice),
             "copy twiddles");
  return R.release();
}

// --- helpers ----------------------------------------------------------------

static void add_seg(SegSet& S, const uint64_t* in, int64_t is, uint64_t* out, int64_t os,
                    int n_polys, int k, const int32_t* primes) {
  if (S.n_seg >= kMaxSeg) throw HegpuError{HEGPU_E_ARG, "too many segments"};
  if (k > kMaxPrimes) throw HegpuError{HEGPU_E_ARG, "too many limbs"};
  Seg& g = S.seg[S.n_seg];
  g.in = in;
  g.out = out;
  g.in_stride = is;
  g.out_stride = os;
  g.other = nullptr;
  g.eout = nullptr;
  g.csrc = nullptr;
  g.csrc_stride = 0;
  g.cpunc = nullptr;
  g.c_nsrc = 0;
  g.cpunc_ld = 0;
  g.eacc = 0;
  g.ein = nullptr;
  g.ein_stride = 0;
  g.cmode = 0;
  g.c_fp_src = 0;
  g.csrc_q = 0;
  g.cnegd = nullptr;
  g.cfw = nullptr;
  g.cfs = nullptr;
  g.other_stride = 0;
  g.eout_stride = 0;
  g.n_polys = n_polys;
  g.k = k;
  g.row_start = S.n_rows;
  for (int l = 0; l < k; ++l) {
    if (primes[l] < 0 || primes[l] >= kMaxPrimes) throw HegpuError{HEGPU_E_ARG, "bad prime index"};
    S.sel[S.n_seg][l] = (uint8_t)primes[l];
  }
  S.n_rows += n_polys * k;
  S.n_seg++;
}

static std::vector<int32_t> range_primes(int first, int count) {
  std::vector<int32_t> v(count);
  for (int i = 0; i < count; ++i) v[i] = first + i;
  return v;
}

static void ntt_simple(Ring& R, bool inverse, const uint64_t* in, int64_t is, uint64_t* out,
                       int64_t os, int n_polys, int k, const int32_t* primes, cudaStream_t st) {
  SegSet S;
  S.n_seg = 0;
  S.n_rows = 0;
  add_seg(S, in, is, out, os, n_polys, k, primes);
  launch_ntt(R.dpc, R.dtw, R.log_n, inverse, S, nullptr, st, &R.fp_mask);
}

// --- hybrid key switching (keys.py:278-339) --------------------------------

// ModUp (keys.py:290-313): d (B eval-form polys of level+1 limbs) -> the
// converted rows of every digit, NTT'd, in the compact layout
// ext[b][j][t][N] (t < n_ext - |group j|).  dcoeff: B*(level+1)*N scratch.
static void ks_modup(Ring& R, const KsLevel& L, const uint64_t* d, int64_t ds, int B,
                     uint64_t* dcoeff, uint64_t* ext, cudaStream_t st) {
  NttTagScope tag_(NTT_TAG_MODUP);
  const int level = L.level, alpha = L.alpha;
  const int k = level + 1, n_ext = L.n_ext, beta = L.beta;
  const size_t N = R.n;
  const std::vector<int32_t> chain = range_primes(0, k);
  if (R.log_n >= 12) {
    // fused path: INTT(d) scaled by (Q_j/q_i)^-1 gives hat_i directly; each
    // digit's conversion runs inside the forward NTT's first pass.
    SegSet S0;
    S0.n_seg = 0;
    S0.n_rows = 0;
    add_seg(S0, d, ds, dcoeff, (int64_t)k * N, B, k, chain.data());
    NttEpilogue E0;
    E0.post = true;
    for (int i = 0; i < k; ++i) {
      E0.fin_s[i] = L.mu_fin_s[i];
      E0.fin_d[i] = L.mu_fin_d[i];
    }
    launch_ntt(R.dpc, R.dtw, R.log_n, true, S0, &E0, st, &R.fp_mask);
    for (int j0 = 0; j0 < beta; j0 += kMaxSeg) {
      const int jn = std::min(kMaxSeg, beta - j0);
      SegSet S;
      S.n_seg = 0;
      S.n_rows = 0;
      for (int jj = 0; jj < jn; ++jj) {
        const int j = j0 + jj;
        const int g0 = j * alpha, g1 = std::min(g0 + alpha, k), g = g1 - g0;
        const int n_dst = n_ext - g;
        if (n_dst <= 0) continue;
        std::vector<int32_t> dsel(n_dst);
        for (int t = 0; t < n_dst; ++t) dsel[t] = L.dst_prime_of_digit[(size_t)j * n_ext + t];
        uint64_t* dst = ext + (size_t)j * n_ext * N;
        const int64_t dsb = (int64_t)beta * n_ext * N;
        add_seg(S, nullptr, 0, dst, dsb, B, n_dst, dsel.data());
        Seg& sg = S.seg[S.n_seg - 1];
        sg.csrc = dcoeff + (size_t)g0 * N;
        sg.csrc_stride = (int64_t)k * N;
        sg.cpunc = L.mu_punc + (size_t)g0 * n_ext;
        sg.c_nsrc = g;
        sg.cpunc_ld = n_ext;
        sg.c_fp_src = 1;
        for (int i = g0; i < g1; ++i) sg.c_fp_src &= R.hpc[i].twf != nullptr ? 1 : 0;
      }
      launch_ntt(R.dpc, R.dtw, R.log_n, false, S, nullptr, st, &R.fp_mask);
    }
    return;
  }
  // 1. d -> coefficient form
  ntt_simple(R, true, d, ds, dcoeff, (int64_t)k * N, B, k, chain.data(), st);
  // 2. ModUp basis conversion of every digit, 3. NTT of the converted rows
  for (int j0 = 0; j0 < beta; j0 += kMaxSeg) {
    const int jn = std::min(kMaxSeg, beta - j0);
    ConvParams C;
    C.n_jobs = jn;
    C.n_polys = B;
    C.log_n = R.log_n;
    C.pc = R.dpc;
    SegSet S;
    S.n_seg = 0;
    S.n_rows = 0;
    for (int jj = 0; jj < jn; ++jj) {
      const int j = j0 + jj;
      const int g0 = j * alpha, g1 = std::min(g0 + alpha, k), g = g1 - g0;
      const int n_dst = n_ext - g;
      ConvJob& J = C.job[jj];
      J.src = dcoeff + (size_t)g0 * N;
      J.src_stride = (int64_t)k * N;
      J.dst = ext + (size_t)j * n_ext * N;
      J.dst_stride = (int64_t)beta * n_ext * N;
      J.n_src = g;
      J.n_dst = n_dst;
      J.inv = L.mu_inv + g0;
      J.inv_sh = L.mu_inv_sh + g0;
      J.punc = L.mu_punc + (size_t)g0 * n_ext;
      J.punc_ld = n_ext;
      for (int i = 0; i < g; ++i) C.src_sel[jj][i] = (uint8_t)(g0 + i);
      std::vector<int32_t> dsel(n_dst);
      for (int t = 0; t < n_dst; ++t) {
        dsel[t] = L.dst_prime_of_digit[(size_t)j * n_ext + t];
        C.dst_sel[jj][t] = (uint8_t)dsel[t];
      }
      if (n_dst > 0)
        add_seg(S, J.dst, J.dst_stride, J.dst, J.dst_stride, B, n_dst, dsel.data());
    }
    launch_conv(C, st);
    launch_ntt(R.dpc, R.dtw, R.log_n, false, S, nullptr, st, &R.fp_mask);
  }
}

// Key inner product (keys.py:316-323): acc (+)= sum_j digit_j * key_j over
// the extended basis.  d / ext are the digit sources (own rows from d,
// converted rows from ext, compact layout).
static void ks_ip(Ring& R, const KsLevel& L, const uint64_t* d, int64_t ds, const uint64_t* ext,
                  int B, const uint64_t* const* key_b, const uint64_t* const* key_a,
                  uint64_t* acc, bool accumulate, cudaStream_t st) {
  const int level = L.level, alpha = L.alpha;
  const int n_ext = L.n_ext, beta = L.beta;
  const size_t N = R.n;
  // 4. inner product with the key digits
  IpParams P;
  P.d = d;
  P.ds = ds;
  P.ext = ext;
  P.ext_sb = (int64_t)beta * n_ext * N;
  P.ext_sj = (int64_t)n_ext * N;
  for (int j = 0; j < beta; ++j) {
    P.kb[j] = key_b[j];
    P.ka[j] = key_a[j];
  }
  P.acc = acc;
  P.acc_sb = (int64_t)2 * n_ext * N;
  P.level = level;
  P.alpha = alpha;
  P.beta = beta;
  P.n_ext = n_ext;
  P.n_chain = R.n_chain;
  P.key_sp_row0 = R.n_chain;
  P.n_batch = B;
  P.log_n = R.log_n;
  P.pc = R.dpc;
  P.accumulate = accumulate ? 1 : 0;
  launch_ks_ip(P, st);
}

// ModDown (keys.py:325-338) of acc [b][2][n_ext][N]: (b, a) = (acc - conv(P-part))
// * P^-1 written to (or with acc_b / acc_a added into) out_b / out_a.
static void ks_moddown(Ring& R, const KsLevel& L, uint64_t* acc, uint64_t* corr, int B,
                       uint64_t* out_b, int64_t os_b, uint64_t* out_a, int64_t os_a,
                       cudaStream_t st, bool acc_b, bool acc_a) {
  NttTagScope tag_(NTT_TAG_MODDOWN);
  const int level = L.level;
  const int k = level + 1, K = R.n_special, n_ext = L.n_ext;
  const size_t N = R.n;
  const size_t sz_corr = (size_t)B * 2 * k * N;
  const std::vector<int32_t> chain = range_primes(0, k);
  // 5. ModDown: INTT(specials), convert specials -> chain, NTT, (acc - corr) P^-1
  const bool fused = R.log_n >= 12 && K > 0;
  if (fused) {
    const std::vector<int32_t> sp = range_primes(R.n_chain, K);
    SegSet S0;
    S0.n_seg = 0;
    S0.n_rows = 0;
    add_seg(S0, acc + (size_t)k * N, (int64_t)n_ext * N, acc + (size_t)k * N, (int64_t)n_ext * N,
            2 * B, K, sp.data());
    NttEpilogue E0;
    E0.post = true;
    for (int i = 0; i < K; ++i) {
      E0.fin_s[i] = L.md_fin_s[i];
      E0.fin_d[i] = L.md_fin_d[i];
    }
    launch_ntt(R.dpc, R.dtw, R.log_n, true, S0, &E0, st, &R.fp_mask);
  } else if (K > 0) {
    const std::vector<int32_t> sp = range_primes(R.n_chain, K);
    ntt_simple(R, true, acc + (size_t)k * N, (int64_t)n_ext * N, acc + (size_t)k * N,
               (int64_t)n_ext * N, 2 * B, K, sp.data(), st);
    ConvParams C;
    C.n_jobs = 1;
    C.n_polys = 2 * B;
    C.log_n = R.log_n;
    C.pc = R.dpc;
    ConvJob& J = C.job[0];
    J.src = acc + (size_t)k * N;
    J.src_stride = (int64_t)n_ext * N;
    J.dst = corr;
    J.dst_stride = (int64_t)k * N;
    J.n_src = K;
    J.n_dst = k;
    J.inv = L.md_inv;
    J.inv_sh = L.md_inv_sh;
    J.punc = L.md_punc;
    J.punc_ld = k;
    for (int i = 0; i < K; ++i) C.src_sel[0][i] = (uint8_t)(R.n_chain + i);
    for (int t = 0; t < k; ++t) C.dst_sel[0][t] = (uint8_t)t;
    launch_conv(C, st);
  } else {
    check_cuda(cudaMemsetAsync(corr, 0, sz_corr * 8, st), "memset");
  }
  SegSet S;
  S.n_seg = 0;
  S.n_rows = 0;
  add_seg(S, corr, (int64_t)2 * k * N, corr, (int64_t)2 * k * N, B, k, chain.data());
  add_seg(S, corr + (size_t)k * N, (int64_t)2 * k * N, corr + (size_t)k * N, (int64_t)2 * k * N,
          B, k, chain.data());
  S.seg[0].other = acc;
  S.seg[0].other_stride = (int64_t)2 * n_ext * N;
  S.seg[0].eout = out_b;
  S.seg[0].eout_stride = os_b;
  S.seg[1].other = acc + (size_t)n_ext * N;
  S.seg[1].other_stride = (int64_t)2 * n_ext * N;
  S.seg[1].eout = out_a;
  S.seg[1].eout_stride = os_a;
  S.seg[0].eacc = acc_b ? 1 : 0;
  S.seg[1].eacc = acc_a ? 1 : 0;
  if (fused) {  // the specials -> chain conversion runs inside the NTT's first pass
    for (int g = 0; g < 2; ++g) {
      S.seg[g].csrc = acc + (size_t)g * n_ext * N + (size_t)k * N;
      S.seg[g].csrc_stride = (int64_t)2 * n_ext * N;
      S.seg[g].cpunc = L.md_punc;
      S.seg[g].c_nsrc = K;
      S.seg[g].cpunc_ld = k;
    }
  }
  NttEpilogue E;
  E.enabled = true;
  for (int t = 0; t < k; ++t) {
    E.c[t] = L.pinv[t];
    E.csh[t] = L.pinv_sh[t];
  }
  launch_ntt(R.dpc, R.dtw, R.log_n, false, S, &E, st, &R.fp_mask);
}


// ModDown of single polys in the extended basis (P-scaled, eval form):
// out = (in - conv(in_P)) * P^-1 over the chain limbs 0..level.  The special
// rows of `in` are overwritten (post-scaled INTT in place).  N >= 2^12.
static void ks_moddown_polys(Ring& R, const KsLevel& L, uint64_t* in, int64_t is, int n_polys,
                             uint64_t* out, int64_t os, uint64_t* corr, cudaStream_t st) {
  NttTagScope tag_(NTT_TAG_MODDOWN);
  const int k = L.level + 1, K = R.n_special;
  const size_t N = R.n;
  if (R.log_n < 12 || K == 0) throw HegpuError{HEGPU_E_ARG, "ModDown of polys needs N >= 2^12"};
  const std::vector<int32_t> sp = range_primes(R.n_chain, K);
  SegSet S0;
  S0.n_seg = 0;
  S0.n_rows = 0;
  add_seg(S0, in + (size_t)k * N, is, in + (size_t)k * N, is, n_polys, K, sp.data());
  NttEpilogue E0;
  E0.post = true;
  for (int i = 0; i < K; ++i) {
    E0.fin_s[i] = L.md_fin_s[i];
    E0.fin_d[i] = L.md_fin_d[i];
  }
  launch_ntt(R.dpc, R.dtw, R.log_n, true, S0, &E0, st, &R.fp_mask);
  const std::vector<int32_t> chain = range_primes(0, k);
  SegSet S;
  S.n_seg = 0;
  S.n_rows = 0;
  add_seg(S, corr, (int64_t)k * N, corr, (int64_t)k * N, n_polys, k, chain.data());
  Seg& sg = S.seg[0];
  sg.other = in;
  sg.other_stride = is;
  sg.eout = out;
  sg.eout_stride = os;
  sg.csrc = in + (size_t)k * N;
  sg.csrc_stride = is;
  sg.cpunc = L.md_punc;
  sg.c_nsrc = K;
  sg.cpunc_ld = k;
  NttEpilogue E;
  E.enabled = true;
  for (int t = 0; t < k; ++t) {
    E.c[t] = L.pinv[t];
    E.csh[t] = L.pinv_sh[t];
  }
  launch_ntt(R.dpc, R.dtw, R.log_n, false, S, &E, st, &R.fp_mask);
}

static void ks_ipdown(Ring& R, const KsLevel& L, const uint64_t* d, int64_t ds,
                      const uint64_t* ext, int B, const uint64_t* const* key_b,
                      const uint64_t* const* key_a, uint64_t* acc, uint64_t* corr,
                      uint64_t* out_b, int64_t os_b, uint64_t* out_a, int64_t os_a,
                      cudaStream_t st, bool acc_b = false, bool acc_a = false) {
  ks_ip(R, L, d, ds, ext, B, key_b, key_a, acc, false, st);
  ks_moddown(R, L, acc, corr, B, out_b, os_b, out_a, os_a, st, acc_b, acc_a);
}

static void ks_apply_impl(Ring& R, int level, int alpha, const uint64_t* d, int64_t ds, int B,
                          const uint64_t* const* key_b, const uint64_t* const* key_a,
                          int n_digits, uint64_t* out_b, uint64_t* out_a, int64_t os,
                          cudaStream_t st, bool acc_b = false, bool acc_a = false) {
  if (B <= 0) return;
  const KsLevel& L = R.ks_level(level, alpha);
  const int k = level + 1, n_ext = L.n_ext, beta = L.beta;
  const size_t N = R.n;
  if (n_digits < beta) throw HegpuError{HEGPU_E_ARG, "switching key has too few digits"};
  if (beta > kMaxDigits) throw HegpuError{HEGPU_E_ARG, "too many digits"};
  const size_t sz_dc = (size_t)B * k * N, sz_ext = (size_t)B * beta * n_ext * N;
  const size_t sz_acc = (size_t)B * 2 * n_ext * N, sz_corr = (size_t)B * 2 * k * N;
  Scratch ws((sz_dc + sz_ext + sz_acc + sz_corr) * 8, st);
  uint64_t* dcoeff = ws.u64();
  uint64_t* ext = dcoeff + sz_dc;
  uint64_t* acc = ext + sz_ext;
  uint64_t* corr = acc + sz_acc;
  ks_modup(R, L, d, ds, B, dcoeff, ext, st);
  ks_ipdown(R, L, d, ds, ext, B, key_b, key_a, acc, corr, out_b, os, out_a, os, st, acc_b,
            acc_a);
}

static void rescale_impl(Ring& R, int level, const uint64_t* in, int64_t is, uint64_t* out,
                         int64_t os, int P, cudaStream_t st);

// ModDown fused with the following rescale (mult = tensor, relinearize,
// rescale): out = (P * in + acc) / (q_level * P) at level - 1, for both
// components, with ONE approximate basis conversion from D = {q_level} + P
// (keys.py:325-338 followed by ops.py:160-178 in the reference, which
// converts from P and then rounds by q_level separately: same message, the
// rounding error differs by at most the conversion's).  in: B (c0, c1) pairs
// at level (c0 at in + b*is, c1 at + in_c1); out at level - 1 likewise.
// `in` is clobbered on the unfused (N < 2^12) path.
static void ks_moddown_rescale(Ring& R, const KsLevel& L, uint64_t* acc, uint64_t* corr, int B,
                               uint64_t* in, int64_t is, int64_t in_c1, uint64_t* out,
                               int64_t os, int64_t out_c1, cudaStream_t st) {
  const int level = L.level, K = R.n_special, n_ext = L.n_ext;
  const size_t N = R.n;
  if (level < 1) throw HegpuError{HEGPU_E_ARG, "rescale at level 0"};
  if (!in && (R.log_n < 12 || K == 0))
    throw HegpuError{HEGPU_E_ARG, "extended-basis ModDown-rescale needs N >= 2^12"};
  if (R.log_n < 12 || K == 0) {
    ks_moddown(R, L, acc, corr, B, in, is, in + in_c1, is, st, true, true);
    rescale_impl(R, level, in, is, out, os, B, st);
    rescale_impl(R, level, in + in_c1, is, out + out_c1, os, B, st);
    return;
  }
  NttTagScope tag_(NTT_TAG_MODDOWN);
  const int32_t lp = level;
  const uint64_t pm = L.p_mod_ql;
  for (int g = 0; g < 2 && in; ++g) {  // the q_level source row: acc + P * in
    uint64_t* row = acc + (size_t)g * n_ext * N + (size_t)level * N;
    const int64_t rs = (int64_t)2 * n_ext * (int64_t)N;
    EwArgs A{HEGPU_OP_AXPYC, in + g * in_c1 + (size_t)level * N, is, row, rs, row, rs, B, 1, &lp,
             &pm};
    launch_elementwise(R.dpc, R.primes, R.log_n, A, st);
  }
  std::vector<int32_t> dsel{level};
  for (int i = 0; i < K; ++i) dsel.push_back(R.n_chain + i);
  SegSet S0;
  S0.n_seg = 0;
  S0.n_rows = 0;
  add_seg(S0, acc + (size_t)level * N, (int64_t)n_ext * N, acc + (size_t)level * N,
          (int64_t)n_ext * N, 2 * B, K + 1, dsel.data());
  NttEpilogue E0;
  E0.post = true;
  for (int i = 0; i <= K; ++i) {
    E0.fin_s[i] = L.mdr_fin_s[i];
    E0.fin_d[i] = L.mdr_fin_d[i];
  }
  launch_ntt(R.dpc, R.dtw, R.log_n, true, S0, &E0, st, &R.fp_mask);
  const std::vector<int32_t> chain = range_primes(0, level);
  SegSet S;
  S.n_seg = 0;
  S.n_rows = 0;
  for (int g = 0; g < 2; ++g) {
    add_seg(S, corr + (size_t)g * level * N, (int64_t)2 * level * N,
            corr + (size_t)g * level * N, (int64_t)2 * level * N, B, level, chain.data());
    Seg& sg = S.seg[g];
    sg.other = acc + (size_t)g * n_ext * N;
    sg.other_stride = (int64_t)2 * n_ext * N;
    sg.eout = out + g * out_c1;
    sg.eout_stride = os;
    sg.eacc = in ? 2 : 0;  // in == nullptr: acc already holds P * in + KS (extended basis)
    sg.ein = in ? in + g * in_c1 : nullptr;
    sg.ein_stride = is;
    sg.csrc = acc + (size_t)g * n_ext * N + (size_t)level * N;
    sg.csrc_stride = (int64_t)2 * n_ext * N;
    sg.cpunc = L.mdr_punc;
    sg.c_nsrc = K + 1;
    sg.cpunc_ld = level;
    sg.cmode = 2;  // centered: (X - y) / D is round(X / D)
    sg.cnegd = L.mdr_negd;
    sg.cfw = reinterpret_cast<const float*>(L.mdr_fw_words);
    sg.cfs = reinterpret_cast<const int32_t*>(L.mdr_fs_words);
  }
  NttEpilogue E;
  E.enabled = true;
  for (int t = 0; t < level; ++t) {
    E.c[t] = L.dinv[t];
    E.csh[t] = L.dinv_sh[t];
    E.s[t] = L.qlinv[t];
    E.ssh[t] = L.qlinv_sh[t];
  }
  launch_ntt(R.dpc, R.dtw, R.log_n, false, S, &E, st, &R.fp_mask);
}

static void ks_apply_rescale_impl(Ring& R, int level, int alpha, const uint64_t* d, int64_t ds,
                                  int B, const uint64_t* const* key_b,
                                  const uint64_t* const* key_a, int n_digits, uint64_t* in,
                                  int64_t is, int64_t in_c1, uint64_t* out, int64_t os,
                                  int64_t out_c1, cudaStream_t st) {
  if (B <= 0) return;
  const KsLevel& L = R.ks_level(level, alpha);
  const int k = level + 1, n_ext = L.n_ext, beta = L.beta;
  const size_t N = R.n;
  if (n_digits < beta) throw HegpuError{HEGPU_E_ARG, "switching key has too few digits"};
  if (beta > kMaxDigits) throw HegpuError{HEGPU_E_ARG, "too many digits"};
  const size_t sz_dc = (size_t)B * k * N, sz_ext = (size_t)B * beta * n_ext * N;
  const size_t sz_acc = (size_t)B * 2 * n_ext * N, sz_corr = (size_t)B * 2 * k * N;
  Scratch ws((sz_dc + sz_ext + sz_acc + sz_corr) * 8, st);
  uint64_t* dcoeff = ws.u64();
  uint64_t* ext = dcoeff + sz_dc;
  uint64_t* acc = ext + sz_ext;
  uint64_t* corr = acc + sz_acc;
  ks_modup(R, L, d, ds, B, dcoeff, ext, st);
  ks_ip(R, L, d, ds, ext, B, key_b, key_a, acc, false, st);
  ks_moddown_rescale(R, L, acc, corr, B, in, is, in_c1, out, os, out_c1, st);
}

// Hoisted rotations (bootstrap baby steps): ModUp of c1 once, then per
// rotation r: permute the digits by X -> X^g[r] (eval-form slot gather),
// inner product with rotation key r, ModDown, and c0' = sigma(c0) + b.
// sigma commutes with the RNS digit decomposition up to the usual
// fast-conversion error (a multiple of the digit modulus), so each output
// decrypts exactly like the unhoisted rotation; limbs differ from it.
// c: B packed ciphertexts at `level` (c0 at c + b*cs, c1 at +c1_off);
// outs[r]: packed output ciphertexts with the same layout.
static void ks_hoisted_impl(Ring& R, int level, int alpha, const uint64_t* c, int64_t cs,
                            int64_t c1_off, int B, int n_rot, const uint64_t* galois,
                            const uint64_t* const* key_b, const uint64_t* const* key_a,
                            int n_digits, uint64_t* const* outs, cudaStream_t st,
                            bool pq_out = false) {
  if (B <= 0 || n_rot <= 0) return;
  const KsLevel& L = R.ks_level(level, alpha);
  const int k = level + 1, n_ext = L.n_ext, beta = L.beta;
  const size_t N = R.n;
  if (n_digits < beta) throw HegpuError{HEGPU_E_ARG, "switching key has too few digits"};
  if (beta > kMaxRotDigits) throw HegpuError{HEGPU_E_ARG, "too many digits for hoisting"};
  // outputs laid out back to back (rotation-major) share one batched ModDown
  const int64_t ocs = pq_out ? (int64_t)2 * n_ext * N : cs;  // output ct stride
  bool uniform = true;
  for (int r = 1; r < n_rot; ++r) uniform &= outs[r] == outs[0] + (int64_t)r * B * ocs;
  if (pq_out) {
    // double hoisting: the rotations stay in the extended basis Q_level + P,
    // P-scaled (c0' = P sigma(c0) + kb, c1' = ka); no ModDown at all.  The
    // inner-product launch writes them directly (c0 term fused).
    if (!uniform) throw HegpuError{HEGPU_E_ARG, "extended-basis outputs must be packed"};
    const size_t sz_dc = (size_t)B * k * N, sz_ext = (size_t)B * beta * n_ext * N;
    Scratch ws((sz_dc + sz_ext) * 8, st);
    uint64_t* dcoeff = ws.u64();
    uint64_t* ext = dcoeff + sz_dc;
    ks_modup(R, L, c + c1_off, cs, B, dcoeff, ext, st);
    const std::vector<uint64_t> sp(R.primes.begin() + R.n_chain, R.primes.end());
    for (int r0 = 0; r0 < n_rot; r0 += kMaxRot) {
      const int nr = std::min(kMaxRot, n_rot - r0);
      IpRotParams P{};
      P.d = c + c1_off;
      P.ds = cs;
      P.ext = ext;
      P.ext_sb = (int64_t)beta * n_ext * N;
      P.ext_sj = (int64_t)n_ext * N;
      for (int r = 0; r < nr; ++r) {
        P.gal[r] = (uint32_t)galois[r0 + r];
        for (int j = 0; j < beta; ++j) {
          P.kb[r][j] = key_b[(size_t)(r0 + r) * n_digits + j];
          P.ka[r][j] = key_a[(size_t)(r0 + r) * n_digits + j];
        }
      }
      P.n_rot = nr;
      P.acc = outs[r0];
      P.acc_sb = ocs;
      P.acc_sr = (int64_t)B * ocs;
      P.level = level;
      P.alpha = alpha;
      P.beta = beta;
      P.n_ext = n_ext;
      P.n_chain = R.n_chain;
      P.key_sp_row0 = R.n_chain;
      P.n_batch = B;
      P.log_n = R.log_n;
      P.pc = R.dpc;
      P.c0 = c;
      P.c0s = cs;
      for (int t = 0; t < k; ++t) {
        P.pm[t] = prod_mod(sp, -1, R.primes[t]);
        P.pm_sh[t] = h_shoup(P.pm[t], R.primes[t]);
      }
      launch_ks_ip_rot(P, st);
    }
    return;
  }
  const int CH = kMaxRot;
  const size_t sz_dc = (size_t)B * k * N, sz_ext = (size_t)B * beta * n_ext * N;
  const size_t sz_acc = (size_t)B * 2 * n_ext * N, sz_corr = (size_t)B * 2 * k * N;
  Scratch ws((sz_dc + sz_ext + CH * (sz_acc + sz_corr)) * 8, st);
  uint64_t* dcoeff = ws.u64();
  uint64_t* ext = dcoeff + sz_dc;
  uint64_t* acc = ext + sz_ext;
  uint64_t* corr = acc + CH * sz_acc;
  const uint64_t* c1 = c + c1_off;
  ks_modup(R, L, c1, cs, B, dcoeff, ext, st);
  const std::vector<int32_t> chain = range_primes(0, k);
  for (int r0 = 0; r0 < n_rot; r0 += CH) {
    const int nr = std::min(CH, n_rot - r0);
    // the nr rotations' inner products in one launch, digits gathered through
    // X -> X^g[r] (no permuted copies), one acc per rotation
    IpRotParams P{};
    P.d = c1;
    P.ds = cs;
    P.d_sr = 0;
    P.ext = ext;
    P.ext_sb = (int64_t)beta * n_ext * N;
    P.ext_sj = (int64_t)n_ext * N;
    P.ext_sr = 0;
    for (int r = 0; r < nr; ++r) {
      P.gal[r] = (uint32_t)galois[r0 + r];
      for (int j = 0; j < beta; ++j) {
        P.kb[r][j] = key_b[(size_t)(r0 + r) * n_digits + j];
        P.ka[r][j] = key_a[(size_t)(r0 + r) * n_digits + j];
      }
    }
    P.n_rot = nr;
    P.sum_mode = 0;
    P.accumulate = 0;
    P.acc = acc;
    P.acc_sb = (int64_t)2 * n_ext * N;
    P.acc_sr = (int64_t)sz_acc;
    P.level = level;
    P.alpha = alpha;
    P.beta = beta;
    P.n_ext = n_ext;
    P.n_chain = R.n_chain;
    P.key_sp_row0 = R.n_chain;
    P.n_batch = B;
    P.log_n = R.log_n;
    P.pc = R.dpc;
    launch_ks_ip_rot(P, st);
    // c0' = sigma(c0) + kb: permute c0 into place, then the ModDown epilogue
    // accumulates kb into it; c1' = ka is written directly
    for (int r = 0; r < nr; ++r)
      launch_automorphism(R.dpc, R.log_n, true, galois[r0 + r], c, cs, outs[r0 + r], cs, B, k,
                          chain.data(), st);
    if (uniform) {
      ks_moddown(R, L, acc, corr, nr * B, outs[r0], cs, outs[r0] + c1_off, cs, st,
                 /*acc_b=*/true, /*acc_a=*/false);
    } else {
      for (int r = 0; r < nr; ++r)
        ks_moddown(R, L, acc + r * sz_acc, corr, B, outs[r0 + r], cs, outs[r0 + r] + c1_off, cs,
                   st, /*acc_b=*/true, /*acc_a=*/false);
    }
  }
}

// Hoisted rotation sum: out = ct + sum_r rot_r(ct).  One ModUp of c1, then
// per rotation the digits are permuted (eval-form gather) and the inner
// product with key r accumulates in the extended basis; the sum is brought
// down by ONE ModDown whose epilogue adds it to c0 + sum_r sigma_r(c0) and
// c1.  Replaces n_rot sequential rotate-and-add key switches (each with its
// own ModUp and ModDown) of the reference's rotate-and-sum loops
// (logreg.py:202-229): same slots, limbs differ by the conversion rounding.
// c / out: B packed ciphertexts (c0 at +b*cs / +b*os, c1 at +c1_off /
// +out_c1); out may not alias c.
static void ks_rotsum_impl(Ring& R, int level, int alpha, const uint64_t* c, int64_t cs,
                           int64_t c1_off, int B, int n_rot, const uint64_t* galois,
                           const uint64_t* const* key_b, const uint64_t* const* key_a,
                           int n_digits, uint64_t* out, int64_t os, int64_t out_c1,
                           cudaStream_t st) {
  if (B <= 0) return;
  const KsLevel& L = R.ks_level(level, alpha);
  const int k = level + 1, n_ext = L.n_ext, beta = L.beta;
  const size_t N = R.n;
  const std::vector<int32_t> chain = range_primes(0, k);
  std::vector<uint32_t> gal(n_rot > 0 ? n_rot : 1);
  for (int r = 0; r < n_rot; ++r) gal[r] = (uint32_t)galois[r];
  // c1' = c1 (+ ModDown of the accumulated inner products below)
  EwArgs A{HEGPU_OP_COPY, c + c1_off, cs, nullptr, 0, out + out_c1, os, B, k, chain.data(),
           nullptr};
  launch_elementwise(R.dpc, R.primes, R.log_n, A, st);
  // c0' = c0 + sum_r sigma_r(c0): one gather-sum pass per 16 rotations
  for (int r0 = 0; r0 < std::max(n_rot, 1); r0 += kMaxRot) {
    const int nr = std::min(kMaxRot, n_rot - r0);
    launch_auto_sum(R.dpc, R.log_n, gal.data() + r0, std::max(nr, 0), c, cs, r0 ? out : nullptr,
                    os, out, os, B, k, st);
  }
  if (n_rot <= 0) return;
  if (n_digits < beta) throw HegpuError{HEGPU_E_ARG, "switching key has too few digits"};
  if (beta > kMaxRotDigits) throw HegpuError{HEGPU_E_ARG, "too many digits for rotsum"};
  const size_t sz_dc = (size_t)B * k * N, sz_ext = (size_t)B * beta * n_ext * N;
  const size_t sz_acc = (size_t)B * 2 * n_ext * N, sz_corr = (size_t)B * 2 * k * N;
  Scratch ws((sz_dc + sz_ext + sz_acc + sz_corr) * 8, st);
  uint64_t* dcoeff = ws.u64();
  uint64_t* ext = dcoeff + sz_dc;
  uint64_t* acc = ext + sz_ext;
  uint64_t* corr = acc + sz_acc;
  ks_modup(R, L, c + c1_off, cs, B, dcoeff, ext, st);
  for (int r0 = 0; r0 < n_rot; r0 += kMaxRot) {
    const int nr = std::min(kMaxRot, n_rot - r0);
    IpRotParams P{};
    P.d = c + c1_off;
    P.ds = cs;
    P.d_sr = 0;
    P.ext = ext;
    P.ext_sb = (int64_t)beta * n_ext * N;
    P.ext_sj = (int64_t)n_ext * N;
    P.ext_sr = 0;
    for (int r = 0; r < nr; ++r) {
      P.gal[r] = gal[r0 + r];
      for (int j = 0; j < beta; ++j) {
        P.kb[r][j] = key_b[(size_t)(r0 + r) * n_digits + j];
        P.ka[r][j] = key_a[(size_t)(r0 + r) * n_digits + j];
      }
    }
    P.n_rot = nr;
    P.sum_mode = 1;
    P.accumulate = r0 > 0;
    P.acc = acc;
    P.acc_sb = (int64_t)2 * n_ext * N;
    P.acc_sr = 0;
    P.level = level;
    P.alpha = alpha;
    P.beta = beta;
    P.n_ext = n_ext;
    P.n_chain = R.n_chain;
    P.key_sp_row0 = R.n_chain;
    P.n_batch = B;
    P.log_n = R.log_n;
    P.pc = R.dpc;
    launch_ks_ip_rot(P, st);
  }
  ks_moddown(R, L, acc, corr, B, out, os, out + out_c1, os, st, /*acc_b=*/true, /*acc_a=*/true);
}

// Giant steps of a BSGS transform with one lazy ModDown (double hoisting):
// out = partial[0] + sum_{g>0} rot_{galois[g]}(partial[g]).  Each giant's key
// inner product accumulates in the extended basis; the sum is brought down
// once.  Decrypts like the per-giant rotate-and-add (bootstrap.py:243-245);
// limbs differ (ModDown is linear only up to its rounding).
// partials: n_giants packed (B, 2, k, N) ciphertexts, giant g at
// partials + g*gstride; out: packed (B, 2, k, N).
// out = partial[0] + sum_g rot_g(partial[g]) at `level`; with `down` the
// final ModDown is fused with the rescale and writes `down` (level - 1)
// instead (out is then clobbered scratch).
static void bsgs_giants_sum_pq(Ring& R, int level, int alpha, uint64_t* partials,
                               int64_t gstride, int B, int n_giants, const uint64_t* galois,
                               const uint64_t* const* key_b, const uint64_t* const* key_a,
                               int n_digits, uint64_t* down, cudaStream_t st,
                               bool ext_out = false);

static void bsgs_giants_sum(Ring& R, int level, int alpha, const uint64_t* partials,
                            int64_t gstride, int B, int n_giants, const uint64_t* galois,
                            const uint64_t* const* key_b, const uint64_t* const* key_a,
                            int n_digits, uint64_t* out, cudaStream_t st, uint64_t* down) {
  const KsLevel& L = R.ks_level(level, alpha);
  const int k = level + 1, n_ext = L.n_ext, beta = L.beta;
  const size_t N = R.n;
  const int64_t cs = (int64_t)2 * k * N;  // packed batch stride
  if (n_digits < beta) throw HegpuError{HEGPU_E_ARG, "switching key has too few digits"};
  if (beta > kMaxRotDigits) throw HegpuError{HEGPU_E_ARG, "too many digits for giant steps"};
  if (gstride < (int64_t)B * cs) throw HegpuError{HEGPU_E_ARG, "giant stride too small"};
  const std::vector<int32_t> chain = range_primes(0, k);
  {  // out.c1 = partial[0].c1 (the ModDown epilogue adds the switched parts)
    EwArgs A{HEGPU_OP_COPY, partials + (size_t)k * N, cs, nullptr, 0, out + (size_t)k * N, cs, B,
             k, chain.data(), nullptr};
    launch_elementwise(R.dpc, R.primes, R.log_n, A, st);
  }
  std::vector<uint32_t> gal(std::max(n_giants, 1));
  for (int g = 0; g < n_giants; ++g) gal[g] = (uint32_t)galois[g];
  // out.c0 = partial[0].c0 + sum_g sigma_g(partial[g].c0), 16 giants per pass
  for (int g0 = 1; g0 < std::max(n_giants, 2); g0 += kMaxRot) {
    const int ng = std::max(0, std::min(kMaxRot, n_giants - g0));
    launch_auto_sum(R.dpc, R.log_n, gal.data() + g0, ng, partials + g0 * gstride, cs,
                    g0 == 1 ? partials : out, cs, out, cs, B, k, st, gstride);
  }
  if (n_giants <= 1) return;
  // ModUp of up to 16 giants' c1 in one batch (uniform stride when the giants
  // are packed back to back), then one inner-product launch that gathers each
  // giant's digits through its automorphism and sums over the giants
  const bool packed = gstride == (int64_t)B * cs;
  const int CH = packed ? kMaxRot : 1;
  const size_t sz_dc = (size_t)CH * B * k * N, sz_ext = (size_t)CH * B * beta * n_ext * N;
  const size_t sz_acc = (size_t)B * 2 * n_ext * N, sz_corr = (size_t)B * 2 * k * N;
  Scratch ws((sz_dc + sz_ext + sz_acc + sz_corr) * 8, st);
  uint64_t* dcoeff = ws.u64();
  uint64_t* ext = dcoeff + sz_dc;
  uint64_t* acc = ext + sz_ext;
  uint64_t* corr = acc + sz_acc;
  bool first = true;
  for (int g0 = 1; g0 < n_giants; g0 += CH) {
    const int ng = std::min(CH, n_giants - g0);
    const uint64_t* c1 = partials + g0 * gstride + (size_t)k * N;
    ks_modup(R, L, c1, cs, ng * B, dcoeff, ext, st);
    IpRotParams P{};
    P.d = c1;
    P.ds = cs;
    P.d_sr = gstride;
    P.ext = ext;
    P.ext_sb = (int64_t)beta * n_ext * N;
    P.ext_sj = (int64_t)n_ext * N;
    P.ext_sr = (int64_t)B * beta * n_ext * N;
    for (int r = 0; r < ng; ++r) {
      P.gal[r] = gal[g0 + r];
      for (int j = 0; j < beta; ++j) {
        P.kb[r][j] = key_b[(size_t)(g0 + r) * n_digits + j];
        P.ka[r][j] = key_a[(size_t)(g0 + r) * n_digits + j];
      }
    }
    P.n_rot = ng;
    P.sum_mode = 1;
    P.accumulate = first ? 0 : 1;
    P.acc = acc;
    P.acc_sb = (int64_t)2 * n_ext * N;
    P.acc_sr = 0;
    P.level = level;
    P.alpha = alpha;
    P.beta = beta;
    P.n_ext = n_ext;
    P.n_chain = R.n_chain;
    P.key_sp_row0 = R.n_chain;
    P.n_batch = B;
    P.log_n = R.log_n;
    P.pc = R.dpc;
    launch_ks_ip_rot(P, st);
    first = false;
  }
  if (down) {
    ks_moddown_rescale(R, L, acc, corr, B, out, cs, (int64_t)k * N, down, (int64_t)2 * level * N,
                       (int64_t)level * N, st);
    return;
  }
  ks_moddown(R, L, acc, corr, B, out, cs, out + (size_t)k * N, cs, st, true, true);
}

// Giant steps of a double-hoisted transform: the partial sums are P-scaled
// extended-basis ciphertexts (babies never went through ModDown).  Per giant
// g >= 1 only c1 is brought down (one-poly ModDown, needed for its digit
// decomposition); the permuted c0 parts and every giant's inner products
// accumulate in the extended basis, and ONE ModDown by q_level * P (fused
// with the transform's rescale) ends at level - 1 in `down`.  partials
// (packed (n_giants, B, 2, n_ext, N)) are clobbered.  N >= 2^12.
static void bsgs_giants_sum_pq(Ring& R, int level, int alpha, uint64_t* partials,
                               int64_t gstride, int B, int n_giants, const uint64_t* galois,
                               const uint64_t* const* key_b, const uint64_t* const* key_a,
                               int n_digits, uint64_t* down, cudaStream_t st, bool ext_out) {
  const KsLevel& L = R.ks_level(level, alpha);
  const int k = level + 1, n_ext = L.n_ext, beta = L.beta;
  const size_t N = R.n;
  const int64_t cs = (int64_t)2 * n_ext * N;
  if (level < 1) throw HegpuError{HEGPU_E_ARG, "rescale at level 0"};
  if (n_digits < beta) throw HegpuError{HEGPU_E_ARG, "switching key has too few digits"};
  if (beta > kMaxRotDigits) throw HegpuError{HEGPU_E_ARG, "too many digits for giant steps"};
  if (gstride != (int64_t)B * cs) throw HegpuError{HEGPU_E_ARG, "partials must be packed"};
  const std::vector<int32_t> ext_rows = [&] {
    std::vector<int32_t> v = range_primes(0, k);
    for (int i = 0; i < R.n_special; ++i) v.push_back(R.n_chain + i);
    return v;
  }();
  std::vector<uint32_t> gal(std::max(n_giants, 1));
  for (int g = 0; g < n_giants; ++g) gal[g] = (uint32_t)galois[g];
  const int CH = kMaxRot;
  const size_t sz_pq = (size_t)B * cs, sz_q = (size_t)CH * B * k * N;
  const size_t sz_ext = (size_t)CH * B * beta * n_ext * N;
  Scratch ws((sz_pq + 2 * sz_q + sz_ext + sz_pq + sz_q) * 8, st);
  // (B, 2, n_ext, N); ext_out: the caller's buffer receives the extended-basis
  // sum and the final ModDown is left to it (a distributed transform reduces
  // the per-rank sums first)
  uint64_t* sum = ext_out ? down : ws.u64();
  uint64_t* c1q = ws.u64() + sz_pq;  // (CH*B, k, N)
  uint64_t* dcoeff = c1q + sz_q;
  uint64_t* ext = dcoeff + sz_q;
  uint64_t* acc = ext + sz_ext;  // (B, 2, n_ext, N)
  uint64_t* corr = acc + sz_pq;  // >= CH*B*k*N and >= B*2*level*N
  // sum.c0 = partial[0].c0 + sum_g sigma_g(partial[g].c0); sum.c1 = partial[0].c1
  for (int g0 = 1; g0 < std::max(n_giants, 2); g0 += kMaxRot) {
    const int ng = std::max(0, std::min(kMaxRot, n_giants - g0));
    launch_auto_sum(R.dpc, R.log_n, gal.data() + g0, ng, partials + g0 * gstride, cs,
                    g0 == 1 ? partials : sum, cs, sum, cs, B, n_ext, st, gstride, k, R.n_chain);
  }
  {
    EwArgs A{HEGPU_OP_COPY, partials + (size_t)n_ext * N, cs, nullptr, 0, sum + (size_t)n_ext * N,
             cs, B, n_ext, ext_rows.data(), nullptr};
    launch_elementwise(R.dpc, R.primes, R.log_n, A, st);
  }
  bool first = true;
  for (int g0 = 1; g0 < n_giants; g0 += CH) {
    const int ng = std::min(CH, n_giants - g0);
    ks_moddown_polys(R, L, partials + g0 * gstride + (size_t)n_ext * N, cs, ng * B, c1q,
                     (int64_t)k * N, corr, st);
    ks_modup(R, L, c1q, (int64_t)k * N, ng * B, dcoeff, ext, st);
    IpRotParams P{};
    P.d = c1q;
    P.ds = (int64_t)k * N;
    P.d_sr = (int64_t)B * k * N;
    P.ext = ext;
    P.ext_sb = (int64_t)beta * n_ext * N;
    P.ext_sj = (int64_t)n_ext * N;
    P.ext_sr = (int64_t)B * beta * n_ext * N;
    for (int r = 0; r < ng; ++r) {
      P.gal[r] = gal[g0 + r];
      for (int j = 0; j < beta; ++j) {
        P.kb[r][j] = key_b[(size_t)(g0 + r) * n_digits + j];
        P.ka[r][j] = key_a[(size_t)(g0 + r) * n_digits + j];
      }
    }
    P.n_rot = ng;
    P.sum_mode = 1;
    P.accumulate = first ? 0 : 1;
    P.acc = acc;
    P.acc_sb = cs;
    P.level = level;
    P.alpha = alpha;
    P.beta = beta;
    P.n_ext = n_ext;
    P.n_chain = R.n_chain;
    P.key_sp_row0 = R.n_chain;
    P.n_batch = B;
    P.log_n = R.log_n;
    P.pc = R.dpc;
    launch_ks_ip_rot(P, st);
    first = false;
  }
  if (!first) {  // sum += the giants' switched parts (both components, extended basis)
    EwArgs A{HEGPU_OP_ADD, sum, (int64_t)n_ext * (int64_t)N, acc, (int64_t)n_ext * (int64_t)N, sum,
             (int64_t)n_ext * (int64_t)N, 2 * B, n_ext, ext_rows.data(), nullptr};
    launch_elementwise(R.dpc, R.primes, R.log_n, A, st);
  }
  if (ext_out) return;
  ks_moddown_rescale(R, L, sum, corr, B, nullptr, 0, 0, down, (int64_t)2 * level * N,
                     (int64_t)level * N, st);
}

static void bsgs_giants_impl(Ring& R, int level, int alpha, const uint64_t* partials,
                             int64_t gstride, int B, int n_giants, const uint64_t* galois,
                             const uint64_t* const* key_b, const uint64_t* const* key_a,
                             int n_digits, uint64_t* out, cudaStream_t st, bool rescale) {
  if (!rescale) {
    bsgs_giants_sum(R, level, alpha, partials, gstride, B, n_giants, galois, key_b, key_a,
                    n_digits, out, st, nullptr);
    return;
  }
  // the level-`level` sum goes to scratch; one ModDown by q_level * P leaves
  // the rescaled result (level - 1) in out
  if (level < 1) throw HegpuError{HEGPU_E_ARG, "rescale at level 0"};
  Scratch tmp((size_t)B * 2 * (level + 1) * R.n * 8, st);
  bsgs_giants_sum(R, level, alpha, partials, gstride, B, n_giants, galois, key_b, key_a,
                  n_digits, tmp.u64(), st, out);
}

// --- rescale (ops.py:164-189) and ModRaise (bootstrap.py:260-275) ----------

static void rescale_impl(Ring& R, int level, const uint64_t* in, int64_t is, uint64_t* out,
                         int64_t os, int P, cudaStream_t st) {
  NttTagScope tag_(NTT_TAG_RESCALE);
  if (level < 1 || level >= R.n_chain) throw HegpuError{HEGPU_E_ARG, "rescale level out of range"};
  if (P <= 0) return;
  const size_t N = R.n;
  const auto& cs = R.rescale_consts(level);
  const bool fused = R.log_n >= 12;
  Scratch ws((size_t)P * (1 + level) * N * 8, st);
  uint64_t* top = ws.u64();
  uint64_t* rest = top + (size_t)P * N;
  const int32_t lp = level;
  ntt_simple(R, true, in + (size_t)level * N, is, top, (int64_t)N, P, 1, &lp, st);
  const std::vector<int32_t> chain = range_primes(0, level);
  if (!fused)
    launch_lift_centered(R.dpc, R.log_n, top, (int64_t)N, R.primes[level], rest,
                         (int64_t)level * N, P, level, chain.data(), st);
  SegSet S;
  S.n_seg = 0;
  S.n_rows = 0;
  add_seg(S, rest, (int64_t)level * N, rest, (int64_t)level * N, P, level, chain.data());
  S.seg[0].other = in;
  S.seg[0].other_stride = is;
  S.seg[0].eout = out;
  S.seg[0].eout_stride = os;
  if (fused) {  // the centered lift of the top limb runs inside the NTT's first pass
    S.seg[0].csrc = top;
    S.seg[0].csrc_stride = (int64_t)N;
    S.seg[0].cmode = 1;
    S.seg[0].csrc_q = R.primes[level];
  }
  NttEpilogue E;
  E.enabled = true;
  for (int i = 0; i < level; ++i) {
    E.c[i] = cs.first[i];
    E.csh[i] = cs.second[i];
  }
  launch_ntt(R.dpc, R.dtw, R.log_n, false, S, &E, st, &R.fp_mask);
}

static void mod_raise_impl(Ring& R, const uint64_t* in, int64_t is, uint64_t* out, int64_t os,
                           int P, int to_level, cudaStream_t st) {
  NttTagScope tag_(NTT_TAG_RESCALE);
  if (to_level < 0 || to_level >= R.n_chain) throw HegpuError{HEGPU_E_ARG, "bad target level"};
  if (P <= 0) return;
  const size_t N = R.n;
  Scratch ws((size_t)P * N * 8, st);
  const int32_t p0 = 0;
  ntt_simple(R, true, in, is, ws.u64(), (int64_t)N, P, 1, &p0, st);
  const std::vector<int32_t> chain = range_primes(0, to_level + 1);
  if (R.log_n >= 12) {
    SegSet S;
    S.n_seg = 0;
    S.n_rows = 0;
    add_seg(S, nullptr, 0, out, os, P, to_level + 1, chain.data());
    S.seg[0].csrc = ws.u64();
    S.seg[0].csrc_stride = (int64_t)N;
    S.seg[0].cmode = 1;
    S.seg[0].csrc_q = R.primes[0];
    launch_ntt(R.dpc, R.dtw, R.log_n, false, S, nullptr, st, &R.fp_mask);
    return;
  }
  launch_lift_centered(R.dpc, R.log_n, ws.u64(), (int64_t)N, R.primes[0], out, os, P,
                       to_level + 1, chain.data(), st);
  ntt_simple(R, false, out, os, out, os, P, to_level + 1, chain.data(), st);
}

// Eval-form limbs of signed int64 coefficient rows: lift (np.mod into every
// limb) fused into the forward NTT's first pass.
void ntt_from_signed(Ring& R, const int64_t* src, int64_t ss, uint64_t* out, int64_t os, int P,
                     int k, const int32_t* primes, cudaStream_t st) {
  if (P <= 0 || k <= 0) return;
  if (R.log_n >= 12) {
    SegSet S;
    S.n_seg = 0;
    S.n_rows = 0;
    add_seg(S, nullptr, 0, out, os, P, k, primes);
    S.seg[0].csrc = reinterpret_cast<const uint64_t*>(src);
    S.seg[0].csrc_stride = ss;
    S.seg[0].cmode = 3;
    launch_ntt(R.dpc, R.dtw, R.log_n, false, S, nullptr, st, &R.fp_mask);
    return;
  }
  launch_lift_signed(R.dpc, R.log_n, src, ss, out, os, P, k, primes, st);
  ntt_simple(R, false, out, os, out, os, P, k, primes, st);
}

// --- host-array kernel-table shims (hebert._kernels) -----------------------

struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) {
    if (bytes) check_cuda(cudaMalloc(&p, bytes), "device alloc");
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  uint64_t* u64() const { return static_cast<uint64_t*>(p); }
};

static void h2d(void* d, const void* h, size_t bytes) {
  check_cuda(cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice), "H2D copy");
}
static void d2h(void* h, const void* d, size_t bytes) {
  check_cuda(cudaMemcpy(h, d, bytes, cudaMemcpyDeviceToHost), "D2H copy");
}

static int ilog2_exact(int n) {
  int l = 0;
  while ((1 << l) < n) ++l;
  if ((1 << l) != n) throw HegpuError{HEGPU_E_ARG, "n must be a power of two"};
  return l;
}

// Per-call constant table for arbitrary primes given as (q, qinv_neg).
static std::vector<PrimeConst> shim_consts(const uint64_t* q, int k, int log_n) {
  if (k > kMaxPrimes) throw HegpuError{HEGPU_E_ARG, "too many rows"};
  std::vector<PrimeConst> pc(k);
  for (int i = 0; i < k; ++i) {
    if (q[i] < 3 || q[i] >= (1ull << 62) || (q[i] & 1) == 0)
      throw HegpuError{HEGPU_E_ARG, "moduli must be odd and < 2^62"};
    pc[i] = make_prime_const(q[i], log_n, 1);
  }
  return pc;
}

static void shim_elementwise(int op, const uint64_t* a, const uint64_t* b, uint64_t* out, int k,
                             int n, const uint64_t* q, const uint64_t* consts) {
  if (k == 0 || n == 0) return;
  const int log_n = ilog2_exact(n);
  if (n < 2) throw HegpuError{HEGPU_E_ARG, "n too small"};
  auto pc = shim_consts(q, k, log_n);
  const size_t bytes = (size_t)k * n * 8;
  DevBuf dpc(pc.size() * sizeof(PrimeConst)), da(bytes), db(b ? bytes : 0), dout(bytes);
  h2d(dpc.p, pc.data(), pc.size() * sizeof(PrimeConst));
  h2d(da.p, a, bytes);
  if (b) h2d(db.p, b, bytes);
  if (op == HEGPU_OP_FMA) h2d(dout.p, out, bytes);
  std::vector<uint64_t> hq(q, q + k);
  std::vector<int32_t> sel = range_primes(0, k);
  EwArgs A{op, da.u64(), 0, b ? db.u64() : nullptr, 0, dout.u64(), 0, 1, k, sel.data(), consts};
  launch_elementwise(static_cast<PrimeConst*>(dpc.p), hq, log_n, A, 0);
  d2h(out, dout.p, bytes);
}

static void shim_ntt(bool inverse, uint64_t* a, int k, int n, const uint64_t* tw_mont,
                     const uint64_t* ninv_mont, const uint64_t* q) {
  if (k == 0) return;
  const int log_n = ilog2_exact(n);
  if (log_n < 2) throw HegpuError{HEGPU_E_ARG, "n too small for the NTT"};
  std::vector<PrimeConst> pc(k);
  std::vector<uint64_t> tw((size_t)k * 4 * n, 0);
  for (int i = 0; i < k; ++i) {
    const uint64_t qi = q[i];
    if (qi < 3 || qi >= (1ull << 62) || (qi & 1) == 0)
      throw HegpuError{HEGPU_E_ARG, "moduli must be odd and < 2^62"};
    const uint64_t rinv = h_inv(h_rmod(qi), qi);  // Montgomery -> natural
    uint64_t* t = tw.data() + (size_t)i * 4 * n + (inverse ? 2 * (size_t)n : 0);
    for (int j = 0; j < n; ++j) {
      const uint64_t w = h_mulmod(tw_mont[(size_t)i * n + j] % qi, rinv, qi);
      t[2 * j] = w;
      t[2 * j + 1] = h_shoup(w, qi);
    }
    pc[i] = make_prime_const(qi, log_n, inverse ? t[2] : 1);
    if (inverse) {
      pc[i].ninv = h_mulmod(ninv_mont[i] % qi, rinv, qi);
      pc[i].ninv_sh = h_shoup(pc[i].ninv, qi);
      pc[i].ilast = h_mulmod(t[2], pc[i].ninv, qi);
      pc[i].ilast_sh = h_shoup(pc[i].ilast, qi);
    }
  }
  const size_t bytes = (size_t)k * n * 8;
  DevBuf dtwf(0);
  if (log_n >= 12) dtwf.p = attach_fp_twiddles(pc, tw.data(), n);
  DevBuf dpc(pc.size() * sizeof(PrimeConst)), dtw(tw.size() * 8), da(bytes);
  h2d(dpc.p, pc.data(), pc.size() * sizeof(PrimeConst));
  h2d(dtw.p, tw.data(), tw.size() * 8);
  h2d(da.p, a, bytes);
  SegSet S;
  S.n_seg = 0;
  S.n_rows = 0;
  std::vector<int32_t> sel = range_primes(0, k);
  add_seg(S, da.u64(), 0, da.u64(), 0, 1, k, sel.data());
  launch_ntt(static_cast<PrimeConst*>(dpc.p), dtw.u64(), log_n, inverse, S, nullptr, 0);
  d2h(a, da.p, bytes);
}

}  // namespace hegpu

// ============================================================================
// C ABI
// ============================================================================
using namespace hegpu;

struct hegpu_ring {
  Ring* r;
};

#define HEGPU_TRY(...)                          \
  try {                                         \
    __VA_ARGS__;                                \
    return HEGPU_OK;                            \
  } catch (const HegpuError& e) {               \
    set_error(e.msg);                           \
    return e.code;                              \
  } catch (const std::bad_alloc&) {             \
    set_error("host out of memory");            \
    return HEGPU_E_NOMEM;                       \
  } catch (const std::exception& e) {           \
    set_error(e.what());                        \
    return HEGPU_E_ARG;                         \
  }

static Ring& RR(hegpu_ring_t r) {
  if (!r || !r->r) throw HegpuError{HEGPU_E_ARG, "null ring handle"};
  return *r->r;
}
static inline cudaStream_t S_(void* s) { return static_cast<cudaStream_t>(s); }

extern "C" {

const char* hegpu_version(void) { return "hegpu 0.1 (sm_100a)"; }
const char* hegpu_last_error(void) { return g_last_error.c_str(); }
int hegpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    (void)cudaGetLastError();
    return 0;
  }
  return n;
}

long long hegpu_launch_count(void) { return g_launches.load(); }

int hegpu_bench_fp_modmul_peak(int iters, double* modmul_per_s) {
  HEGPU_TRY(*modmul_per_s = bench_fp_modmul_peak(iters))
}

int hegpu_bench_modmul_peak(int iters, double* modmul_per_s) {
  HEGPU_TRY(*modmul_per_s = bench_modmul_peak(iters))
}

int hegpu_profile_enable(int on) {
  HEGPU_TRY({
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (auto& r : g_prof) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    g_prof.clear();
    g_prof_on.store(on != 0);
  })
}

int hegpu_profile_read(double* ms, long long* counts, double* bytes, double* modmuls,
                       int n_classes) {
  HEGPU_TRY({
    check_cuda(cudaDeviceSynchronize(), "profile sync");
    std::lock_guard<std::mutex> lk(g_prof_mu);
    for (int c = 0; c < n_classes; ++c) {
      ms[c] = 0;
      counts[c] = 0;
      bytes[c] = 0;
      modmuls[c] = 0;
    }
    for (auto& r : g_prof) {
      float t = 0;
      check_cuda(cudaEventElapsedTime(&t, r.a, r.b), "event time");
      const int sub = r.sub > 0 ? PROF_NUM_CLASSES + r.sub - 1 : -1;
      for (int c : {r.cls, sub}) {
        if (c < 0 || c >= n_classes) continue;
        ms[c] += t;
        counts[c] += 1;
        bytes[c] += r.bytes;
        modmuls[c] += r.modmuls;
      }
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    g_prof.clear();
  })
}

int hegpu_ring_create(int log_n, const uint64_t* chain, int n_chain, const uint64_t* special,
                      int n_special, hegpu_ring_t* out) {
  HEGPU_TRY({
    if (!out) throw HegpuError{HEGPU_E_ARG, "null output"};
    Ring* r = create_ring(log_n, chain, n_chain, special, n_special);
    *out = new hegpu_ring{r};
  })
}

int hegpu_ring_destroy(hegpu_ring_t ring) {
  HEGPU_TRY({
    if (ring) {
      delete ring->r;
      delete ring;
    }
  })
}

int hegpu_ring_get_tables(hegpu_ring_t ring, int p, uint64_t* host_out4n) {
  HEGPU_TRY({
    Ring& R = RR(ring);
    if (p < 0 || p >= R.n_primes) throw HegpuError{HEGPU_E_ARG, "prime index out of range"};
    d2h(host_out4n, R.dtw + (size_t)p * 4 * R.n, (size_t)4 * R.n * 8);
  })
}

int hegpu_ntt(hegpu_ring_t ring, int inverse, const uint64_t* in, int64_t in_stride,
              uint64_t* out, int64_t out_stride, int n_polys, int k, const int32_t* primes,
              void* stream) {
  HEGPU_TRY({
    Ring& R = RR(ring);
    for (int l = 0; l < k; ++l)
      if (primes[l] >= R.n_primes) throw HegpuError{HEGPU_E_ARG, "prime index out of range"};
    ntt_simple(R, inverse != 0, in, in_stride, out, out_stride, n_polys, k, primes, S_(stream));
  })
}

int hegpu_elementwise(hegpu_ring_t ring, int op, const uint64_t* a, int64_t a_stride,
                      const uint64_t* b, int64_t b_stride, uint64_t* out, int64_t out_stride,
                      int n_polys, int k, const int32_t* primes, const uint64_t* consts,
                      void* stream) {
  HEGPU_TRY({
    Ring& R = RR(ring);
    EwArgs A{op, a, a_stride, b, b_stride, out, out_stride, n_polys, k, primes, consts};
    launch_elementwise(R.dpc, R.primes, R.log_n, A, S_(stream));
  })
}

int hegpu_lift_signed(hegpu_ring_t ring, const int64_t* src, int64_t src_stride, uint64_t* out,
                      int64_t out_stride, int n_polys, int k, const int32_t* primes,
                      void* stream) {
  HEGPU_TRY({
    Ring& R = RR(ring);
    launch_lift_signed(R.dpc, R.log_n, src, src_stride, out, out_stride, n_polys, k, primes,
                       S_(stream));
  })
}

int hegpu_lift_centered(hegpu_ring_t ring, const uint64_t* src, int64_t src_stride,
                        int src_prime, uint64_t* out, int64_t out_stride, int n_polys, int k,
                        const int32_t* primes, void* stream) {
  HEGPU_TRY({
    Ring& R = RR(ring);
    if (src_prime < 0 || src_prime >= R.n_primes) throw HegpuError{HEGPU_E_ARG, "bad src prime"};
    launch_lift_centered(R.dpc, R.log_n, src, src_stride, R.primes[src_prime], out, out_stride,
                         n_polys, k, primes, S_(stream));
  })
}

int hegpu_encode_diags(hegpu_ring_t ring, int kind, int half, double fold, double scale,
                       int n_diags, const int32_t* d, const int32_t* g0, const uint8_t* conj,
                       void* scratch, int64_t* out, void* stream) {
  HEGPU_TRY({
    Ring& R = RR(ring);
    launch_encode_diags(R, kind, half, fold, scale, n_diags, d, g0, conj,
                        static_cast<double2*>(scratch), out, S_(stream));
  })
}

int hegpu_ntt_from_signed(hegpu_ring_t ring, const int64_t* src, int64_t src_stride,
                          uint64_t* out, int64_t out_stride, int n_polys, int k,
                          const int32_t* primes, void* stream) {
  HEGPU_TRY({
    Ring& R = RR(ring);
    for (int l = 0; l < k; ++l)
      if (primes[l] < 0 || primes[l] >= R.n_primes)
        throw HegpuError{HEGPU_E_ARG, "prime index out of range"};
    ntt_from_signed(R, src, src_stride, out, out_stride, n_polys, k, primes, S_(stream));
  })
}

int hegpu_pcg64_uniform(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                        const uint64_t* bounds, int k, int n, uint64_t* out,
                        int64_t out_stride, long long* consumed, void* stream) {
  HEGPU_TRY(*consumed = pcg64_uniform_fill(state_hi, state_lo, inc_hi, inc_lo, bounds, k, n, out,
                                           out_stride, S_(stream)))
}

int hegpu_sample_encrypt(int64_t* out, int n, uint64_t seed, double sigma, void* stream) {
  HEGPU_TRY(sample_encrypt(out, n, seed, sigma, S_(stream)))
}

int hegpu_encode_overflow(hegpu_ring_t ring, int* flag) {
  HEGPU_TRY({
    Ring& R = RR(ring);
    *flag = encode_overflow_check(R) ? 1 : 0;
  })
}

int hegpu_automorphism(hegpu_ring_t ring, int eval_form, uint64_t g, const uint64_t* in,
                       int64_t in_stride, uint64_t* out, int64_t out_stride, int n_polys, int k,
                       const int32_t* primes, void* stream) {
  HEGPU_TRY({
    Ring& R = RR(ring);
    if (in == out) throw HegpuError{HEGPU_E_ARG, "automorphism cannot run in place"};
    launch_automorphism(R.dpc, R.log_n, eval_form != 0, g, in, in_stride, out, out_stride,
                        n_polys, k, primes, S_(stream));
  })
}

int hegpu_tensor(hegpu_ring_t ring, const uint64_t* a0, const uint64_t* a1, int64_t a_stride,
                 const uint64_t* b0, const uint64_t* b1, int64_t b_stride, uint64_t* d0,
                 uint64_t* d1, uint64_t* d2, int64_t d_stride, int n_polys, int k,
                 void* stream) {
  return hegpu_tensor_periodic(ring, a0, a1, a_stride, n_polys, b0, b1, b_stride, d0, d1, d2,
                               d_stride, n_polys, k, stream);
}

int hegpu_tensor_periodic(hegpu_ring_t ring, const uint64_t* a0, const uint64_t* a1,
                          int64_t a_stride, int a_period, const uint64_t* b0, const uint64_t* b1,
                          int64_t b_stride, uint64_t* d0, uint64_t* d1, uint64_t* d2,
                          int64_t d_stride, int n_polys, int k, void* stream) {
  HEGPU_TRY({
    Ring& R = RR(ring);
    if (k > R.n_chain) throw HegpuError{HEGPU_E_ARG, "too many limbs"};
    if (a_period < 1) throw HegpuError{HEGPU_E_ARG, "a_period must be >= 1"};
    TensorParams T;
    T.amod = a_period;
    T.a0 = a0;
    T.a1 = a1;
    T.b0 = b0;
    T.b1 = b1;
    T.d0 = d0;
    T.d1 = d1;
    T.d2 = d2;
    T.as = a_stride;
    T.bs = b_stride;
    T.ds = d_stride;
    T.k = k;
    launch_tensor(R.dpc, R.log_n, T, n_polys, S_(stream));
  })
}

int hegpu_ks_apply(hegpu_ring_t ring, int level, int alpha, const uint64_t* d, int64_t d_stride,
                   int n_batch, const uint64_t* const* key_b, const uint64_t* const* key_a,
                   int n_digits, uint64_t* out_b, uint64_t* out_a, int64_t out_stride,
                   int accumulate, void* stream) {
  HEGPU_TRY({
    Ring& R = RR(ring);
    ks_apply_impl(R, level, alpha, d, d_stride, n_batch, key_b, key_a, n_digits, out_b, out_a,
                  out_stride, S_(stream), (accumulate & 1) != 0, (accumulate & 2) != 0);
  })
}

int hegpu_ks_apply_rescale(hegpu_ring_t ring, int level, int alpha, const uint64_t* d,
                           int64_t d_stride, int n_batch, const uint64_t* const* key_b,
                           const uint64_t* const* key_a, int n_digits, uint64_t* in,
                           int64_t in_stride, int64_t in_c1_off, uint64_t* out,
                           int64_t out_stride, int64_t out_c1_off, void* stream) {
  HEGPU_TRY({
    Ring& R = RR(ring);
    ks_apply_rescale_impl(R, level, alpha, d, d_stride, n_batch, key_b, key_a, n_digits, in,
                          in_stride, in_c1_off, out, out_stride, out_c1_off, S_(stream));
  })
}

int hegpu_ks_rotsum(hegpu_ring_t ring, int level, int alpha, const uint64_t* c, int64_t cs,
                    int64_t c1_off, int n_batch, int n_rot, const uint64_t* galois,
                    const uint64_t* const* key_b, const uint64_t* const* key_a, int n_digits,
                    uint64_t* out, int64_t out_stride, int64_t out_c1_off, void* stream) {
  HEGPU_TRY({
    Ring& R = RR(ring);
    if (out == c) throw HegpuError{HEGPU_E_ARG, "rotsum output may not alias the input"};
    ks_rotsum_impl(R, level, alpha, c, cs, c1_off, n_batch, n_rot, galois, key_b, key_a,
                   n_digits, out, out_stride, out_c1_off, S_(stream));
  })
}

int hegpu_ks_hoisted(hegpu_ring_t ring, int level, int alpha, const uint64_t* c, int64_t cs,
                     int64_t c1_off, int n_batch, int n_rot, const uint64_t* galois,
                     const uint64_t* const* key_b, const uint64_t* const* key_a, int n_digits,
                     uint64_t* const* outs, int pq_out, void* stream) {
  HEGPU_TRY({
    Ring& R = RR(ring);
    ks_hoisted_impl(R, level, alpha, c, cs, c1_off, n_batch, n_rot, galois, key_b, key_a,
                    n_digits, outs, S_(stream), pq_out != 0);
  })
}

int hegpu_bsgs_giants(hegpu_ring_t ring, int level, int alpha, const uint64_t* partials,
                      int64_t gstride, int n_batch, int n_giants, const uint64_t* galois,
                      const uint64_t* const* key_b, const uint64_t* const* key_a, int n_digits,
                      uint64_t* out, int rescale, int pq_in, void* stream) {
  HEGPU_TRY({
    Ring& R = RR(ring);
    if (pq_in) {
      if (!rescale) throw HegpuError{HEGPU_E_ARG, "extended-basis giants need rescale = 1"};
      bsgs_giants_sum_pq(R, level, alpha, const_cast<uint64_t*>(partials), gstride, n_batch,
                         n_giants, galois, key_b, key_a, n_digits, out, S_(stream), pq_in == 2);
      return HEGPU_OK;
    }
    bsgs_giants_impl(R, level, alpha, partials, gstride, n_batch, n_giants, galois, key_b, key_a,
                     n_digits, out, S_(stream), rescale != 0);
  })
}

int hegpu_set_allocator(hegpu_alloc_fn alloc, hegpu_free_fn free_fn) {
  HEGPU_TRY({
    if ((alloc == nullptr) != (free_fn == nullptr))
      throw HegpuError{HEGPU_E_ARG, "allocator needs both alloc and free (or neither)"};
    g_alloc = alloc;
    g_free = free_fn;
  })
}

int hegpu_moddown_rescale_ext(hegpu_ring_t ring, int level, int alpha, uint64_t* in,
                              int n_batch, uint64_t* out, void* stream) {
  HEGPU_TRY({
    Ring& R = RR(ring);
    if (n_batch <= 0) return HEGPU_OK;
    const KsLevel& L = R.ks_level(level, alpha);
    Scratch corr((size_t)n_batch * 2 * level * R.n * 8, S_(stream));
    ks_moddown_rescale(R, L, in, corr.u64(), n_batch, nullptr, 0, 0, out,
                       (int64_t)2 * level * R.n, (int64_t)level * R.n, S_(stream));
  })
}

int hegpu_rescale(hegpu_ring_t ring, int level, const uint64_t* in, int64_t in_stride,
                  uint64_t* out, int64_t out_stride, int n_polys, void* stream) {
  HEGPU_TRY({
    Ring& R = RR(ring);
    rescale_impl(R, level, in, in_stride, out, out_stride, n_polys, S_(stream));
  })
}

int hegpu_mod_raise(hegpu_ring_t ring, const uint64_t* in, int64_t in_stride, uint64_t* out,
                    int64_t out_stride, int n_polys, int to_level, void* stream) {
  HEGPU_TRY({
    Ring& R = RR(ring);
    mod_raise_impl(R, in, in_stride, out, out_stride, n_polys, to_level, S_(stream));
  })
}

int hegpu_encrypt_combine(hegpu_ring_t ring, const uint64_t* v, const uint64_t* e0,
                          const uint64_t* e1, const uint64_t* m, const uint64_t* pk_b,
                          const uint64_t* pk_a, uint64_t* c0, uint64_t* c1, int k,
                          void* stream) {
  HEGPU_TRY({
    Ring& R = RR(ring);
    if (k > R.n_chain) throw HegpuError{HEGPU_E_ARG, "too many limbs"};
    EncParams E;
    E.v = v;
    E.e0 = e0;
    E.e1 = e1;
    E.m = m;
    E.pb = pk_b;
    E.pa = pk_a;
    E.c0 = c0;
    E.c1 = c1;
    launch_encrypt(R.dpc, R.log_n, E, k, S_(stream));
  })
}

int hegpu_diag_mac(hegpu_ring_t ring, const uint64_t* const* ct_ptrs, int64_t ct_c1_off,
                   int64_t ct_bstride, const uint64_t* const* pt_ptrs, int n_terms,
                   int n_batch, uint64_t* out, int64_t out_c1_off, int64_t out_bstride, int k,
                   int accumulate, void* stream) {
  HEGPU_TRY({
    Ring& R = RR(ring);
    if (k > R.n_chain) throw HegpuError{HEGPU_E_ARG, "too many limbs"};
    launch_diag_mac(R.dpc, R.log_n, ct_ptrs, ct_c1_off, ct_bstride, pt_ptrs, n_terms, n_batch,
                    out, out_c1_off, out_bstride, k, accumulate, S_(stream));
  })
}

int hegpu_bsgs(hegpu_ring_t ring, const uint64_t* const* babies, int n_terms, int64_t c1_off,
               int64_t bstride, int n_batch, const uint64_t* pt_base, int64_t pt_stride,
               int pt_log_run, const int32_t* pt_idx, int n_giants, uint64_t* out,
               int64_t out_gstride, int k, int n_special_rows, void* stream) {
  HEGPU_TRY({
    Ring& R = RR(ring);
    if (n_special_rows < 0 || n_special_rows > R.n_special)
      throw HegpuError{HEGPU_E_ARG, "bad special row count"};
    if (k - n_special_rows > R.n_chain || k <= n_special_rows)
      throw HegpuError{HEGPU_E_ARG, "too many limbs"};
    launch_bsgs(R.dpc, R.log_n, babies, n_terms, c1_off, bstride, n_batch, pt_base, pt_stride,
                pt_log_run, pt_idx, n_giants, out, out_gstride, k, S_(stream),
                k - n_special_rows, R.n_chain);
  })
}

// --- host-array kernel table -----------------------------------------------

int hegpu_k_ntt_forward_inplace(uint64_t* a, int k, int n, const uint64_t* psi_rev,
                                const uint64_t* q, const uint64_t* qinv) {
  (void)qinv;
  HEGPU_TRY(shim_ntt(false, a, k, n, psi_rev, nullptr, q))
}

int hegpu_k_ntt_inverse_inplace(uint64_t* a, int k, int n, const uint64_t* ipsi_rev,
                                const uint64_t* ninv, const uint64_t* q, const uint64_t* qinv) {
  (void)qinv;
  HEGPU_TRY(shim_ntt(true, a, k, n, ipsi_rev, ninv, q))
}

int hegpu_k_elementwise_mont(const uint64_t* a, const uint64_t* b, uint64_t* out, int k, int n,
                             const uint64_t* q, const uint64_t* qinv) {
  (void)qinv;
  HEGPU_TRY(shim_elementwise(HEGPU_OP_MONT, a, b, out, k, n, q, nullptr))
}

int hegpu_k_elementwise_mulmod(const uint64_t* a, const uint64_t* b, uint64_t* out, int k,
                               int n, const uint64_t* q, const uint64_t* qinv,
                               const uint64_t* r2) {
  (void)qinv;
  (void)r2;
  HEGPU_TRY(shim_elementwise(HEGPU_OP_MUL, a, b, out, k, n, q, nullptr))
}

int hegpu_k_rowwise_mont(const uint64_t* a, const uint64_t* c, uint64_t* out, int k, int n,
                         const uint64_t* q, const uint64_t* qinv) {
  (void)qinv;
  HEGPU_TRY(shim_elementwise(HEGPU_OP_ROWMONT, a, nullptr, out, k, n, q, c))
}

int hegpu_k_addmod_rows(const uint64_t* a, const uint64_t* b, uint64_t* out, int k, int n,
                        const uint64_t* q) {
  HEGPU_TRY(shim_elementwise(HEGPU_OP_ADD, a, b, out, k, n, q, nullptr))
}

int hegpu_k_submod_rows(const uint64_t* a, const uint64_t* b, uint64_t* out, int k, int n,
                        const uint64_t* q) {
  HEGPU_TRY(shim_elementwise(HEGPU_OP_SUB, a, b, out, k, n, q, nullptr))
}

int hegpu_k_fma_inplace(uint64_t* acc, const uint64_t* a, const uint64_t* b, int k, int n,
                        const uint64_t* q, const uint64_t* qinv, const uint64_t* r2) {
  (void)qinv;
  (void)r2;
  HEGPU_TRY(shim_elementwise(HEGPU_OP_FMA, a, b, acc, k, n, q, nullptr))
}

int hegpu_k_fma_gather_inplace(uint64_t* acc, const uint64_t* a, const uint64_t* key,
                               int key_rows, const int64_t* rows, int k, int n,
                               const uint64_t* q, const uint64_t* qinv, const uint64_t* r2) {
  (void)qinv;
  (void)r2;
  HEGPU_TRY({
    std::vector<uint64_t> gathered((size_t)k * n);
    for (int i = 0; i < k; ++i) {
      if (rows[i] < 0 || rows[i] >= key_rows) throw HegpuError{HEGPU_E_ARG, "key row out of range"};
      std::memcpy(gathered.data() + (size_t)i * n, key + (size_t)rows[i] * n, (size_t)n * 8);
    }
    shim_elementwise(HEGPU_OP_FMA, a, gathered.data(), acc, k, n, q, nullptr);
  })
}

int hegpu_k_base_convert(const uint64_t* hat, int l, int n, const uint64_t* punc, int kt,
                         const uint64_t* q_to, const uint64_t* qinv_to, uint64_t* out) {
  (void)qinv_to;
  HEGPU_TRY({
    if (kt == 0 || n == 0) return HEGPU_OK;
    const int log_n = ilog2_exact(n);
    if (l > 32) throw HegpuError{HEGPU_E_ARG, "too many source rows"};
    auto pc = shim_consts(q_to, kt, log_n);
    DevBuf dpc(pc.size() * sizeof(PrimeConst)), dh((size_t)std::max(l, 1) * n * 8),
        dp((size_t)std::max(l * kt, 1) * 8), dout((size_t)kt * n * 8);
    h2d(dpc.p, pc.data(), pc.size() * sizeof(PrimeConst));
    if (l) h2d(dh.p, hat, (size_t)l * n * 8);
    if (l) h2d(dp.p, punc, (size_t)l * kt * 8);
    ConvParams C;
    C.n_jobs = 1;
    C.n_polys = 1;
    C.log_n = log_n;
    C.pc = static_cast<PrimeConst*>(dpc.p);
    ConvJob& J = C.job[0];
    J.src = dh.u64();
    J.src_stride = 0;
    J.dst = dout.u64();
    J.dst_stride = 0;
    J.n_src = l;
    J.n_dst = kt;
    J.inv = nullptr;
    J.inv_sh = nullptr;
    J.punc = dp.u64();
    J.punc_ld = kt;
    for (int i = 0; i < l; ++i) C.src_sel[0][i] = 0;  // hat rows are used as given
    for (int t = 0; t < kt; ++t) C.dst_sel[0][t] = (uint8_t)t;
    launch_conv(C, 0);
    d2h(out, dout.p, (size_t)kt * n * 8);
  })
}

}  // extern "C"
