// TMA-staged evaluation-key streaming fused with the key-switch inner product
// (keys.py:299-323 / fma_gather_inplace, _kernels.py:271-286; rotation form
// keys.py:316-323 + ring.py:471-482).
//
// Persistent CTAs, one per SM.  A producer warp (one elected lane) streams,
// per (row, 512-coefficient tile, batch group, rotation) stage:
//   * the key tiles of all digits with ONE 3-D tensor-map load each for b and
//     a (cp.async.bulk.tensor: box {512 coeffs, 1 row, beta digits} of the
//     (dnum, L+1+K, N) key tensor), and
//   * the digit tiles of the batch group with 1-D bulk copies (the digits are
//     read through X -> X^g: the 512 outputs of a tile gather from ONE aligned
//     512-slot source block, so the whole source block is staged and the
//     permutation is applied in shared memory),
// into a ring of kStages shared-memory stages guarded by full/empty mbarriers.
// Sixteen consumer warps multiply-accumulate in 128 bits (Mac128) and write the
// outputs; they never wait on global loads.
//
// The same kernel serves the plain key switch (one rotation, g = 1).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "ring.cuh"

namespace hegpu {

namespace {

constexpr int kBox = 256;  // TMA box extent limit per dimension

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

}  // namespace

struct IpRotTmaParams {
  IpRotParams P;
  // key tensor (dnum, L+1+K, N) viewed 4-D as {256, N/256, rows, dnum} u64,
  // box {256, kTile/256, 1, beta}: one load lands [beta][kTile] in smem
  CUtensorMap kmap_b[kMaxRot];
  CUtensorMap kmap_a[kMaxRot];
  int n_tiles, n_groups;
  long long n_work;
};

// Source index of output slot i under X -> X^g (see k_auto_eval).
__device__ __forceinline__ uint32_t tma_auto_src(uint32_t i, uint32_t g, int log_n) {
  const uint32_t mask2n = (2u << log_n) - 1u;
  const uint32_t bi = __brev(i) >> (32 - log_n);
  const uint32_t e = (uint32_t)(((uint64_t)(2u * bi + 1u) * g) & mask2n);
  return __brev((e - 1u) >> 1) >> (32 - log_n);
}

// TILE coefficients per stage (one per consumer thread, TILE/32 consumer
// warps + 1 producer warp), BG batch elements per thread, CPS CTAs per SM.
template <int TILE, int BG, int BETA, int STAGES, int CPS>
__global__ void __launch_bounds__(TILE + 32, CPS)
    k_ks_ip_rot_tma(const __grid_constant__ IpRotTmaParams T) {
  constexpr int kTile = TILE;
  constexpr int kConsumerWarps = TILE / 32;
  const IpRotParams& P = T.P;
  constexpr int kStageWords = (2 * BETA + BETA * BG) * kTile;
  extern __shared__ __align__(1024) uint64_t smem[];
  uint64_t* full = smem + STAGES * kStageWords;
  uint64_t* empty = full + STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int N = 1 << P.log_n;
  const int beta = P.beta;
  const int n_tiles = T.n_tiles, n_groups = T.n_groups;

  if (warp == kConsumerWarps) {
    // ---------------- producer: one elected lane streams every stage --------
    if (lane == 0) {
      uint32_t k = 0;
      for (long long w = blockIdx.x; w < T.n_work; w += gridDim.x) {
        const int g = (int)(w % n_groups);
        const long long rt = w / n_groups;
        const int t = (int)(rt % n_tiles);
        const int r = (int)(rt / n_tiles);
        const int b0 = g * BG;
        const int nb = min(BG, P.n_batch - b0);
        const int krow = r <= P.level ? r : P.key_sp_row0 + (r - P.level - 1);
        const uint32_t bytes = (uint32_t)((2 * beta + beta * nb) * kTile * 8);
        for (int rot = 0; rot < P.n_rot; ++rot, ++k) {
          const int s = k % STAGES;
          mbar_wait(empty + s, ((k / STAGES) & 1) ^ 1);
          uint64_t* st = smem + (size_t)s * kStageWords;
          mbar_expect_tx(full + s, bytes);
          tma_load_4d(st, &T.kmap_b[rot], 0, t * (kTile / kBox), krow, 0, full + s);
          tma_load_4d(st + BETA * kTile, &T.kmap_a[rot], 0, t * (kTile / kBox), krow, 0, full + s);
          const uint32_t blk = tma_auto_src((uint32_t)(t * kTile), P.gal[rot], P.log_n) &
                               ~(uint32_t)(kTile - 1);
          uint64_t* vs = st + 2 * BETA * kTile;
          for (int j = 0; j < beta; ++j) {
            const int g0 = j * P.alpha;
            const int g1 = min(g0 + P.alpha, P.level + 1);
            const uint64_t* src;
            int64_t bstr;
            if (r >= g0 && r < g1) {
              src = P.d + (size_t)r * N + (size_t)b0 * P.ds + rot * P.d_sr;
              bstr = P.ds;
            } else {
              src = P.ext + j * P.ext_sj + (size_t)(r < g0 ? r : r - (g1 - g0)) * N +
                    (size_t)b0 * P.ext_sb + rot * P.ext_sr;
              bstr = P.ext_sb;
            }
            for (int b = 0; b < nb; ++b)
              bulk_g2s(vs + (size_t)(j * BG + b) * kTile, src + (size_t)b * bstr + blk,
                       kTile * 8, full + s);
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers: 512 threads, one coefficient each ------------
  const int tid = threadIdx.x;
  uint32_t k = 0;
  for (long long w = blockIdx.x; w < T.n_work; w += gridDim.x) {
    const int g = (int)(w % n_groups);
    const long long rt = w / n_groups;
    const int t = (int)(rt % n_tiles);
    const int r = (int)(rt / n_tiles);
    const int b0 = g * BG;
    const int nb = min(BG, P.n_batch - b0);
    const int prime = r <= P.level ? r : P.n_chain + (r - P.level - 1);
    const PrimeConst pc = P.pc[prime];
    const int x = t * kTile + tid;
    Mac128 ab[BG], aa[BG];
#pragma unroll
    for (int b = 0; b < BG; ++b) {
      ab[b].zero();
      aa[b].zero();
    }
    int since = 0;
    for (int rot = 0; rot < P.n_rot; ++rot, ++k) {
      const int s = k % STAGES;
      const uint32_t src = tma_auto_src((uint32_t)x, P.gal[rot], P.log_n);
      const int so = (int)(src & (kTile - 1));
      mbar_wait(full + s, (k / STAGES) & 1);
      const uint64_t* st = smem + (size_t)s * kStageWords;
      const uint64_t* vs = st + 2 * BETA * kTile;
#pragma unroll
      for (int j = 0; j < BETA; ++j) {
        if (j < beta) {
          const uint64_t kb = st[j * kTile + tid];
          const uint64_t ka = st[(BETA + j) * kTile + tid];
#pragma unroll
          for (int b = 0; b < BG; ++b) {
            const uint64_t v = b < nb ? vs[(j * BG + b) * kTile + so] : 0;
            ab[b].add(v, kb);
            aa[b].add(v, ka);
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
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + s);  // this warp is done with the stage
      if (!P.sum_mode || rot == P.n_rot - 1) {
        uint64_t* o = P.acc + (P.sum_mode ? 0 : rot * P.acc_sr) + (size_t)r * N + x;
#pragma unroll
        for (int b = 0; b < BG; ++b) {
          if (b < nb) {
            uint64_t* ob = o + (size_t)(b0 + b) * P.acc_sb;
            uint64_t vb = mont_mul(ab[b].redc(pc), pc.r2, pc.q, pc.qinv_neg);
            uint64_t va = mont_mul(aa[b].redc(pc), pc.r2, pc.q, pc.qinv_neg);
            if (P.c0 && r <= P.level)
              vb = add_mod(vb,
                           shoup(__ldg(P.c0 + (size_t)(b0 + b) * P.c0s + (size_t)r * N + src),
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
}

// --------------------------------------------------------------------------
// host side
// --------------------------------------------------------------------------

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// (dnum, rows, N) u64 key tensor at `base` as 4-D {256, N/256, rows, dnum},
// box {256, kTile/256, 1, beta}
static bool encode_key_map(CUtensorMap* m, const uint64_t* base, int log_n, int rows, int dnum,
                           int beta, int kTile) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t n = 1ull << log_n;
  cuuint64_t dims[4] = {(cuuint64_t)kBox, n / kBox, (cuuint64_t)rows, (cuuint64_t)dnum};
  cuuint64_t strides[3] = {kBox * 8, n * 8, n * 8 * (cuuint64_t)rows};
  cuuint32_t box[4] = {(cuuint32_t)kBox, (cuuint32_t)(kTile / kBox), 1, (cuuint32_t)beta};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, const_cast<uint64_t*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

static bool g_tma_disabled() {
  static const bool off = [] {
    const char* e = getenv("HEGPU_NO_TMA");
    return e && e[0] == '1';
  }();
  return off;
}

template <int TILE, int BG, int BETA, int STAGES, int CPS>
static void launch_tma(IpRotTmaParams& T, cudaStream_t st) {
  constexpr size_t smem =
      (size_t)STAGES * (2 * BETA + BETA * BG) * TILE * 8 + 2 * STAGES * sizeof(uint64_t);
  static bool configured = false;
  if (!configured) {
    check_cuda(cudaFuncSetAttribute(k_ks_ip_rot_tma<TILE, BG, BETA, STAGES, CPS>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "ks tma smem attribute");
    configured = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long slots = (long long)sms * CPS;
  const long long grid = T.n_work < slots ? T.n_work : slots;
  k_ks_ip_rot_tma<TILE, BG, BETA, STAGES, CPS><<<(int)grid, TILE + 32, smem, st>>>(T);
}

// configuration (experiments: HEGPU_TMA_CFG = 0..4)
static int g_tma_cfg() {
  static const int cfg = [] {
    const char* e = getenv("HEGPU_TMA_CFG");
    return e ? atoi(e) : 0;
  }();
  return cfg;
}

template <int BETA>
static void dispatch_tma(IpRotTmaParams& T, int bgmax, cudaStream_t st) {
  const int cfg = g_tma_cfg();
  const int nb = T.P.n_batch;
  switch (cfg) {
    case 1:  // 512-tile, up to 4 batch per thread, 2 stages
      if (nb >= 4) return launch_tma<512, 4, BETA, 2, 1>(T, st);
      if (nb >= 2) return launch_tma<512, 2, BETA, 3, 1>(T, st);
      return launch_tma<512, 1, BETA, 3, 1>(T, st);
    case 2:  // 256-tile, 2 CTAs / SM
      if (nb >= 4) return launch_tma<256, 4, BETA, 2, 2>(T, st);
      if (nb >= 2) return launch_tma<256, 2, BETA, 3, 2>(T, st);
      return launch_tma<256, 1, BETA, 4, 2>(T, st);
    case 3:  // 256-tile, 1 CTA / SM, deep ring
      if (nb >= 4) return launch_tma<256, 4, BETA, 4, 1>(T, st);
      if (nb >= 2) return launch_tma<256, 2, BETA, 6, 1>(T, st);
      return launch_tma<256, 1, BETA, 8, 1>(T, st);
    default:  // 512-tile, up to 2 batch per thread
      if (nb >= 2) return launch_tma<512, 2, BETA, 3, 1>(T, st);
      return launch_tma<512, 1, BETA, 3, 1>(T, st);
  }
}

static int tma_bg(int cfg, int nb) {
  if (cfg == 1 || cfg == 2 || cfg == 3) return nb >= 4 ? 4 : nb >= 2 ? 2 : 1;
  return nb >= 2 ? 2 : 1;
}

static int tma_tile(int cfg) { return (cfg == 2 || cfg == 3) ? 256 : 512; }

// Returns false when the TMA path does not apply (the caller falls back to
// the register-staged kernel): disabled, N < 512, more than 4 digits, or key
// digits that are not one (dnum, L+1+K, N) tensor.
bool launch_ks_ip_rot_tma(const IpRotParams& P, cudaStream_t st) {
  if (g_tma_disabled() || P.log_n < 10 || P.beta > 4 || P.n_rot < 1 || P.n_rot > kMaxRot)
    return false;
  // Multi-rotation gathers stay on the register-staged kernel: measured on
  // the B200 (tools/microbench.py ip, profiles/r02_ks_tma_variants.txt) the
  // staged ring is 10-25% slower there and 10-20% faster for one rotation.
  if (P.n_rot > 1 && !getenv("HEGPU_TMA_ROT")) return false;
  const int K = P.n_ext - P.level - 1;
  const int rows = P.n_chain + K;
  const size_t N = (size_t)1 << P.log_n;
  for (int r = 0; r < P.n_rot; ++r)
    for (int j = 1; j < P.beta; ++j)
      if (P.kb[r][j] != P.kb[r][0] + (size_t)j * rows * N ||
          P.ka[r][j] != P.ka[r][0] + (size_t)j * rows * N)
        return false;
  static thread_local IpRotTmaParams T;  // large: keep it off the stack
  T.P = P;
  const int cfg = g_tma_cfg();
  const int tile = tma_tile(cfg);
  for (int r = 0; r < P.n_rot; ++r) {
    // the tensor spans the digits this launch uses (beta <= dnum)
    if (!encode_key_map(&T.kmap_b[r], P.kb[r][0], P.log_n, rows, P.beta, P.beta, tile) ||
        !encode_key_map(&T.kmap_a[r], P.ka[r][0], P.log_n, rows, P.beta, P.beta, tile))
      throw HegpuError{HEGPU_E_CUDA, "cuTensorMapEncodeTiled failed for a key tensor"};
  }
  const int bg = tma_bg(cfg, P.n_batch);
  T.n_tiles = (int)(N / tile);
  T.n_groups = (P.n_batch + bg - 1) / bg;
  T.n_work = (long long)P.n_ext * T.n_tiles * T.n_groups;
  if (P.beta <= 2)
    dispatch_tma<2>(T, bg, st);
  else
    dispatch_tma<4>(T, bg, st);
  check_cuda(cudaGetLastError(), "ks tma inner product launch");
  return true;
}

}  // namespace hegpu
