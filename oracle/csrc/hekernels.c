/*
 * TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference kernel table
 * hebert/_kernels.py (numba path, _kernels.py:122-317), used by the oracle as
 * the parity checker and as the CPU baseline of bench.py.  Never linked into
 * the product.
 *
 * Each function follows the reference kernel line by line: Montgomery REDC
 * with R = 2^64 (_kernels.py:134-142), CT forward NTT with Montgomery-form
 * bit-reversed twiddles (:144-171), GS inverse with a final N^-1 pass
 * (:173-204), elementwise/rowwise products (:206-227, :288-298), add/sub
 * (:229-253), gathered FMA (:271-286) and fast basis conversion (:300-317).
 * Parallelism is OpenMP over limbs, like numba's prange over limbs.
 */
#include <stdint.h>
#include <string.h>

typedef unsigned __int128 u128;

static inline uint64_t mont(uint64_t a, uint64_t b, uint64_t q, uint64_t qinv) {
  u128 t = (u128)a * b;
  uint64_t t_lo = (uint64_t)t;
  uint64_t m = t_lo * qinv;
  uint64_t r = (uint64_t)(t >> 64) + (uint64_t)(((u128)m * q) >> 64) + (t_lo != 0);
  return r >= q ? r - q : r;
}

void ok_ntt_forward(uint64_t* a, int k, int n, const uint64_t* psi_rev, const uint64_t* qv,
                    const uint64_t* qinvv) {
#pragma omp parallel for schedule(static)
  for (int li = 0; li < k; ++li) {
    const uint64_t q = qv[li], qinv = qinvv[li];
    uint64_t* limb = a + (size_t)li * n;
    const uint64_t* psi = psi_rev + (size_t)li * n;
    int t = n;
    for (int m = 1; m < n; m <<= 1) {
      t >>= 1;
      for (int i = 0; i < m; ++i) {
        const uint64_t s = psi[m + i];
        const int j1 = 2 * i * t;
        for (int j = j1; j < j1 + t; ++j) {
          const uint64_t u = limb[j];
          const uint64_t v = mont(limb[j + t], s, q, qinv);
          uint64_t sm = u + v;
          if (sm >= q) sm -= q;
          uint64_t df = u + (q - v);
          if (df >= q) df -= q;
          limb[j] = sm;
          limb[j + t] = df;
        }
      }
    }
  }
}

void ok_ntt_inverse(uint64_t* a, int k, int n, const uint64_t* ipsi_rev, const uint64_t* ninvv,
                    const uint64_t* qv, const uint64_t* qinvv) {
#pragma omp parallel for schedule(static)
  for (int li = 0; li < k; ++li) {
    const uint64_t q = qv[li], qinv = qinvv[li];
    uint64_t* limb = a + (size_t)li * n;
    const uint64_t* ipsi = ipsi_rev + (size_t)li * n;
    int t = 1;
    for (int m = n; m > 1; m >>= 1) {
      const int h = m >> 1;
      for (int i = 0; i < h; ++i) {
        const uint64_t s = ipsi[h + i];
        const int j1 = 2 * i * t;
        for (int j = j1; j < j1 + t; ++j) {
          const uint64_t u = limb[j], v = limb[j + t];
          uint64_t sm = u + v;
          if (sm >= q) sm -= q;
          uint64_t df = u + (q - v);
          if (df >= q) df -= q;
          limb[j] = sm;
          limb[j + t] = mont(df, s, q, qinv);
        }
      }
      t <<= 1;
    }
    const uint64_t ninv = ninvv[li];
    for (int j = 0; j < n; ++j) limb[j] = mont(limb[j], ninv, q, qinv);
  }
}

void ok_mulmod(const uint64_t* a, const uint64_t* b, uint64_t* out, int k, int n,
               const uint64_t* qv, const uint64_t* qinvv, const uint64_t* r2v) {
#pragma omp parallel for schedule(static)
  for (int li = 0; li < k; ++li) {
    const uint64_t q = qv[li], qinv = qinvv[li], r2 = r2v[li];
    const size_t o = (size_t)li * n;
    for (int j = 0; j < n; ++j) out[o + j] = mont(mont(a[o + j], b[o + j], q, qinv), r2, q, qinv);
  }
}

void ok_mont(const uint64_t* a, const uint64_t* b, uint64_t* out, int k, int n,
             const uint64_t* qv, const uint64_t* qinvv) {
#pragma omp parallel for schedule(static)
  for (int li = 0; li < k; ++li) {
    const size_t o = (size_t)li * n;
    for (int j = 0; j < n; ++j) out[o + j] = mont(a[o + j], b[o + j], qv[li], qinvv[li]);
  }
}

void ok_rowwise(const uint64_t* a, const uint64_t* c, uint64_t* out, int k, int n,
                const uint64_t* qv, const uint64_t* qinvv) {
#pragma omp parallel for schedule(static)
  for (int li = 0; li < k; ++li) {
    const size_t o = (size_t)li * n;
    for (int j = 0; j < n; ++j) out[o + j] = mont(a[o + j], c[li], qv[li], qinvv[li]);
  }
}

void ok_addmod(const uint64_t* a, const uint64_t* b, uint64_t* out, int k, int n,
               const uint64_t* qv) {
#pragma omp parallel for schedule(static)
  for (int li = 0; li < k; ++li) {
    const uint64_t q = qv[li];
    const size_t o = (size_t)li * n;
    for (int j = 0; j < n; ++j) {
      uint64_t s = a[o + j] + b[o + j];
      out[o + j] = s >= q ? s - q : s;
    }
  }
}

void ok_submod(const uint64_t* a, const uint64_t* b, uint64_t* out, int k, int n,
               const uint64_t* qv) {
#pragma omp parallel for schedule(static)
  for (int li = 0; li < k; ++li) {
    const uint64_t q = qv[li];
    const size_t o = (size_t)li * n;
    for (int j = 0; j < n; ++j) {
      uint64_t s = a[o + j] + (q - b[o + j]);
      out[o + j] = s >= q ? s - q : s;
    }
  }
}

void ok_fma_gather(uint64_t* acc, const uint64_t* a, const uint64_t* key, const int64_t* rows,
                   int k, int n, const uint64_t* qv, const uint64_t* qinvv, const uint64_t* r2v) {
#pragma omp parallel for schedule(static)
  for (int li = 0; li < k; ++li) {
    const uint64_t q = qv[li], qinv = qinvv[li], r2 = r2v[li];
    const uint64_t* krow = key + (size_t)rows[li] * n;
    const size_t o = (size_t)li * n;
    for (int j = 0; j < n; ++j) {
      uint64_t v = mont(mont(a[o + j], krow[j], q, qinv), r2, q, qinv);
      uint64_t s = acc[o + j] + v;
      acc[o + j] = s >= q ? s - q : s;
    }
  }
}

void ok_base_convert(const uint64_t* hat, int l, int n, const uint64_t* punc, int kt,
                     const uint64_t* q_to, const uint64_t* qinv_to, uint64_t* out) {
#pragma omp parallel for schedule(static)
  for (int j = 0; j < kt; ++j) {
    const uint64_t q = q_to[j], qinv = qinv_to[j];
    uint64_t* row = out + (size_t)j * n;
    memset(row, 0, (size_t)n * 8);
    for (int i = 0; i < l; ++i) {
      const uint64_t c = punc[(size_t)i * kt + j];
      const uint64_t* src = hat + (size_t)i * n;
      for (int x = 0; x < n; ++x) {
        uint64_t s = row[x] + mont(src[x], c, q, qinv);
        row[x] = s >= q ? s - q : s;
      }
    }
  }
}
