// Throughput probe: FP64 pipe vs the 64-bit integer Shoup modmul on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fpmodpeak tools/fpmodpeak.cu
//
// fp modmul (q < 2^50, operands are integers held in doubles, |a| < 2^52):
//   h = a*w; l = fma(a,w,-h)         exact product h + l
//   t = rint(a * (w/q))              quotient estimate (magic-constant rint)
//   r = fma(-t, q, h) + l            exact, in (-q, q)
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>

__device__ __forceinline__ double fmodmul(double a, double w, double wq, double q) {
  const double M = 6755399441055744.0;  // 1.5 * 2^52
  double h = a * w;
  double l = fma(a, w, -h);
  double t = fma(a, wq, M) - M;
  double r = fma(-t, q, h);
  return r + l;
}

__global__ void k_dfma(double* out, double seed, int iters) {
  double a[16];
  for (int i = 0; i < 16; ++i) a[i] = seed + i + threadIdx.x;
  double x = 1.0000001, y = 0.9999999;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], x, y);
  }
  double r = 0;
  for (int i = 0; i < 16; ++i) r += a[i];
  if (r == 1.2345) out[0] = r;
}

__global__ void k_fmod(double* out, double w, double wq, double q, int iters) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = (double)((threadIdx.x * 8 + c + blockIdx.x) % 100000);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fmodmul(x[c], w, wq, q);
  }
  double acc = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) acc += x[c];
  if (acc == 0.5) out[0] = acc;
}

__global__ void k_shoup(uint64_t* out, uint64_t q, uint64_t w, uint64_t wsh, int iters) {
  uint64_t x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = (threadIdx.x * 8 + c + blockIdx.x) % q;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = x[c] * w - __umul64hi(x[c], wsh) * q;
  }
  uint64_t acc = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) acc ^= x[c];
  if (acc == 0x123456789ull) out[0] = acc;
}

// correctness: random a in (-q, q), w in [0, q)
__global__ void k_check(const double* a, const double* w, const double* wq, double q,
                        uint64_t qi, int n, int* bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double r = fmodmul(a[i], w[i], wq[i], q);
  if (!(r > -q && r < q)) { atomicAdd(bad, 1); return; }
  __int128 ai = (__int128)(int64_t)a[i];
  __int128 p = ai * (__int128)(int64_t)w[i];
  int64_t m = (int64_t)(p % (__int128)qi);
  int64_t rr = (int64_t)r;
  int64_t d = (rr - m) % (int64_t)qi;
  if (d != 0) atomicAdd(bad, 1);
}

int main() {
  double* d;
  cudaMalloc(&d, 64);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096, blocks = 148 * 8, threads = 256;
  float ms;
  k_dfma<<<blocks, threads>>>(d, 1, 16);
  cudaEventRecord(e0);
  k_dfma<<<blocks, threads>>>(d, 1, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)blocks * threads * iters * 16;
  printf("dfma: %.3f T/s (%.1f per SM per clk @1.965GHz)\n", ops / ms / 1e9,
         ops / ms / 1e9 * 1e12 / 148 / 1.965e9);

  const uint64_t qi = 0xffffe80001ull;  // 40-bit chain prime
  const double q = (double)qi;
  const uint64_t wi = 0x123456789ull % qi;
  const double w = (double)wi, wq = w / q;
  k_fmod<<<blocks, threads>>>(d, w, wq, q, 16);
  cudaEventRecord(e0);
  k_fmod<<<blocks, threads>>>(d, w, wq, q, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  ops = (double)blocks * threads * iters * 8;
  printf("fp64 modmul: %.3f T/s (%.2f per SM per clk)\n", ops / ms / 1e9,
         ops / ms / 1e9 * 1e12 / 148 / 1.965e9);

  uint64_t* du;
  cudaMalloc(&du, 64);
  const uint64_t q60 = 0xffffffffffc0001ull, w60 = 0x123456789abcdull % q60;
  const uint64_t wsh = (uint64_t)(((unsigned __int128)w60 << 64) / q60);
  k_shoup<<<blocks, threads>>>(du, q60, w60, wsh, 16);
  cudaEventRecord(e0);
  k_shoup<<<blocks, threads>>>(du, q60, w60, wsh, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("int64 shoup modmul: %.3f T/s (%.2f per SM per clk)\n", ops / ms / 1e9,
         ops / ms / 1e9 * 1e12 / 148 / 1.965e9);

  // correctness on random operands, 40-, 45- and 50-bit primes
  const uint64_t primes[3] = {0xffffe80001ull, 0x1fffffc20001ull, 0x3ffffffd80001ull};
  const int n = 1 << 22;
  double *ha = (double*)malloc(n * 8), *hw = (double*)malloc(n * 8), *hq = (double*)malloc(n * 8);
  double *da, *dw, *dq;
  int* dbad;
  cudaMalloc(&da, n * 8);
  cudaMalloc(&dw, n * 8);
  cudaMalloc(&dq, n * 8);
  cudaMalloc(&dbad, 4);
  srand(1);
  for (uint64_t p : primes) {
    for (int i = 0; i < n; ++i) {
      uint64_t r1 = ((uint64_t)rand() << 42) ^ ((uint64_t)rand() << 21) ^ rand();
      uint64_t r2 = ((uint64_t)rand() << 42) ^ ((uint64_t)rand() << 21) ^ rand();
      int64_t av = (int64_t)(r1 % (2 * p - 1)) - (int64_t)(p - 1);
      if (i < 4) av = (i & 1) ? (int64_t)(p - 1) : -(int64_t)(p - 1);
      uint64_t wv = (i < 4) ? p - 1 : r2 % p;
      ha[i] = (double)av;
      hw[i] = (double)wv;
      hq[i] = (double)wv / (double)p;
    }
    cudaMemcpy(da, ha, n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dw, hw, n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dq, hq, n * 8, cudaMemcpyHostToDevice);
    cudaMemset(dbad, 0, 4);
    k_check<<<n / 256, 256>>>(da, dw, dq, (double)p, p, n, dbad);
    int bad = 0;
    cudaMemcpy(&bad, dbad, 4, cudaMemcpyDeviceToHost);
    printf("check q=%#llx (%d bits): %d bad of %d\n", (unsigned long long)p,
           64 - __builtin_clzll(p), bad, n);
  }
  return 0;
}
