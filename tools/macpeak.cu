// Throughput probe: 128-bit multiply-accumulate variants, register-resident.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o macpeak tools/macpeak.cu
#include <cstdint>
#include <cstdio>
#include "../paper_2210_02574_b200/csrc/common.cuh"
using namespace hegpu;

template <int ACC>
__global__ void k_mac(uint64_t* out, uint64_t seed, int iters) {
  Mac128 a[ACC];
  for (int i = 0; i < ACC; ++i) a[i].zero();
  uint64_t x = seed ^ threadIdx.x, y = seed * 3 + blockIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) a[i].add(x + i, y);
    x += 0x9e3779b97f4a7c15ull;
  }
  uint64_t r = 0;
  for (int i = 0; i < ACC; ++i) r ^= a[i].L ^ a[i].H ^ a[i].M ^ a[i].c;
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

__global__ void k_imad(uint64_t* out, uint32_t seed, int iters) {
  uint64_t a[16];
  for (int i = 0; i < 16; ++i) a[i] = seed + i;
  uint32_t x = seed ^ threadIdx.x, y = seed * 3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = (uint64_t)x * (uint64_t)(y + i) + a[i];
    x += 7;
  }
  uint64_t r = 0;
  for (int i = 0; i < 16; ++i) r ^= a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
  uint64_t* d;
  cudaMalloc(&d, 148 * 8 * 1024 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int threads : {256, 512}) {
    for (int blocks : {148 * 4, 148 * 8}) {
      k_mac<8><<<blocks, threads>>>(d, 1, iters);
      cudaEventRecord(e0);
      k_mac<8><<<blocks, threads>>>(d, 1, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double macs = (double)blocks * threads * iters * 8;
      printf("mac128 acc=8 thr=%d blocks=%d: %.3f T mac/s\n", threads, blocks, macs / ms / 1e9);
      k_imad<<<blocks, threads>>>(d, 1, iters);
      cudaEventRecord(e0);
      k_imad<<<blocks, threads>>>(d, 1, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * threads * iters * 16;
      printf("imad.wide thr=%d blocks=%d: %.3f T op/s (%.1f per SM per clk @1.965GHz)\n", threads,
             blocks, ops / ms / 1e9, ops / ms / 1e9 * 1e12 / 148 / 1.965e9);
    }
  }
  return 0;
}
