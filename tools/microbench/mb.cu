// Microbenchmarks for design decisions: FP64 pipe rate, random L2/HBM gather and atomics.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void ffma_kernel(float* out, int iters, float a, float b) {
  float x0 = threadIdx.x * 1e-3f, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void imadhi_kernel(unsigned* out, int iters, unsigned m) {
  unsigned x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0+4, x5=x0+5, x6=x0+6, x7=x0+7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = __umulhi(x0, m) + x0; x1 = __umulhi(x1, m) + x1; x2 = __umulhi(x2, m) + x2; x3 = __umulhi(x3, m) + x3;
      x4 = __umulhi(x4, m) + x4; x5 = __umulhi(x5, m) + x5; x6 = __umulhi(x6, m) + x6; x7 = __umulhi(x7, m) + x7;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 ^ x1 ^ x2 ^ x3 ^ x4 ^ x5 ^ x6 ^ x7;
}
__global__ void gather_kernel(const uint32_t* __restrict__ tab, uint32_t mask, uint32_t* out, int iters) {
  uint32_t h = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
    uint32_t idx[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { h = h * 1664525u + 1013904223u; idx[k] = (h ^ (h >> 13)) & mask; }
#pragma unroll
    for (int k = 0; k < 8; ++k) acc += __ldg(tab + idx[k]);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void scatter_atomic_kernel(uint32_t* tab, uint32_t mask, int iters) {
  uint32_t h = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { h = h * 1664525u + 1013904223u; atomicMin(tab + ((h ^ (h >> 13)) & mask), h); }
  }
}
__global__ void scatter_store_kernel(uint32_t* tab, uint32_t mask, int iters) {
  uint32_t h = blockIdx.x * blockDim.x + threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { h = h * 1664525u + 1013904223u; tab[(h ^ (h >> 13)) & mask] = h; }
  }
}
__global__ void copy_kernel(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("dev %s SMs %d l2 %d MB smem/block optin %zu\n", p.name, p.multiProcessorCount, p.l2CacheSize >> 20, p.sharedMemPerBlockOptin);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  int sms = p.multiProcessorCount;
  double* dout; CK(cudaMalloc(&dout, 1 << 26));
  for (int rep = 0; rep < 3; ++rep) {
    int blocks = sms * 8, threads = 256, iters = 2000;
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(dout, iters, 0.999, 1e-3); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * iters * 16 * 8;
    printf("DFMA: %.3f ms  %.3f Tinst/s (%.1f TFLOP/s)  per SM per clk @1965: %.1f\n", ms, ops / ms / 1e9, 2 * ops / ms / 1e9, ops / (ms * 1e-3) / sms / 1.965e9);
    cudaEventRecord(e0); ffma_kernel<<<blocks, threads>>>((float*)dout, iters, 0.999f, 1e-3f); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA: %.3f ms  %.3f Tinst/s per SM per clk @1965: %.1f\n", ms, ops / ms / 1e9, ops / (ms * 1e-3) / sms / 1.965e9);
    cudaEventRecord(e0); imadhi_kernel<<<blocks, threads>>>((unsigned*)dout, iters, 0x9e3779b9u); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("IMAD.HI+IADD: %.3f ms  %.3f Tpairs/s per SM per clk @1965: %.1f\n", ms, ops / ms / 1e9, ops / (ms * 1e-3) / sms / 1.965e9);
  }
  for (int lg : {22, 24, 26, 28}) {  // table of 2^lg u32
    size_t n = (size_t)1 << lg;
    uint32_t* tab; CK(cudaMalloc(&tab, n * 4)); CK(cudaMemset(tab, 0x7f, n * 4));
    int blocks = sms * 8, threads = 256, iters = 64;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0); gather_kernel<<<blocks, threads>>>(tab, (uint32_t)(n - 1), (uint32_t*)dout, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      double acc = (double)blocks * threads * iters * 8;
      printf("gather table 2^%d u32 (%zu MB): %.3f ms  %.3f G acc/s\n", lg, n * 4 >> 20, ms, acc / ms / 1e6);
      cudaEventRecord(e0); scatter_atomic_kernel<<<blocks, threads>>>(tab, (uint32_t)(n - 1), iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      printf("atomicMin table 2^%d: %.3f ms  %.3f G atom/s\n", lg, ms, acc / ms / 1e6);
      cudaEventRecord(e0); scatter_store_kernel<<<blocks, threads>>>(tab, (uint32_t)(n - 1), iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      printf("scatter store table 2^%d: %.3f ms  %.3f G st/s\n", lg, ms, acc / ms / 1e6);
    }
    cudaFree(tab);
  }
  {
    size_t bytes = (size_t)4 << 30; uint4 *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes)); cudaMemset(a, 1, bytes);
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0); copy_kernel<<<sms * 16, 512>>>(a, b, bytes / 16); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1); printf("copy 4GiB: %.3f ms %.1f GB/s (r+w)\n", ms, 2.0 * bytes / ms / 1e6);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
