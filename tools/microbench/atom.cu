// Random-access throughput on B200 for the K1 design: n ops into an n-entry u32 array
// (n = 2^24: 64 MB, L2-resident) -- atomicAdd, atomicMin, plain store, gather load.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t mix(uint64_t x, uint32_t n) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33;
  return static_cast<uint32_t>((x * n) >> 32 >> 0) & (n - 1);
}
__global__ void k_add(uint32_t* a, uint32_t n) { uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; if (i < n) atomicAdd(a + mix(i, n), 1u); }
__global__ void k_red(uint32_t* a, uint32_t n) { uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; if (i < n) { uint32_t* p = a + mix(i, n); asm volatile("red.global.add.u32 [%0], 1;" :: "l"(p)); } }
__global__ void k_min(uint32_t* a, uint32_t n) { uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; if (i < n) atomicMin(a + mix(i, n), i); }
__global__ void k_st(uint32_t* a, uint32_t n) { uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; if (i < n) a[mix(i, n)] = i; }
__global__ void k_ld(const uint32_t* a, uint32_t* o, uint32_t n) { uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; if (i < n) o[i] = __ldg(a + mix(i, n)); }
__global__ void k_seq(uint32_t* a, uint32_t n) { uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; if (i < n) a[i] = mix(i, n); }
int main() {
  for (int lg = 22; lg <= 26; lg += 2) {
    uint32_t n = 1u << lg;
    uint32_t *a, *o;
    cudaMalloc(&a, n * 4ull); cudaMalloc(&o, n * 4ull);
    cudaMemset(a, 0, n * 4ull);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto T = [&](const char* name, auto f) {
      f(); cudaDeviceSynchronize();
      float best = 1e9;
      for (int r = 0; r < 5; ++r) { cudaEventRecord(e0); f(); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
      printf("n=2^%d %-10s %8.1f us  %6.2f Gop/s\n", lg, name, best * 1e3, n / (best * 1e-3) / 1e9);
    };
    unsigned g = (n + 255) / 256;
    T("seq-store", [&] { k_seq<<<g, 256>>>(o, n); });
    T("atomicAdd", [&] { k_add<<<g, 256>>>(a, n); });
    T("red.add", [&] { k_red<<<g, 256>>>(a, n); });
    T("atomicMin", [&] { k_min<<<g, 256>>>(a, n); });
    T("rnd-store", [&] { k_st<<<g, 256>>>(a, n); });
    T("rnd-load", [&] { k_ld<<<g, 256>>>(a, o, n); });
    cudaFree(a); cudaFree(o);
  }
  return 0;
}
