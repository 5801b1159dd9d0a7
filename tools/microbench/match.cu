// Throughput of __match_any_sync (MATCH.ANY) and shared-memory atomics on 12-bit keys
// (K1 radix design input). nvcc -gencode arch=compute_100a,code=sm_100a -O3 match.cu -o match
#include <cstdio>
#include <cstdint>
__global__ void match_kernel(const uint32_t* in, uint32_t* out, int iters) {
  uint32_t x = in[blockIdx.x * blockDim.x + threadIdx.x];
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
    const uint32_t d = (x >> 7) & 4095u;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    acc += __popc(peers);
    x = x * 1664525u + 1013904223u + acc;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void atom_kernel(const uint32_t* in, uint32_t* out, int iters) {
  __shared__ uint32_t cnt[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) cnt[i] = 0;
  __syncthreads();
  uint32_t x = in[blockIdx.x * blockDim.x + threadIdx.x];
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
    const uint32_t d = (x >> 7) & 4095u;
    acc += atomicAdd(&cnt[d], 1u);
    x = x * 1664525u + 1013904223u + acc;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void plain_kernel(const uint32_t* in, uint32_t* out, int iters) {
  uint32_t x = in[blockIdx.x * blockDim.x + threadIdx.x];
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
    const uint32_t d = (x >> 7) & 4095u;
    acc += __popc(d);
    x = x * 1664525u + 1013904223u + acc;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  const int blocks = 148 * 8, threads = 256, iters = 4096;
  uint32_t *in, *out;
  cudaMalloc(&in, blocks * threads * 4);
  cudaMalloc(&out, blocks * threads * 4);
  uint32_t* h = new uint32_t[blocks * threads];
  for (int i = 0; i < blocks * threads; ++i) h[i] = i * 2654435761u;
  cudaMemcpy(in, h, blocks * threads * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int k = 0; k < 3; ++k) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (k == 0) match_kernel<<<blocks, threads>>>(in, out, iters);
      if (k == 1) atom_kernel<<<blocks, threads>>>(in, out, iters);
      if (k == 2) plain_kernel<<<blocks, threads>>>(in, out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double ops = double(blocks) * threads * iters;
      if (rep) printf("%s: %.3f ms, %.3g ops/s (%.2f ns per warp-op per SM)\n", k == 0 ? "match_any" : k == 1 ? "smem atomicAdd" : "plain",
                      ms, ops / (ms * 1e-3), ms * 1e6 / (ops / 32 / 148));
    }
  }
  return 0;
}
