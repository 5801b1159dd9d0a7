// Per-instruction throughput microbenchmarks (instructions per SM per clock) for the
// FP64 / conversion / integer ops the pricing kernel mixes. 8 independent chains per thread.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)
#define ITERS 1000
#define BODY8(S) S(0) S(1) S(2) S(3) S(4) S(5) S(6) S(7)

#define KERN_D(name, OP) \
__global__ void name(double* out, double a, double b) { \
  double x[8]; for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k; \
  for (int i = 0; i < ITERS; ++i) { _Pragma("unroll") for (int u = 0; u < 4; ++u) { _Pragma("unroll") for (int k = 0; k < 8; ++k) { OP; } } } \
  double s = 0; for (int k = 0; k < 8; ++k) s += x[k]; out[blockIdx.x * blockDim.x + threadIdx.x] = s; }

KERN_D(k_dadd, x[k] = __dadd_rn(x[k], a))
KERN_D(k_dmul, x[k] = __dmul_rn(x[k], a))
KERN_D(k_dfma, x[k] = fma(x[k], a, b))
KERN_D(k_dsetp, x[k] = (x[k] > a) ? x[k] * a : x[k] + b )
KERN_D(k_i2f64, x[k] = (double)(unsigned)(__double2loint(x[k])) )
KERN_D(k_hilo, x[k] = __hiloint2double(0x43300000, __double2loint(x[k]) + 7) - 4503599627370496.0 )
KERN_D(k_rcp64h, { double r; asm volatile("{ .reg .f32 t; .reg .b32 lo, hi; mov.b64 {lo,hi}, %1; rcp.approx.ftz.f64 %0, %1; }" : "=d"(r) : "d"(x[k])); x[k] = r; })
KERN_D(k_d2f2d, x[k] = (double)(float)(x[k] * 1.0001) )
KERN_D(k_log, x[k] = log(x[k] + 2.0) )
KERN_D(k_exp, x[k] = exp(x[k] * 1e-3) )
KERN_D(k_div, x[k] = a / x[k] )

#define KERN_U(name, OP) \
__global__ void name(unsigned* out, unsigned a, unsigned b) { \
  unsigned x[8]; for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k * 77u; \
  for (int i = 0; i < ITERS; ++i) { _Pragma("unroll") for (int u = 0; u < 4; ++u) { _Pragma("unroll") for (int k = 0; k < 8; ++k) { OP; } } } \
  unsigned s = 0; for (int k = 0; k < 8; ++k) s ^= x[k]; out[blockIdx.x * blockDim.x + threadIdx.x] = s; }

KERN_U(k_imadhi, x[k] = __umulhi(x[k], a))
KERN_U(k_imad, x[k] = x[k] * a + b)
KERN_U(k_lop, x[k] = (x[k] ^ a) + (x[k] >> 3))
KERN_U(k_imadwide, { unsigned long long t = (unsigned long long)x[k] * a + b; x[k] = (unsigned)(t >> 32) ^ (unsigned)t; })
KERN_U(k_u32div, x[k] = x[k] / a + b)
KERN_U(k_flo, x[k] = __clz(x[k]) + x[k])

__global__ void k_ffma(float* out, float a, float b) {
  float x[8]; for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
  for (int i = 0; i < ITERS; ++i) { _Pragma("unroll") for (int u = 0; u < 4; ++u) { _Pragma("unroll") for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b); } }
  float s = 0; for (int k = 0; k < 8; ++k) s += x[k]; out[blockIdx.x * blockDim.x + threadIdx.x] = s; }

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount, clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  double* dout; CK(cudaMalloc(&dout, 1 << 26));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  int blocks = sms * 8, threads = 256;
  double ops = (double)blocks * threads * ITERS * 32;
  // measure clock with FFMA (assume 128/SM/clk)
  k_ffma<<<blocks, threads>>>((float*)dout, 0.999f, 1e-3f); cudaDeviceSynchronize();
  cudaEventRecord(e0); k_ffma<<<blocks, threads>>>((float*)dout, 0.999f, 1e-3f); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  double ghz = ops / (ms * 1e-3) / sms / 128 / 1e9;
  printf("FFMA-implied clock %.3f GHz (attr %.3f)\n", ghz, clk_khz / 1e6);
#define RUN_D(k) { k<<<blocks, threads>>>(dout, 0.9999, 1e-3); cudaDeviceSynchronize(); cudaEventRecord(e0); k<<<blocks, threads>>>(dout, 0.9999, 1e-3); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); \
   printf("%-12s %8.3f ms  %6.1f ops/SM/clk\n", #k, ms, ops / (ms * 1e-3) / sms / (ghz * 1e9)); }
#define RUN_U(k) { k<<<blocks, threads>>>((unsigned*)dout, 0x9e3779b9u, 12345u); cudaDeviceSynchronize(); cudaEventRecord(e0); k<<<blocks, threads>>>((unsigned*)dout, 0x9e3779b9u, 12345u); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); \
   printf("%-12s %8.3f ms  %6.1f ops/SM/clk\n", #k, ms, ops / (ms * 1e-3) / sms / (ghz * 1e9)); }
  RUN_D(k_dadd) RUN_D(k_dmul) RUN_D(k_dfma) RUN_D(k_dsetp) RUN_D(k_i2f64) RUN_D(k_hilo) RUN_D(k_rcp64h) RUN_D(k_d2f2d)
  RUN_D(k_log) RUN_D(k_exp) RUN_D(k_div)
  RUN_U(k_imadhi) RUN_U(k_imad) RUN_U(k_lop) RUN_U(k_imadwide) RUN_U(k_u32div) RUN_U(k_flo)
  CK(cudaGetLastError());
  return 0;
}
