// Dependent-chain latencies (cycles) of the instructions on the pricing kernel's critical paths.
#include <cstdio>
#include <cstdint>
__global__ void lat_dfma(double* out, long long* cyc, double a, double b, int n) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); }
  long long t1 = clock64();
  out[threadIdx.x] = x; cyc[0] = t1 - t0;
}
__global__ void lat_dadd(double* out, long long* cyc, double a, int n) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __dadd_rn(x, a); x = __dadd_rn(x, a); x = __dadd_rn(x, a); x = __dadd_rn(x, a); }
  long long t1 = clock64();
  out[threadIdx.x] = x; cyc[0] = t1 - t0;
}
__global__ void lat_imadhi(unsigned* out, long long* cyc, unsigned a, int n) {
  unsigned x = threadIdx.x + 12345;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = __umulhi(x, a) + 7; x = __umulhi(x, a) + 7; x = __umulhi(x, a) + 7; x = __umulhi(x, a) + 7; }
  long long t1 = clock64();
  out[threadIdx.x] = x; cyc[0] = t1 - t0;
}
__global__ void lat_ffma(float* out, long long* cyc, float a, float b, int n) {
  float x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = fmaf(x, a, b); x = fmaf(x, a, b); x = fmaf(x, a, b); x = fmaf(x, a, b); }
  long long t1 = clock64();
  out[threadIdx.x] = x; cyc[0] = t1 - t0;
}
__global__ void lat_rcp(double* out, long long* cyc, int n) {
  double x = threadIdx.x + 1.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r + 1.0; }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x; cyc[0] = t1 - t0;
}
int main() {
  double* d; long long* c; cudaMalloc(&d, 1 << 20); cudaMalloc(&c, 64);
  long long h; int n = 4096;
  lat_dfma<<<1, 1>>>(d, c, 0.999, 1e-3, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  lat_dfma<<<1, 1>>>(d, c, 0.999, 1e-3, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("DFMA latency %.2f cyc\n", h / (4.0 * n));
  lat_dadd<<<1, 1>>>(d, c, 1e-3, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("DADD latency %.2f cyc\n", h / (4.0 * n));
  lat_imadhi<<<1, 1>>>((unsigned*)d, c, 0x9e3779b9u, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("IMAD.HI+IADD latency %.2f cyc\n", h / (4.0 * n));
  lat_ffma<<<1, 1>>>((float*)d, c, 0.999f, 1e-3f, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("FFMA latency %.2f cyc\n", h / (4.0 * n));
  lat_rcp<<<1, 1>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("MUFU.RCP64H+DADD latency %.2f cyc\n", h / (4.0 * n));
  return 0;
}
