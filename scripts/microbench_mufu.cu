#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__global__ void kmufu(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = ex2(a[i]) * -0.5f;
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;
}
__global__ void kclk(long long* c) { c[0] = clock64(); }
int main() {
  float* o; cudaMalloc(&o, 4);
  int sms = 148, iters = 20000;
  for (int threads : {128, 256, 512, 1024}) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    kmufu<<<sms * 2, threads>>>(o, 100);
    cudaEventRecord(e0);
    kmufu<<<sms * 2, threads>>>(o, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double exps = (double)sms * 2 * threads * iters * 8;
    printf("threads %4d: %.3f ms, %.2f Gexp/s, %.2f exp/clk/SM at max clock %d MHz (ex2 + fmul per element)\n",
           threads, ms, exps / ms / 1e6, exps / (ms * 1e-3) / (clk * 1e3) / sms, clk / 1000);
  }
  return 0;
}
