#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float tnh(float x) { float y; asm volatile("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float rcp(float x) { float y; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <int OP> __global__ void k(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = (OP == 0 ? tnh(a[i]) : OP == 1 ? ex2(a[i]) : rcp(a[i] + 2.f)) * 0.5f;
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;
}
template <int OP> void run(const char* name, float* o) {
  int sms = 148, iters = 20000, threads = 512;
  k<OP><<<sms * 2, threads>>>(o, 100);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<OP><<<sms * 2, threads>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double n = (double)sms * 2 * threads * iters * 8;
  printf("%s: %.2f per clk per SM (at %d MHz nominal)\n", name, n / (ms * 1e-3) / (clk * 1e3) / sms, clk / 1000);
}
int main() { float* o; cudaMalloc(&o, 4); run<0>("tanh.approx", o); run<1>("ex2.approx", o); run<2>("rcp.approx", o); return 0; }
