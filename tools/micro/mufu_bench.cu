// Throughput of exp2 variants per SM: MUFU ex2.f32, ex2.f16x2, ex2.bf16x2, and an FMA-pipe polynomial.
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
__device__ __forceinline__ float ex2f(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ unsigned ex2h2(unsigned x) { unsigned y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ unsigned ex2b2(unsigned x) { unsigned y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ float ex2poly(float x) {
  x = fmaxf(x, -127.f);
  const float t = x + 12582912.f;
  const float j = t - 12582912.f;
  const float f = x - j;
  float p = fmaf(fmaf(fmaf(0.0555041086648216f, f, 0.2402264923172690f), f, 0.6931471805599453f), f, 1.0f);
  return __int_as_float(__float_as_int(p) + ((__float_as_int(t) - 0x4B400000) << 23));
}
template <int MODE>
__global__ void k(float* out, int iters) {
  float a[8]; unsigned h[8];
  for (int i = 0; i < 8; ++i) { a[i] = -0.001f * (threadIdx.x + i); h[i] = 0xB800B800u + i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = ex2f(a[i]) - 1.0f;
      if (MODE == 1) h[i] = ex2h2(h[i]) ^ 0x80008000u;
      if (MODE == 2) h[i] = ex2b2(h[i]) ^ 0x80008000u;
      if (MODE == 3) a[i] = ex2poly(a[i]) - 1.0f;
    }
  }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i] + (float)h[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE> float run(float* d, int blocks, int threads, int iters) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE><<<blocks, threads>>>(d, 10); cudaDeviceSynchronize();
  cudaEventRecord(e0); k<MODE><<<blocks, threads>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); return ms;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* d; cudaMalloc(&d, sms * 1024 * 4 * 4);
  const int threads = 512, blocks = sms * 2, iters = 4096;
  const double ops = (double)blocks * threads * iters * 8;  // per element-op (x2 for packed)
  const char* names[] = {"ex2.approx.f32 (MUFU)", "ex2.approx.f16x2", "ex2.approx.bf16x2", "poly exp2 (FMA pipe)"};
  float ms[4] = {run<0>(d, blocks, threads, iters), run<1>(d, blocks, threads, iters), run<2>(d, blocks, threads, iters),
                 run<3>(d, blocks, threads, iters)};
  for (int m = 0; m < 4; ++m) {
    double el = ops * ((m == 1 || m == 2) ? 2 : 1);
    double per_clk_sm = el / (ms[m] * 1e-3) / (clk * 1e3) / sms;
    printf("%-24s %8.3f ms  %.2f exp2/clk/SM (at %.0f MHz nominal)\n", names[m], ms[m], per_clk_sm, clk / 1e3);
  }
  return 0;
}
