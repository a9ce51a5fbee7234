// Per-SM throughput of the MUFU ops the fused FF's GELU could use (tanh.approx f32 / bf16x2 /
// f16x2, ex2.approx f32 / bf16x2, rcp.approx f32) and of the whole gelu_bf16x2 (common.cuh),
// in results per clock per SM (a bf16x2 op counts 2).  8 independent chains per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tanh_bench tanh_bench.cu
#include <cstdio>
#include "../../paper_2501_09253_b200/csrc/common.cuh"
using namespace ps;

__device__ __forceinline__ float tanhf_a(float x) { float y; asm volatile("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ unsigned tanhb2(unsigned x) { unsigned y; asm volatile("tanh.approx.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ unsigned tanhh2(unsigned x) { unsigned y; asm volatile("tanh.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ float ex2f_a(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ unsigned ex2b2(unsigned x) { unsigned y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ float rcpf_a(float x) { float y; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

template <int MODE>
__global__ void k(float* out, int iters, long long* cyc) {
  float a[8];
  unsigned h[8];
  for (int i = 0; i < 8; ++i) {
    a[i] = 0.001f * (threadIdx.x + i);
    h[i] = 0x3C003C00u + i;
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = tanhf_a(a[i]) * 1.5f;
      if (MODE == 1) h[i] = tanhb2(h[i]) ^ 0x00010001u;
      if (MODE == 2) h[i] = tanhh2(h[i]) ^ 0x00010001u;
      if (MODE == 3) a[i] = ex2f_a(a[i]) - 1.0f;
      if (MODE == 4) h[i] = ex2b2(h[i]) ^ 0x80008000u;
      if (MODE == 5) a[i] = rcpf_a(a[i]) + 1.0f;
      if (MODE == 6) h[i] = gelu_bf16x2(h[i]) ^ 0x00010001u;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = clock64() - t0;
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i] + (float)h[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char* name, int sms, int per_op) {
  float* o;
  long long* c;
  cudaMalloc(&o, sms * 1024 * 4);
  cudaMalloc(&c, 8);
  const int iters = 2000;
  k<MODE><<<sms, 1024>>>(o, 100, c);
  k<MODE><<<sms, 1024>>>(o, iters, c);
  cudaDeviceSynchronize();
  long long cyc;
  cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
  printf("%-30s %6.2f results/clk/SM\n", name, 1024.0 * iters * 8 * per_op / cyc);
  cudaFree(o);
  cudaFree(c);
}

// the fused FF's chunk epilogue shape: 8 warps per SM (2 per SMSP), 32 independent bf16x2 GELUs
// per thread per chunk (from fp32 pairs + bias, as ff_pair_kernel), cycles per chunk
template <int NW, int NPAIR>
__global__ void chunk_k(float* out, int iters, long long* cyc) {
  float x[2 * NPAIR];
  for (int i = 0; i < 2 * NPAIR; ++i) x[i] = 0.001f * (threadIdx.x + i);
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NPAIR; ++i) {
      const uint32_t g = gelu_bf16x2(pack_bf16(x[2 * i] + 0.5f, x[2 * i + 1] + 0.25f));
      acc += g;
      x[2 * i] += __uint_as_float(g & 0x8000u);  // keep a dependence across iterations
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = clock64() - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
}
template <int NW, int NPAIR>
void run_chunk(int sms) {
  float* o;
  long long* c;
  cudaMalloc(&o, sms * NW * 32 * 4);
  cudaMalloc(&c, 8);
  const int iters = 200;
  chunk_k<NW, NPAIR><<<sms, NW * 32>>>(o, 10, c);
  chunk_k<NW, NPAIR><<<sms, NW * 32>>>(o, iters, c);
  cudaDeviceSynchronize();
  long long cyc;
  cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
  printf("chunk GELU, %2d warps/SM, %2d pairs/thread: %6.0f cycles per chunk (%5.2f results/clk/SM)\n", NW, NPAIR,
         (double)cyc / iters, 2.0 * NPAIR * NW * 32 * iters / cyc);
  cudaFree(o);
  cudaFree(c);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("tanh.approx.f32", sms, 1);
  run<1>("tanh.approx.bf16x2", sms, 2);
  run<2>("tanh.approx.f16x2", sms, 2);
  run<3>("ex2.approx.f32", sms, 1);
  run<4>("ex2.approx.bf16x2", sms, 2);
  run<5>("rcp.approx.f32", sms, 1);
  run<6>("gelu_bf16x2 (common.cuh)", sms, 2);
  run_chunk<8, 32>(sms);
  run_chunk<12, 21>(sms);
  run_chunk<16, 16>(sms);
  run_chunk<8, 16>(sms);
  return 0;
}
