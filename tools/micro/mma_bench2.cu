// tcgen05.mma cta_group::2 (CTA pair, M = 256) throughput with operands resident in
// shared memory: SS with B split across the pair (N/2 rows per CTA) for N = 64..256,
// and TS (A from TMEM).  Compare with mma_bench (cta_group::1).
#include <cstdio>
#include "../../paper_2501_09253_b200/csrc/common.cuh"
using namespace ps;

template <int N, bool TS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma2_kernel(int iters, unsigned long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;          // 128 x 64 bf16 (16 KB), this CTA's rows
  uint8_t* sb = smem + 16384;  // N/2 x 64 bf16, this CTA's half of B
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool leader = cluster_rank() == 0;
  for (int i = threadIdx.x; i < (16384 + N / 2 * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc_2sm(&tslot, 512);
  fence_proxy_async();
  tc_fence_before(); cluster_sync(); tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 0) {
    const uint32_t idesc = idesc_bf16_f32(256, N);
    const long long t0 = clock64();
    if (lane == 0 && leader) {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (TS) mma_bf16_ts_2sm(tmem, tmem + 256 + k * 8, sdesc_sw128(sb + k * 32), idesc, 1);
          else mma_bf16_ss_2sm(tmem, sdesc_sw128(sa + k * 32), sdesc_sw128(sb + k * 32), idesc, 1);
        }
      }
      mma_commit_2sm(&bar, 0x3);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    if (lane == 0 && blockIdx.x == 0) *cycles = t1 - t0;
  }
  tc_fence_before(); cluster_sync(); tc_fence_after();
  if (warp == 0) tmem_dealloc_2sm(tmem, 512);
}

template <int N, bool TS>
void run(const char* name, int sms) {
  const int iters = 20000;
  unsigned long long* d; cudaMalloc(&d, 8);
  const int smem = 16384 + N / 2 * 128 + 2048;
  cudaFuncSetAttribute(mma2_kernel<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma2_kernel<N, TS><<<sms, 128, smem>>>(100, d);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  mma2_kernel<N, TS><<<sms, 128, smem>>>(iters, d);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  // per SM: 128 rows x N x 16 x 4 per iteration
  const double flop = 2.0 * 128 * N * 16 * 4 * (double)iters * sms;
  const double per_clk = 2.0 * 128 * N * 16 * 4 * (double)iters / cyc;
  printf("%-30s %7.1f TFLOP/s  %6.0f FLOP/clk/SM (peak 8192)  err=%s\n", name, flop / ms / 1e9, per_clk,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64, false>("2CTA SS M256 N64", sms);
  run<128, false>("2CTA SS M256 N128", sms);
  run<160, false>("2CTA SS M256 N160", sms);
  run<256, false>("2CTA SS M256 N256", sms);
  run<128, true>("2CTA TS M256 N128 (A tmem)", sms);
  run<160, true>("2CTA TS M256 N160 (A tmem)", sms);
  return 0;
}
