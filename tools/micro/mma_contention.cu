// SS M128 N128 tcgen05.mma throughput alone vs. with a concurrent bulk-copy (TMA engine)
// stream writing another smem region, and vs. concurrent tcgen05.ld traffic.
#include <cstdio>
#include "../../paper_2501_09253_b200/csrc/common.cuh"
using namespace ps;

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <int MODE>  // 0: MMA only, 1: + bulk copies, 2: + tcgen05.ld by 4 warps, 3: per-4-MMA wait+fence+commit, 4: per-4-MMA commit only
__global__ void __launch_bounds__(256, 1) k(int iters, const uint8_t* gsrc, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = smem;            // 16 KB
  uint8_t* sb = smem + 16384;    // 16 KB
  uint8_t* sc = smem + 32768;    // 4 x 32 KB copy targets
  __shared__ uint64_t bar, bar2, cbar[4];
  __shared__ uint32_t tslot;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); for (int i = 0; i < 4; ++i) mbar_init(&cbar[i], 1); fence_mbar_init(); done = 0; }
  if (warp == 0) tmem_alloc(&tslot, 512);
  fence_proxy_async();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tslot;
  if (MODE == 10 && warp == 1) {  // second issuer: half the groups into TMEM cols 128..255
    const uint32_t idesc = idesc_bf16_f32(128, 128);
    if (lane == 0) {
      for (int it = 0; it < iters / 2; ++it) {
        mbar_wait(&cbar[0], 1); tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(tmem + 128, sdesc_sw128(sa + kk * 32), sdesc_sw128(sb + kk * 32), idesc, 1);
        mma_commit(&cbar[3]);
      }
      mma_commit(&bar2);
    }
  }
  if (warp == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, 128);
    const long long t0 = clock64();
    if (lane == 0) {
      for (int it = 0; it < (MODE == 10 ? iters / 2 : iters); ++it) {
        if (MODE == 10) { mbar_wait(&cbar[0], 1); tc_fence_after(); }
        if (MODE == 9) {
          uint32_t ok = 0;
          while (!ok) asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(smem_u32(&cbar[0])), "r"(1u) : "memory");
          tc_fence_after();
        }
        if (MODE == 3) { mbar_wait(&cbar[0], 1); tc_fence_after(); }  // already-complete phase: the attention pattern
        if (MODE == 5) { mbar_wait(&cbar[0], 1); }
        if (MODE == 6) { tc_fence_after(); }
        if (MODE == 7 && (it & 1) == 0) { mbar_wait(&cbar[0], 1); tc_fence_after(); }  // per 8 MMAs
        if (MODE == 8 && (it & 3) == 0) { mbar_wait(&cbar[0], 1); tc_fence_after(); }  // per 16 MMAs
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) mma_bf16_ss(tmem, sdesc_sw128(sa + kk * 32), sdesc_sw128(sb + kk * 32), idesc, 1);
        if (MODE >= 3) mma_commit(&cbar[1 + (it & 1)]);
      }
      mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    if (MODE == 10) mbar_wait(&bar2, 0);
    const long long t1 = clock64();
    if (lane == 0) { done = 1; if (blockIdx.x == 0) out[0] = t1 - t0; }
  } else if (warp == 1 && MODE == 1) {
    if (lane == 0) {
      unsigned long long bytes = 0; uint32_t ph[4] = {0, 0, 0, 0}; int s = 0;
      for (int i = 0; i < 4; ++i) { mbar_arrive_expect_tx(&cbar[i], 32768); bulk_g2s(sc + i * 32768, gsrc + (size_t)(blockIdx.x * 4 + i) * 32768, 32768, &cbar[i]); }
      while (!done) {
        mbar_wait(&cbar[s], ph[s]); ph[s] ^= 1; bytes += 32768;
        mbar_arrive_expect_tx(&cbar[s], 32768);
        bulk_g2s(sc + s * 32768, gsrc + (size_t)(blockIdx.x * 4 + s) * 32768, 32768, &cbar[s]);
        s = (s + 1) & 3;
      }
      for (int i = 0; i < 4; ++i) { mbar_wait(&cbar[s], ph[s]); ph[s] ^= 1; s = (s + 1) & 3; }
      if (blockIdx.x == 0) out[1] = bytes;
    }
  } else if (warp >= 4 && MODE == 2) {
    const uint32_t lb = (uint32_t)((warp & 3) * 32) << 16;
    unsigned long long n = 0;
    while (!done) {
      uint32_t r[32];
      PS_TMEM_LD32(tmem + lb + 256, r);
      tmem_ld_wait();
      n += r[0] & 1;
      ++n;
    }
    if (blockIdx.x == 0 && warp == 4 && lane == 0) out[1] = n;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int MODE> void run(const char* name, int sms, const uint8_t* g) {
  const int iters = 20000;
  unsigned long long* d; cudaMalloc(&d, 16); cudaMemset(d, 0, 16);
  const int smem = 32768 + 4 * 32768 + 2048;
  cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<MODE><<<sms, 256, smem>>>(100, g, d); cudaDeviceSynchronize();
  k<MODE><<<sms, 256, smem>>>(iters, g, d); cudaDeviceSynchronize();
  unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  const double per_clk = 2.0 * 128 * 128 * 16 * 4 * (double)iters / h[0];
  printf("%-34s %6.0f FLOP/clk/SM (%.0f%% of 8192)  side traffic %.1f B/clk  err=%s\n", name, per_clk,
         100 * per_clk / 8192, MODE == 1 ? (double)h[1] / h[0] : (MODE == 2 ? 128.0 * 128 * h[1] / h[0] : 0.0),
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint8_t* g; cudaMalloc(&g, (size_t)sms * 4 * 32768); cudaMemset(g, 0, (size_t)sms * 4 * 32768);
  run<0>("SS N128 alone", sms, g);
  run<1>("SS N128 + bulk copies to smem", sms, g);
  run<2>("SS N128 + tcgen05.ld (4 warps)", sms, g);
  run<3>("SS N128, wait+fence+commit / 4 MMAs", sms, g);
  run<4>("SS N128, commit / 4 MMAs", sms, g);
  run<5>("SS N128, wait / 4 MMAs", sms, g);
  run<6>("SS N128, fence / 4 MMAs", sms, g);
  run<7>("SS N128, wait+fence / 8 MMAs", sms, g);
  run<8>("SS N128, wait+fence / 16 MMAs", sms, g);
  run<9>("SS N128, test_wait+fence / 4 MMAs", sms, g);
  run<10>("SS N128, 2 issuers, wait+fence / 4", sms, g);
  return 0;
}
