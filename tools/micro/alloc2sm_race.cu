// Minimal repro for compute-sanitizer racecheck's report on tcgen05.alloc.cta_group::2: a CTA
// pair allocates TMEM collectively (warp 0 of each CTA), orders the write of the address with
// tcgen05.fence::before_thread_sync -> barrier.cluster -> tcgen05.fence::after_thread_sync (the
// documented pattern), reads the address slot, deallocates.  No other shared-memory access.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o alloc2sm_race alloc2sm_race.cu
//   compute-sanitizer --tool racecheck ./alloc2sm_race
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __cluster_dims__(2, 1, 1) alloc_pair(uint32_t* out) {
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(32)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = slot;
  if (threadIdx.x == 0) out[blockIdx.x] = t;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(32) : "memory");
}

// variant: the kernels' layout -- warp 2 allocates into a slot in DYNAMIC shared memory right
// after mbarriers that warp 0 lane 0 initialises concurrently; 256 threads
__global__ void __cluster_dims__(2, 1, 1) alloc_pair_dyn(uint32_t* out) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(dsm + 4096);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 4);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bars + i)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if ((threadIdx.x >> 5) == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(64)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t t = *slot;
  if (threadIdx.x == 0) out[2 + blockIdx.x] = t;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if ((threadIdx.x >> 5) == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(64) : "memory");
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 8 * sizeof(uint32_t));
  alloc_pair<<<2, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaFuncSetAttribute(alloc_pair_dyn, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  alloc_pair_dyn<<<2, 256, 100 * 1024>>>(d);
  cudaError_t e2 = cudaDeviceSynchronize();
  printf("alloc_pair_dyn: %s\n", cudaGetErrorString(e2));
  uint32_t h[2];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("alloc_pair: %s, tmem addresses %u %u\n", cudaGetErrorString(e), h[0], h[1]);
  return e == cudaSuccess ? 0 : 1;
}
