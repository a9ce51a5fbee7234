// Read-only HBM bandwidth on this part: what a streaming read-reduction can reach at the sizes the
// patch kernels read (76 MB = one bf16 config-2 activation, 152 MB = two), L2 flushed before every
// launch, CUDA events.  Variants: LDG.128 / LDG.256 grid-stride with U loads in flight per thread at
// several CTAs per SM, and a 1-D bulk-copy (cp.async.bulk) ring into shared memory; plus a copy
// kernel for the copy figure MEASURED_PEAKS.json uses.  The read-only kernels' denominator
// (hbm_kernels[].read_peak in bench.py) comes from this.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o read_bw read_bw.cu && ./read_bw
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ float sink_f;

template <int U>
__global__ void __launch_bounds__(256) rd128(const uint4* __restrict__ p, int64_t nv, float* out) {
  float s = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k0 < nv; k0 += stride * U) {
    uint4 r[U];
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const int64_t k = k0 + i * stride;
      r[i] = k < nv ? __ldg(p + k) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int i = 0; i < U; ++i) s += __uint_as_float(r[i].x ^ r[i].y ^ r[i].z ^ r[i].w);
  }
  if (s == 1.2345f) *out = s;
}

__device__ __forceinline__ void ld8(const void* p, uint32_t (&w)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
               : "l"(p));
}

template <int U>
__global__ void __launch_bounds__(256) rd256(const uint8_t* __restrict__ p, int64_t nv, float* out) {
  float s = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k0 < nv; k0 += stride * U) {
    uint32_t r[U][8];
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const int64_t k = k0 + i * stride;
      if (k < nv) ld8(p + k * 32, r[i]);
      else for (int e = 0; e < 8; ++e) r[i][e] = 0;
    }
#pragma unroll
    for (int i = 0; i < U; ++i) s += __uint_as_float(r[i][0] ^ r[i][3] ^ r[i][5] ^ r[i][7]);
  }
  if (s == 1.2345f) *out = s;
}

// contiguous chunk per warp (the gn_partials access shape: each warp streams its own slice)
template <int U>
__global__ void __launch_bounds__(64) rd256_slices(const uint8_t* __restrict__ p, int64_t slice_bytes, int n_slices,
                                                   float* out) {
  const int warp = blockIdx.x * 2 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (warp >= n_slices) return;
  const uint8_t* b = p + (int64_t)warp * slice_bytes;
  const int nv = (int)(slice_bytes / 32);
  float s = 0.f;
  for (int k0 = 0; k0 < nv; k0 += 32 * U) {
    uint32_t r[U][8];
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const int k = k0 + i * 32 + lane;
      if (k < nv) ld8(b + (int64_t)k * 32, r[i]);
      else for (int e = 0; e < 8; ++e) r[i][e] = 0;
    }
#pragma unroll
    for (int i = 0; i < U; ++i) s += __uint_as_float(r[i][0] ^ r[i][3] ^ r[i][5] ^ r[i][7]);
  }
  if (s == 1.2345f) *out = s;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su32(b)), "r"(c)); }
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar)) : "memory");
}

// bulk ring: each CTA owns a contiguous range; S stages of CH bytes; thread 0 issues, all read smem.
template <int S, int CH>
__global__ void __launch_bounds__(256) rd_bulk(const uint8_t* __restrict__ p, int64_t bytes, float* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[S];
  const int64_t nch = bytes / CH;
  const int64_t per = (nch + gridDim.x - 1) / gridDim.x;
  const int64_t c0 = blockIdx.x * per, c1 = (c0 + per < nch ? c0 + per : nch);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mb_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int s = 0; s < S && c0 + s < c1; ++s) {
      mb_expect(&full[s], CH);
      bulk(sm + s * CH, p + (c0 + s) * CH, CH, &full[s]);
    }
  float acc = 0.f;
  for (int64_t c = c0, j = 0; c < c1; ++c, ++j) {
    const int s = (int)(j % S);
    mb_wait(&full[s], (uint32_t)((j / S) & 1));
    const uint4* q = reinterpret_cast<const uint4*>(sm + s * CH);
    for (int k = threadIdx.x; k < CH / 16; k += blockDim.x) {
      const uint4 r = q[k];
      acc += __uint_as_float(r.x ^ r.w);
    }
    __syncthreads();
    if (threadIdx.x == 0 && c + S < c1) {
      mb_expect(&full[s], CH);
      bulk(sm + s * CH, p + (c + S) * CH, CH, &full[s]);
    }
  }
  if (acc == 1.2345f) *out = acc;
}

__global__ void cp128(const uint4* __restrict__ a, uint4* __restrict__ b, int64_t nv) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nv; k += stride) b[k] = __ldg(a + k);
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t maxb = 1ll << 30;
  uint8_t *buf, *buf2, *flush;
  float* out;
  CK(cudaMalloc(&buf, maxb));
  CK(cudaMalloc(&buf2, maxb));
  CK(cudaMalloc(&flush, 256ll << 20));
  CK(cudaMalloc(&out, 4));
  CK(cudaMemset(buf, 1, maxb));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  uint8_t* flush2;
  CK(cudaMalloc(&flush2, 256ll << 20));
  CK(cudaMemset(flush2, 0, 256ll << 20));
  bool clean = false;
  auto timeit = [&](auto&& launch, int reps) {
    std::vector<float> t;
    for (int r = 0; r < reps; ++r) {
      cudaMemsetAsync(flush, r, 256ll << 20);  // L2 full of dirty lines ...
      if (clean)  // ... written back by a 256 MB read of another buffer: L2 holds clean lines only
        rd128<4><<<sms * 8, 256>>>((const uint4*)flush2, (256ll << 20) / 16, out);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      t.push_back(ms);
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2] * 1e3f;  // median us
  };
  const int64_t sizes[3] = {76021760ll, 152043520ll, 1ll << 30};
  for (int mode = 0; mode < 2; ++mode)
  for (int64_t bytes : sizes) {
    clean = mode == 1;
    auto rep = [&](const char* name, float us, double traffic) {
      printf("{\"flush\": \"%s\", \"bytes\": %lld, \"variant\": \"%s\", \"us\": %.2f, \"gbs\": %.1f}\n",
             clean ? "clean" : "dirty", (long long)bytes, name, us, traffic / us / 1e3);
    };
    const int64_t nv16 = bytes / 16, nv32 = bytes / 32;
    for (int per_sm : {4, 8}) {
      const int grid = sms * per_sm;
      char nm[64];
      snprintf(nm, 64, "ldg128_u4_%dcta", per_sm);
      rep(nm, timeit([&] { rd128<4><<<grid, 256>>>((const uint4*)buf, nv16, out); }, 15), bytes);
      snprintf(nm, 64, "ldg128_u8_%dcta", per_sm);
      rep(nm, timeit([&] { rd128<8><<<grid, 256>>>((const uint4*)buf, nv16, out); }, 15), bytes);
      snprintf(nm, 64, "ldg256_u2_%dcta", per_sm);
      rep(nm, timeit([&] { rd256<2><<<grid, 256>>>(buf, nv32, out); }, 15), bytes);
      snprintf(nm, 64, "ldg256_u4_%dcta", per_sm);
      rep(nm, timeit([&] { rd256<4><<<grid, 256>>>(buf, nv32, out); }, 15), bytes);
    }
    {
      const int64_t slice = 20480;
      const int n = (int)(bytes / slice);
      rep("ldg256_u4_slices20k", timeit([&] { rd256_slices<4><<<(n + 1) / 2, 64>>>(buf, slice, n, out); }, 15), bytes);
      rep("ldg256_u2_slices20k", timeit([&] { rd256_slices<2><<<(n + 1) / 2, 64>>>(buf, slice, n, out); }, 15), bytes);
    }
    {
      constexpr int S = 4, CH = 32768;
      cudaFuncSetAttribute(rd_bulk<S, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * CH);
      for (int per_sm : {1, 2}) {
        char nm[64];
        snprintf(nm, 64, "bulk_4x32k_%dcta", per_sm);
        rep(nm, timeit([&] { rd_bulk<S, CH><<<sms * per_sm, 256, S * CH>>>(buf, bytes, out); }, 15), bytes);
      }
      constexpr int S2 = 6, CH2 = 16384;
      cudaFuncSetAttribute(rd_bulk<S2, CH2>, cudaFuncAttributeMaxDynamicSharedMemorySize, S2 * CH2);
      for (int per_sm : {2, 3}) {
        char nm[64];
        snprintf(nm, 64, "bulk_6x16k_%dcta", per_sm);
        rep(nm, timeit([&] { rd_bulk<S2, CH2><<<sms * per_sm, 256, S2 * CH2>>>(buf, bytes, out); }, 15), bytes);
      }
    }
    rep("copy128 (r+w bytes)", timeit([&] { cp128<<<sms * 8, 256>>>((const uint4*)buf, (uint4*)buf2, nv16); }, 15),
        2.0 * bytes);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
