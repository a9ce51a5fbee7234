// CSP split / reassemble (K2), NCHW halo frames (K3, API layout), step wrapper
// (K10: prompt bias, blend) and dtype conversion.  All HBM-bound: 16-byte
// vector accesses along the contiguous pixel axis, grid-stride over the
// 148 SMs.
#include <stdlib.h>

#include "common.cuh"
#include "ps_internal.h"

namespace ps {

static inline int grid_for(int64_t work, int threads) {
  int64_t b = (work + threads - 1) / threads;
  const int64_t cap = 148 * 16;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

// Copy one patch row segment (ps elements) between an image (C, L, L) and the
// patch array (P, C, ps, ps).  VEC elements per thread-step (16 bytes).
template <typename T, int VEC, bool TO_PATCHES>
__global__ void csp_copy_kernel(const uint64_t* __restrict__ img_ptrs, const int32_t* __restrict__ req_off,
                                const int32_t* __restrict__ sides, int n_req, int C, int ps, T* __restrict__ patches,
                                int64_t total_vec) {
  const int vps = ps / VEC;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < total_vec;
       v += (int64_t)gridDim.x * blockDim.x) {
    // v -> (patch, c, y, xv)
    int64_t t = v;
    const int xv = (int)(t % vps);
    t /= vps;
    const int y = (int)(t % ps);
    t /= ps;
    const int c = (int)(t % C);
    const int p = (int)(t / C);
    // owning request: binary search over request offsets (n_req is small)
    int lo = 0, hi = n_req - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (__ldg(req_off + mid) <= p) lo = mid; else hi = mid - 1;
    }
    const int side = __ldg(sides + lo);
    const int k = p - __ldg(req_off + lo);
    const int r = k / side, cc = k % side;
    const int L = side * ps;
    T* img = reinterpret_cast<T*>(img_ptrs[lo]);
    const int64_t io = ((int64_t)c * L + (int64_t)r * ps + y) * L + (int64_t)cc * ps + xv * VEC;
    const int64_t po = (((int64_t)p * C + c) * ps + y) * ps + xv * VEC;
    if constexpr (VEC * sizeof(T) == 16) {
      if (TO_PATCHES)
        *reinterpret_cast<uint4*>(patches + po) = __ldg(reinterpret_cast<const uint4*>(img + io));
      else
        *reinterpret_cast<uint4*>(img + io) = __ldg(reinterpret_cast<const uint4*>(patches + po));
    } else {
#pragma unroll
      for (int i = 0; i < VEC; ++i) {
        if (TO_PATCHES) patches[po + i] = img[io + i];
        else img[io + i] = patches[po + i];
      }
    }
  }
}

// Patch-major variants (config-2 sizes): one CTA per (patch, CPB channels); the owning
// request is resolved once per CTA, and every thread keeps 8 independent 16-byte loads in
// flight before storing (the grid-stride versions above are latency-bound: index math and
// a dependent request lookup per 16 bytes).
constexpr int PM_UNR = 8;

__device__ __forceinline__ void pm_locate(int p, const int32_t* req_off, const int32_t* sides, int n_req,
                                          int& req, int& side, int& k) {
  int lo = 0, hi = n_req - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(req_off + mid) <= p) lo = mid; else hi = mid - 1;
  }
  req = lo;
  side = __ldg(sides + lo);
  k = p - __ldg(req_off + lo);
}

template <typename T, bool TO_PATCHES>
__global__ void __launch_bounds__(256) csp_copy_pm_kernel(const uint64_t* __restrict__ img_ptrs,
                                                          const int32_t* __restrict__ req_off,
                                                          const int32_t* __restrict__ sides, int n_req, int C,
                                                          int ps, int cpb, T* __restrict__ patches) {
  constexpr int VEC = 16 / sizeof(T);
  const int p = blockIdx.x, c0 = blockIdx.y * cpb;
  int req, side, k;
  pm_locate(p, req_off, sides, n_req, req, side, k);
  const int r = k / side, cc = k - r * side, L = side * ps;
  T* img = reinterpret_cast<T*>(img_ptrs[req]);
  const int vps = ps / VEC;
  const int nc = min(cpb, C - c0);
  const int n = nc * ps * vps;
  for (int base = threadIdx.x; base < n; base += 256 * PM_UNR) {
    uint4 v[PM_UNR];
    int64_t dst[PM_UNR];
#pragma unroll
    for (int u = 0; u < PM_UNR; ++u) {
      const int i = base + u * 256;
      dst[u] = -1;
      if (i < n) {
        const int xv = i % vps, y = (i / vps) % ps, c = c0 + i / (vps * ps);
        const int64_t io = ((int64_t)c * L + (int64_t)r * ps + y) * L + (int64_t)cc * ps + xv * VEC;
        const int64_t po = (((int64_t)p * C + c) * ps + y) * ps + xv * VEC;
        v[u] = __ldg(reinterpret_cast<const uint4*>(TO_PATCHES ? img + io : patches + po));
        dst[u] = TO_PATCHES ? po : io;
      }
    }
#pragma unroll
    for (int u = 0; u < PM_UNR; ++u)
      if (dst[u] >= 0) *reinterpret_cast<uint4*>((TO_PATCHES ? patches : img) + dst[u]) = v[u];
  }
}

// h = bf16(latent + prompt[request]) over (patch, CPB channels) CTAs, 8 float4 in flight
__global__ void __launch_bounds__(256) prompt_bias_pm_kernel(const float* __restrict__ lat,
                                                             const float* __restrict__ prompts,
                                                             const int32_t* __restrict__ ri, int C, int hw, int cpb,
                                                             __nv_bfloat16* __restrict__ h) {
  const int p = blockIdx.x, c0 = blockIdx.y * cpb;
  const int nc = min(cpb, C - c0);
  const int n = nc * hw / 4;
  const float* pr = prompts + (int64_t)__ldg(ri + p) * C;
  const int64_t off4 = (((int64_t)p * C + c0) * hw) / 4;
  for (int base = threadIdx.x; base < n; base += 256 * PM_UNR) {
    float4 x[PM_UNR];
#pragma unroll
    for (int u = 0; u < PM_UNR; ++u) {
      const int i = base + u * 256;
      if (i < n) x[u] = __ldg(reinterpret_cast<const float4*>(lat) + off4 + i);
    }
#pragma unroll
    for (int u = 0; u < PM_UNR; ++u) {
      const int i = base + u * 256;
      if (i < n) {
        const float b = __ldg(pr + c0 + (i * 4) / hw);
        uint2 o;
        o.x = pack_bf16(x[u].x + b, x[u].y + b);
        o.y = pack_bf16(x[u].z + b, x[u].w + b);
        reinterpret_cast<uint2*>(h)[off4 + i] = o;
      }
    }
  }
}

// (1 - r) x + r tanh(h) per request rate, over (patch, CPB channels) CTAs
__global__ void __launch_bounds__(256) blend_pm_kernel(const float* __restrict__ lat,
                                                       const __nv_bfloat16* __restrict__ hh,
                                                       const float* __restrict__ rates,
                                                       const int32_t* __restrict__ ri, int C, int hw, int cpb,
                                                       float* __restrict__ out) {
  const int p = blockIdx.x, c0 = blockIdx.y * cpb;
  const int nc = min(cpb, C - c0);
  const int n = nc * hw / 4;
  const float r = __ldg(rates + __ldg(ri + p));
  const int64_t off4 = (((int64_t)p * C + c0) * hw) / 4;
  for (int base = threadIdx.x; base < n; base += 256 * PM_UNR) {
    float4 x[PM_UNR];
    uint2 hv[PM_UNR];
#pragma unroll
    for (int u = 0; u < PM_UNR; ++u) {
      const int i = base + u * 256;
      if (i < n) {
        x[u] = __ldg(reinterpret_cast<const float4*>(lat) + off4 + i);
        hv[u] = __ldg(reinterpret_cast<const uint2*>(hh) + off4 + i);
      }
    }
#pragma unroll
    for (int u = 0; u < PM_UNR; ++u) {
      const int i = base + u * 256;
      if (i < n) {
        const __nv_bfloat162 h01 = *reinterpret_cast<const __nv_bfloat162*>(&hv[u].x);
        const __nv_bfloat162 h23 = *reinterpret_cast<const __nv_bfloat162*>(&hv[u].y);
        float4 o;
        o.x = (1.f - r) * x[u].x + r * tanh_exp(__low2float(h01));
        o.y = (1.f - r) * x[u].y + r * tanh_exp(__high2float(h01));
        o.z = (1.f - r) * x[u].z + r * tanh_exp(__low2float(h23));
        o.w = (1.f - r) * x[u].w + r * tanh_exp(__high2float(h23));
        reinterpret_cast<float4*>(out)[off4 + i] = o;
      }
    }
  }
}

// channels per CTA so one CTA moves ~32 KB of the patch array
static inline int pm_cpb(int C, int ps, int elem_bytes) {
  int cpb = (32 * 1024) / (ps * ps * elem_bytes);
  if (cpb < 1) cpb = 1;
  if (cpb > C) cpb = C;
  return cpb;
}

// Split along image rows: one CTA per (request, patch row, CPB channels) reads whole image
// rows (side * ps contiguous pixels per channel row) and scatters them to that patch row's
// patches -- long contiguous DRAM reads; the writes land as full 16-byte patch-row pieces.
template <typename T>
__global__ void __launch_bounds__(256) csp_split_rows_kernel(const uint64_t* __restrict__ img_ptrs,
                                                             const int32_t* __restrict__ req_off,
                                                             const int32_t* __restrict__ sides, int n_req, int C,
                                                             int ps, int cpb, T* __restrict__ patches) {
  constexpr int VEC = 16 / sizeof(T);
  // blockIdx.x -> (request, patch row): walk the requests' row counts
  int pr = blockIdx.x, req = 0;
  for (; req < n_req; ++req) {
    const int sd = __ldg(sides + req);
    if (pr < sd) break;
    pr -= sd;
  }
  if (req >= n_req) return;  // the grid is sized by P >= the number of patch rows
  const int side = __ldg(sides + req), L = side * ps, p0 = __ldg(req_off + req) + pr * side;
  const T* img = reinterpret_cast<const T*>(img_ptrs[req]);
  const int c0 = blockIdx.y * cpb, nc = min(cpb, C - c0);
  const int vrow = L / VEC;                      // 16-byte vectors per image row
  const int n = nc * ps * vrow;
  for (int base = threadIdx.x; base < n; base += 256 * PM_UNR) {
    uint4 v[PM_UNR];
    int64_t dst[PM_UNR];
#pragma unroll
    for (int u = 0; u < PM_UNR; ++u) {
      const int i = base + u * 256;
      dst[u] = -1;
      if (i < n) {
        const int xv = i % vrow, y = (i / vrow) % ps, c = c0 + i / (vrow * ps);
        const int x = xv * VEC, pc = x / ps, xp = x - pc * ps;
        v[u] = __ldg(reinterpret_cast<const uint4*>(img + ((int64_t)c * L + (int64_t)pr * ps + y) * L + x));
        dst[u] = (((int64_t)(p0 + pc) * C + c) * ps + y) * ps + xp;
      }
    }
#pragma unroll
    for (int u = 0; u < PM_UNR; ++u)
      if (dst[u] >= 0) *reinterpret_cast<uint4*>(patches + dst[u]) = v[u];
  }
}

// Fused step ends for the fixed-composition pipeline (pipeline.py):
//  * split + prompt bias: the image rows land in the CSP fp32 latents AND as the first block
//    input h = bf16(latent + prompt[request]) (model.py:163) -- one read of the latents;
//  * blend + reassemble: (1 - r) x + r tanh(h) (model.py:129-131) written straight into the
//    per-request output images -- no CSP intermediate.
__global__ void __launch_bounds__(256) csp_split_bias_rows_kernel(const uint64_t* __restrict__ img_ptrs,
                                                                  const int32_t* __restrict__ req_off,
                                                                  const int32_t* __restrict__ sides, int n_req,
                                                                  int C, int ps, int cpb,
                                                                  const float* __restrict__ prompts,
                                                                  float* __restrict__ patches,
                                                                  __nv_bfloat16* __restrict__ h) {
  pdl_wait();
  int pr = blockIdx.x, req = 0;
  for (; req < n_req; ++req) {
    const int sd = __ldg(sides + req);
    if (pr < sd) break;
    pr -= sd;
  }
  if (req >= n_req) return;
  const int side = __ldg(sides + req), L = side * ps, p0 = __ldg(req_off + req) + pr * side;
  const float* img = reinterpret_cast<const float*>(img_ptrs[req]);
  const float* pr_bias = prompts + (int64_t)req * C;
  const int c0 = blockIdx.y * cpb, nc = min(cpb, C - c0);
  const int vrow = L / 4;
  const int n = nc * ps * vrow;
  for (int base = threadIdx.x; base < n; base += 256 * PM_UNR) {
    float4 v[PM_UNR];
    int64_t dst[PM_UNR];
    float bb[PM_UNR];
#pragma unroll
    for (int u = 0; u < PM_UNR; ++u) {
      const int i = base + u * 256;
      dst[u] = -1;
      if (i < n) {
        const int xv = i % vrow, y = (i / vrow) % ps, c = c0 + i / (vrow * ps);
        const int x = xv * 4, pc = x / ps, xp = x - pc * ps;
        v[u] = __ldg(reinterpret_cast<const float4*>(img + ((int64_t)c * L + (int64_t)pr * ps + y) * L + x));
        dst[u] = (((int64_t)(p0 + pc) * C + c) * ps + y) * ps + xp;
        bb[u] = __ldg(pr_bias + c);
      }
    }
#pragma unroll
    for (int u = 0; u < PM_UNR; ++u)
      if (dst[u] >= 0) {
        if (patches != nullptr) *reinterpret_cast<float4*>(patches + dst[u]) = v[u];
        uint2 o;
        o.x = pack_bf16(v[u].x + bb[u], v[u].y + bb[u]);
        o.y = pack_bf16(v[u].z + bb[u], v[u].w + bb[u]);
        *reinterpret_cast<uint2*>(h + dst[u]) = o;
      }
  }
}

__global__ void __launch_bounds__(256) blend_reassemble_kernel(const float* __restrict__ lat,
                                                               const __nv_bfloat16* __restrict__ hh,
                                                               const float* __restrict__ rates,
                                                               const uint64_t* __restrict__ img_ptrs,
                                                               const int32_t* __restrict__ req_off,
                                                               const int32_t* __restrict__ sides, int n_req, int C,
                                                               int ps, int cpb,
                                                               const uint64_t* __restrict__ src_ptrs) {
  pdl_wait();
  const int p = blockIdx.x, c0 = blockIdx.y * cpb;
  int req, side, k;
  pm_locate(p, req_off, sides, n_req, req, side, k);
  const int r = k / side, cc = k - r * side, L = side * ps;
  float* img = reinterpret_cast<float*>(img_ptrs[req]);
  // x from the request's input image (same coordinates as the output) when given: the
  // split then skips writing the fp32 CSP copy
  const float* src = src_ptrs ? reinterpret_cast<const float*>(src_ptrs[req]) : nullptr;
  const float rate = __ldg(rates + req);
  const int vps = ps / 4;
  const int nc = min(cpb, C - c0);
  const int n = nc * ps * vps;
  for (int base = threadIdx.x; base < n; base += 256 * PM_UNR) {
    float4 x[PM_UNR];
    uint2 hv[PM_UNR];
    int64_t io[PM_UNR];
#pragma unroll
    for (int u = 0; u < PM_UNR; ++u) {
      const int i = base + u * 256;
      io[u] = -1;
      if (i < n) {
        const int xv = i % vps, y = (i / vps) % ps, c = c0 + i / (vps * ps);
        const int64_t po = (((int64_t)p * C + c) * ps + y) * ps + xv * 4;
        io[u] = ((int64_t)c * L + (int64_t)r * ps + y) * L + (int64_t)cc * ps + xv * 4;
        x[u] = __ldg(reinterpret_cast<const float4*>(src ? src + io[u] : lat + po));
        hv[u] = __ldg(reinterpret_cast<const uint2*>(hh + po));
      }
    }
#pragma unroll
    for (int u = 0; u < PM_UNR; ++u)
      if (io[u] >= 0) {
        const __nv_bfloat162 h01 = *reinterpret_cast<const __nv_bfloat162*>(&hv[u].x);
        const __nv_bfloat162 h23 = *reinterpret_cast<const __nv_bfloat162*>(&hv[u].y);
        float4 o;
        o.x = (1.f - rate) * x[u].x + rate * tanh_exp(__low2float(h01));
        o.y = (1.f - rate) * x[u].y + rate * tanh_exp(__high2float(h01));
        o.z = (1.f - rate) * x[u].z + rate * tanh_exp(__low2float(h23));
        o.w = (1.f - rate) * x[u].w + rate * tanh_exp(__high2float(h23));
        *reinterpret_cast<float4*>(img + io[u]) = o;
      }
  }
}


// Step ends v2 (patch-major, one thread = 8 pixels of one patch row): the CTA owns
// (patch, CPB channels); thread vector j of a channel covers patch row y = j / (PS/8), pixels
// x = 8 (j % (PS/8)) .. +8, i.e. one 32-byte image read (two 16-byte halves of the same
// 128-byte image row segment the neighbouring lanes read) and one 16-byte bf16 CSP write that
// is contiguous with its lanes' -- no per-element division (PS is a template power of two), the
// request is resolved once per CTA, every CTA has work, and each thread keeps U independent
// 32-byte loads in flight.  `nonfinite` (optional): set to 1 when an input latent is not finite
// (kernels.py:20-24 rejects those; the pipeline raises after the step).
constexpr int SE_THREADS = 256;
constexpr int SE_UNR = 4;

template <int PS>
__global__ void __launch_bounds__(SE_THREADS) split_bias_v2_kernel(const uint64_t* __restrict__ img_ptrs,
                                                                   const int32_t* __restrict__ req_off,
                                                                   const int32_t* __restrict__ sides, int n_req,
                                                                   int C, int cpb, const float* __restrict__ prompts,
                                                                   float* __restrict__ patches,
                                                                   __nv_bfloat16* __restrict__ h,
                                                                   int* __restrict__ nonfinite) {
  constexpr int VPR = PS / 8;           // vectors per patch row
  constexpr int VPC = PS * VPR;         // vectors per channel
  pdl_wait();
  const int p = blockIdx.x, c0 = blockIdx.y * cpb;
  int req, side, k;
  pm_locate(p, req_off, sides, n_req, req, side, k);
  const int r = k / side, cc = k - r * side, L = side * PS;
  const float* img = reinterpret_cast<const float*>(img_ptrs[req]) + (int64_t)r * PS * L + cc * PS;
  const float* pb = prompts + (int64_t)req * C;
  const int n = min(cpb, C - c0) * VPC;
  const int64_t out0 = ((int64_t)p * C + c0) * PS * PS;
  bool bad = false;
  for (int base = threadIdx.x; base < n; base += SE_THREADS * SE_UNR) {
    uint32_t v[SE_UNR][8];
#pragma unroll
    for (int u = 0; u < SE_UNR; ++u) {
      const int j = base + u * SE_THREADS;
      if (j < n) {
        const int c = j / VPC, jj = j % VPC, y = jj / VPR, x = (jj % VPR) * 8;
        ld_global_nc_v8(img + ((int64_t)(c0 + c) * L + y) * L + x, v[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < SE_UNR; ++u) {
      const int j = base + u * SE_THREADS;
      if (j < n) {
        const float b = __ldg(pb + c0 + j / VPC);
        float f[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          f[e] = __uint_as_float(v[u][e]);
          bad |= !isfinite(f[e]);
        }
        if (patches != nullptr) st_global_v8(patches + out0 + (int64_t)j * 8, v[u]);
        uint4 o;
        o.x = pack_bf16(f[0] + b, f[1] + b);
        o.y = pack_bf16(f[2] + b, f[3] + b);
        o.z = pack_bf16(f[4] + b, f[5] + b);
        o.w = pack_bf16(f[6] + b, f[7] + b);
        *reinterpret_cast<uint4*>(h + out0 + (int64_t)j * 8) = o;
      }
    }
  }
  if (nonfinite != nullptr && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1);
}

template <int PS>
__global__ void __launch_bounds__(SE_THREADS) blend_reassemble_v2_kernel(const float* __restrict__ lat,
                                                                         const __nv_bfloat16* __restrict__ hh,
                                                                         const float* __restrict__ rates,
                                                                         const uint64_t* __restrict__ img_ptrs,
                                                                         const int32_t* __restrict__ req_off,
                                                                         const int32_t* __restrict__ sides, int n_req,
                                                                         int C, int cpb,
                                                                         const uint64_t* __restrict__ src_ptrs) {
  constexpr int VPR = PS / 8;
  constexpr int VPC = PS * VPR;
  pdl_wait();
  const int p = blockIdx.x, c0 = blockIdx.y * cpb;
  int req, side, k;
  pm_locate(p, req_off, sides, n_req, req, side, k);
  const int r = k / side, cc = k - r * side, L = side * PS;
  const int64_t img0 = (int64_t)r * PS * L + cc * PS;
  float* dst = reinterpret_cast<float*>(img_ptrs[req]) + img0;
  const float* src = src_ptrs ? reinterpret_cast<const float*>(src_ptrs[req]) + img0 : nullptr;
  const float rate = __ldg(rates + req);
  const int n = min(cpb, C - c0) * VPC;
  const int64_t csp0 = ((int64_t)p * C + c0) * PS * PS;
  for (int base = threadIdx.x; base < n; base += SE_THREADS * SE_UNR) {
    uint32_t x[SE_UNR][8];
    uint4 hv[SE_UNR];
    int64_t io[SE_UNR];
#pragma unroll
    for (int u = 0; u < SE_UNR; ++u) {
      const int j = base + u * SE_THREADS;
      if (j < n) {
        const int c = j / VPC, jj = j % VPC, y = jj / VPR, xo = (jj % VPR) * 8;
        io[u] = ((int64_t)(c0 + c) * L + y) * L + xo;
        ld_global_nc_v8(src ? src + io[u] : lat + csp0 + (int64_t)j * 8, x[u]);
        hv[u] = __ldg(reinterpret_cast<const uint4*>(hh + csp0 + (int64_t)j * 8));
      }
    }
#pragma unroll
    for (int u = 0; u < SE_UNR; ++u) {
      const int j = base + u * SE_THREADS;
      if (j < n) {
        const uint32_t hw4[4] = {hv[u].x, hv[u].y, hv[u].z, hv[u].w};
        uint32_t o[8];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const __nv_bfloat162 h2 = *reinterpret_cast<const __nv_bfloat162*>(&hw4[e]);
          o[2 * e] = __float_as_uint((1.f - rate) * __uint_as_float(x[u][2 * e]) + rate * tanh_exp(__low2float(h2)));
          o[2 * e + 1] =
              __float_as_uint((1.f - rate) * __uint_as_float(x[u][2 * e + 1]) + rate * tanh_exp(__high2float(h2)));
        }
        st_global_v8(dst + io[u], o);
      }
    }
  }
}

// channels per CTA of the v2 step ends: ~8 KB of bf16 CSP output per CTA round
static inline int se_cpb(int C, int ps) {
  int cpb = (SE_THREADS * SE_UNR * 8) / (ps * ps);
  if (cpb < 1) cpb = 1;
  if (cpb > C) cpb = C;
  return cpb;
}


template <bool TO_PATCHES>
static int csp_copy(cudaStream_t st, const uint64_t* ptrs, const int32_t* off, const int32_t* sides, int n_req,
                    int C, int ps, int dtype, void* patches, int P) {
  const int64_t elems = (int64_t)P * C * ps * ps;
  if (elems == 0) return PS_OK;
  const int th = 256;
  if (TO_PATCHES && dtype == PS_DTYPE_F32 && ps % 4 == 0 && P <= 65535) {
    // one CTA per patch row; the row count (sum of the sides, <= P) is on the device, so the
    // grid is sized by P and surplus CTAs return at once
    const int rows = P;
    const int cpb = pm_cpb(C, ps, 4);
    csp_split_rows_kernel<float><<<dim3(rows, (C + cpb - 1) / cpb), th, 0, st>>>(ptrs, off, sides, n_req, C, ps,
                                                                               cpb, (float*)patches);
  } else if (dtype == PS_DTYPE_F32 && ps % 4 == 0 && P <= 65535) {
    const int cpb = pm_cpb(C, ps, 4);
    csp_copy_pm_kernel<float, TO_PATCHES><<<dim3(P, (C + cpb - 1) / cpb), th, 0, st>>>(ptrs, off, sides, n_req, C,
                                                                                    ps, cpb, (float*)patches);
  } else if (dtype == PS_DTYPE_F64 && ps % 2 == 0 && P <= 65535) {
    // fp64 patches (the numpy-interface drop-in keeps the reference's float64 pixels exact)
    const int cpb = pm_cpb(C, ps, 8);
    csp_copy_pm_kernel<double, TO_PATCHES><<<dim3(P, (C + cpb - 1) / cpb), th, 0, st>>>(ptrs, off, sides, n_req, C,
                                                                                     ps, cpb, (double*)patches);
  } else if (dtype == PS_DTYPE_F64) {
    csp_copy_kernel<double, 1, TO_PATCHES><<<grid_for(elems, th), th, 0, st>>>(ptrs, off, sides, n_req, C, ps,
                                                                            (double*)patches, elems);
  } else if (dtype == PS_DTYPE_BF16 && ps % 8 == 0 && P <= 65535) {
    const int cpb = pm_cpb(C, ps, 2);
    csp_copy_pm_kernel<__nv_bfloat16, TO_PATCHES><<<dim3(P, (C + cpb - 1) / cpb), th, 0, st>>>(
        ptrs, off, sides, n_req, C, ps, cpb, (__nv_bfloat16*)patches);
  } else if (dtype == PS_DTYPE_F32) {
    if (ps % 4 == 0)
      csp_copy_kernel<float, 4, TO_PATCHES><<<grid_for(elems / 4, th), th, 0, st>>>(ptrs, off, sides, n_req, C, ps,
                                                                                 (float*)patches, elems / 4);
    else
      csp_copy_kernel<float, 1, TO_PATCHES><<<grid_for(elems, th), th, 0, st>>>(ptrs, off, sides, n_req, C, ps,
                                                                             (float*)patches, elems);
  } else if (dtype == PS_DTYPE_BF16) {
    if (ps % 8 == 0)
      csp_copy_kernel<__nv_bfloat16, 8, TO_PATCHES><<<grid_for(elems / 8, th), th, 0, st>>>(
          ptrs, off, sides, n_req, C, ps, (__nv_bfloat16*)patches, elems / 8);
    else
      csp_copy_kernel<__nv_bfloat16, 1, TO_PATCHES><<<grid_for(elems, th), th, 0, st>>>(
          ptrs, off, sides, n_req, C, ps, (__nv_bfloat16*)patches, elems);
  } else {
    return set_error(PS_ERR_INPUT, "csp copy: unsupported dtype %d", dtype);
  }
  count_launch();
  return check_launch(TO_PATCHES ? "csp_split" : "csp_reassemble");
}

// NCHW halo frames: frame (fy, fx) of patch p reads its own patch for the
// interior, else the neighbour in that direction (patched.py:64-88), else 0.
template <typename T>
__global__ void halo_nchw_kernel(const T* __restrict__ src, const int32_t* __restrict__ nbr, int P, int C, int ps,
                                 T* __restrict__ dst) {
  const int f = ps + 2;
  const int64_t total = (int64_t)P * C * f * f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int fx = (int)(i % f);
    const int fy = (int)((i / f) % f);
    const int c = (int)((i / ((int64_t)f * f)) % C);
    const int p = (int)(i / ((int64_t)f * f * C));
    const int ry = fy == 0 ? -1 : (fy == f - 1 ? 1 : 0);
    const int rx = fx == 0 ? -1 : (fx == f - 1 ? 1 : 0);
    // direction index N,NE,E,SE,S,SW,W,NW
    int q = p, sy = fy - 1, sx = fx - 1;
    if (ry != 0 || rx != 0) {
      int d;
      if (ry < 0) d = rx < 0 ? 7 : (rx > 0 ? 1 : 0);
      else if (ry > 0) d = rx < 0 ? 5 : (rx > 0 ? 3 : 4);
      else d = rx < 0 ? 6 : 2;
      q = __ldg(nbr + (int64_t)p * 8 + d);
      sy = ry < 0 ? ps - 1 : (ry > 0 ? 0 : fy - 1);
      sx = rx < 0 ? ps - 1 : (rx > 0 ? 0 : fx - 1);
    }
    T v = T(0.f);
    if (q >= 0) v = src[(((int64_t)q * C + c) * ps + sy) * ps + sx];
    dst[i] = v;
  }
}

__global__ void prompt_bias_kernel(const float* __restrict__ lat, const float* __restrict__ prompts,
                                   const int32_t* __restrict__ ri, int P, int C, int hw,
                                   __nv_bfloat16* __restrict__ h) {
  const int64_t total4 = (int64_t)P * C * hw / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total4; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i * 4;
    const int c = (int)((e / hw) % C);
    const int p = (int)(e / ((int64_t)hw * C));
    const float b = __ldg(prompts + (int64_t)__ldg(ri + p) * C + c);
    const float4 x = __ldg(reinterpret_cast<const float4*>(lat) + i);
    uint2 o;
    o.x = pack_bf16(x.x + b, x.y + b);
    o.y = pack_bf16(x.z + b, x.w + b);
    reinterpret_cast<uint2*>(h)[i] = o;
  }
}

__global__ void blend_kernel(const float* __restrict__ lat, const __nv_bfloat16* __restrict__ h,
                             const float* __restrict__ rates, const int32_t* __restrict__ ri, int P, int C, int hw,
                             float* __restrict__ out) {
  const int64_t total4 = (int64_t)P * C * hw / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total4; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i * 4;
    const int p = (int)(e / ((int64_t)hw * C));
    const float r = __ldg(rates + __ldg(ri + p));
    const float4 x = __ldg(reinterpret_cast<const float4*>(lat) + i);
    const uint2 hv = __ldg(reinterpret_cast<const uint2*>(h) + i);
    const __nv_bfloat162 h01 = *reinterpret_cast<const __nv_bfloat162*>(&hv.x);
    const __nv_bfloat162 h23 = *reinterpret_cast<const __nv_bfloat162*>(&hv.y);
    float4 o;
    o.x = (1.f - r) * x.x + r * tanh_exp(__low2float(h01));
    o.y = (1.f - r) * x.y + r * tanh_exp(__high2float(h01));
    o.z = (1.f - r) * x.z + r * tanh_exp(__low2float(h23));
    o.w = (1.f - r) * x.w + r * tanh_exp(__high2float(h23));
    reinterpret_cast<float4*>(out)[i] = o;
  }
}

template <typename S, typename D>
__global__ void convert_kernel(const S* __restrict__ src, D* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = D(float(src[i]));
}

}  // namespace ps

using namespace ps;

extern "C" {

int ps_csp_split_bias(void* stream, const uint64_t* src_ptrs, const int32_t* request_offset, const int32_t* sides,
                      int n_req, int C, int ps_, float* dst, int n_patches, const float* prompts, void* h,
                      int* nonfinite) {
  if (n_req < 1 || C < 1 || ps_ < 1 || ps_ % 4) return set_error(PS_ERR_INPUT, "csp_split_bias: bad sizes");
  if (n_patches == 0) return PS_OK;
  if (n_patches > 65535) return set_error(PS_ERR_INPUT, "csp_split_bias: too many patches");
  cudaStream_t st = (cudaStream_t)stream;
  if (ps_ == 16 || ps_ == 32 || ps_ == 64) {
    const int cpb = se_cpb(C, ps_);
    const dim3 grid(n_patches, (C + cpb - 1) / cpb);
    if (ps_ == 16)
      launch_pdl(split_bias_v2_kernel<16>, grid, dim3(SE_THREADS), 0, st, src_ptrs, request_offset, sides, n_req, C,
                 cpb, prompts, dst, (__nv_bfloat16*)h, nonfinite);
    else if (ps_ == 32)
      launch_pdl(split_bias_v2_kernel<32>, grid, dim3(SE_THREADS), 0, st, src_ptrs, request_offset, sides, n_req, C,
                 cpb, prompts, dst, (__nv_bfloat16*)h, nonfinite);
    else
      launch_pdl(split_bias_v2_kernel<64>, grid, dim3(SE_THREADS), 0, st, src_ptrs, request_offset, sides, n_req, C,
                 cpb, prompts, dst, (__nv_bfloat16*)h, nonfinite);
  } else {
    if (nonfinite != nullptr) return set_error(PS_ERR_INPUT, "csp_split_bias: finiteness flag needs ps in {16,32,64}");
    const int cpb = pm_cpb(C, ps_, 4);
    launch_pdl(csp_split_bias_rows_kernel, dim3(n_patches, (C + cpb - 1) / cpb), dim3(256), 0, st, src_ptrs,
               request_offset, sides, n_req, C, ps_, cpb, prompts, dst, (__nv_bfloat16*)h);
  }
  count_launch();
  return check_launch("csp_split_bias");
}

int ps_blend_reassemble(void* stream, const float* latent, const void* h, const float* rates,
                        const int32_t* request_offset, const int32_t* sides, int n_req, int C, int ps_,
                        const uint64_t* dst_ptrs, int n_patches, const uint64_t* src_ptrs) {
  if (n_req < 1 || C < 1 || ps_ < 1 || ps_ % 4) return set_error(PS_ERR_INPUT, "blend_reassemble: bad sizes");
  if (latent == nullptr && src_ptrs == nullptr) return set_error(PS_ERR_INPUT, "blend_reassemble: no latent source");
  if (n_patches == 0) return PS_OK;
  if (n_patches > 65535) return set_error(PS_ERR_INPUT, "blend_reassemble: too many patches");
  cudaStream_t st = (cudaStream_t)stream;
  if (ps_ == 16 || ps_ == 32 || ps_ == 64) {
    const int cpb = se_cpb(C, ps_);
    const dim3 grid(n_patches, (C + cpb - 1) / cpb);
    const __nv_bfloat16* hb = (const __nv_bfloat16*)h;
    if (ps_ == 16)
      launch_pdl(blend_reassemble_v2_kernel<16>, grid, dim3(SE_THREADS), 0, st, latent, hb, rates, dst_ptrs,
                 request_offset, sides, n_req, C, cpb, src_ptrs);
    else if (ps_ == 32)
      launch_pdl(blend_reassemble_v2_kernel<32>, grid, dim3(SE_THREADS), 0, st, latent, hb, rates, dst_ptrs,
                 request_offset, sides, n_req, C, cpb, src_ptrs);
    else
      launch_pdl(blend_reassemble_v2_kernel<64>, grid, dim3(SE_THREADS), 0, st, latent, hb, rates, dst_ptrs,
                 request_offset, sides, n_req, C, cpb, src_ptrs);
  } else {
    const int cpb = pm_cpb(C, ps_, 4);
    launch_pdl(blend_reassemble_kernel, dim3(n_patches, (C + cpb - 1) / cpb), dim3(256), 0, st, latent,
               (const __nv_bfloat16*)h, rates, dst_ptrs, request_offset, sides, n_req, C, ps_, cpb, src_ptrs);
  }
  count_launch();
  return check_launch("blend_reassemble");
}

int ps_csp_split(void* stream, const uint64_t* src_ptrs, const int32_t* request_offset, const int32_t* sides,
                 int n_req, int C, int ps_, int dtype, void* dst, int n_patches) {
  if (n_req < 1 || C < 1 || ps_ < 1) return set_error(PS_ERR_INPUT, "csp_split: bad sizes");
  return csp_copy<true>((cudaStream_t)stream, src_ptrs, request_offset, sides, n_req, C, ps_, dtype, dst, n_patches);
}

int ps_csp_reassemble(void* stream, const void* src, const uint64_t* dst_ptrs, const int32_t* request_offset,
                      const int32_t* sides, int n_req, int C, int ps_, int dtype, int n_patches) {
  if (n_req < 1 || C < 1 || ps_ < 1) return set_error(PS_ERR_INPUT, "csp_reassemble: bad sizes");
  return csp_copy<false>((cudaStream_t)stream, dst_ptrs, request_offset, sides, n_req, C, ps_, dtype,
                         const_cast<void*>(src), n_patches);
}

int ps_halo_frames_nchw(void* stream, const void* src, int dtype, const int32_t* neighbors, int P, int C, int ps_,
                        void* dst) {
  const int64_t total = (int64_t)P * C * (ps_ + 2) * (ps_ + 2);
  if (total == 0) return PS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == PS_DTYPE_F32)
    halo_nchw_kernel<float><<<grid_for(total, 256), 256, 0, st>>>((const float*)src, neighbors, P, C, ps_,
                                                                  (float*)dst);
  else if (dtype == PS_DTYPE_F64)
    halo_nchw_kernel<double><<<grid_for(total, 256), 256, 0, st>>>((const double*)src, neighbors, P, C, ps_,
                                                                    (double*)dst);
  else if (dtype == PS_DTYPE_BF16)
    halo_nchw_kernel<__nv_bfloat16><<<grid_for(total, 256), 256, 0, st>>>((const __nv_bfloat16*)src, neighbors, P, C,
                                                                          ps_, (__nv_bfloat16*)dst);
  else
    return set_error(PS_ERR_INPUT, "halo: unsupported dtype");
  count_launch();
  return check_launch("halo_frames_nchw");
}

int ps_prompt_bias(void* stream, const float* latent, const float* prompts, const int32_t* request_index, int P,
                   int C, int ps_, void* h) {
  const int hw = ps_ * ps_;
  if (hw % 4) return set_error(PS_ERR_INPUT, "prompt_bias: ps*ps must be a multiple of 4");
  const int64_t n4 = (int64_t)P * C * hw / 4;
  if (n4 == 0) return PS_OK;
  if (hw >= 64 && P <= 65535) {
    const int cpb = pm_cpb(C, ps_, 4);
    prompt_bias_pm_kernel<<<dim3(P, (C + cpb - 1) / cpb), 256, 0, (cudaStream_t)stream>>>(
        latent, prompts, request_index, C, hw, cpb, (__nv_bfloat16*)h);
    count_launch();
    return check_launch("prompt_bias");
  }
  prompt_bias_kernel<<<grid_for(n4, 256), 256, 0, (cudaStream_t)stream>>>(latent, prompts, request_index, P, C, hw,
                                                                          (__nv_bfloat16*)h);
  count_launch();
  return check_launch("prompt_bias");
}

int ps_blend(void* stream, const float* latent, const void* h, const float* rates, const int32_t* request_index,
             int P, int C, int ps_, float* out) {
  const int hw = ps_ * ps_;
  if (hw % 4) return set_error(PS_ERR_INPUT, "blend: ps*ps must be a multiple of 4");
  const int64_t n4 = (int64_t)P * C * hw / 4;
  if (n4 == 0) return PS_OK;
  if (hw >= 64 && P <= 65535) {
    const int cpb = pm_cpb(C, ps_, 4);
    blend_pm_kernel<<<dim3(P, (C + cpb - 1) / cpb), 256, 0, (cudaStream_t)stream>>>(
        latent, (const __nv_bfloat16*)h, rates, request_index, C, hw, cpb, out);
    count_launch();
    return check_launch("blend");
  }
  blend_kernel<<<grid_for(n4, 256), 256, 0, (cudaStream_t)stream>>>(latent, (const __nv_bfloat16*)h, rates,
                                                                    request_index, P, C, hw, out);
  count_launch();
  return check_launch("blend");
}

int ps_convert(void* stream, const void* src, int sd, void* dst, int dd, int64_t n) {
  if (n == 0) return PS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int g = grid_for(n, 256);
  if (sd == PS_DTYPE_F32 && dd == PS_DTYPE_BF16)
    convert_kernel<float, __nv_bfloat16><<<g, 256, 0, st>>>((const float*)src, (__nv_bfloat16*)dst, n);
  else if (sd == PS_DTYPE_BF16 && dd == PS_DTYPE_F32)
    convert_kernel<__nv_bfloat16, float><<<g, 256, 0, st>>>((const __nv_bfloat16*)src, (float*)dst, n);
  else
    return set_error(PS_ERR_INPUT, "convert: unsupported dtype pair");
  count_launch();
  return check_launch("convert");
}

}  // extern "C"
