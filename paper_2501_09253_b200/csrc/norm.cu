// GroupNorm statistics pooled per image (K4a), NCHW -> channels-last transposes
// with GroupNorm / LayerNorm applied on the fly (K4b, LN), the fused
// "stitcher" that emits channels-last halo frames of the normalised output
// (K3+K4b), and the channels-last -> NCHW transpose with residual add.
//
// Reference: stitched_group_norm (patched.py:116-144) pools two-pass mean/var
// over all patches of one request (axes 0,2,3,4), eps 1e-5 (kernels.py:57);
// layer_norm (kernels.py:209-227) normalises every position over channels.
// Here: per-(patch, group) (mean, M2) in fp32 from a CTA-local two-pass, pooled
// per request with Chan's formula in fp64; halos are zero outside the image.
#include "common.cuh"
#include "ps_internal.h"

namespace ps {

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  const int nw = blockDim.x >> 5;
  for (int i = 0; i < nw; ++i) t += red[i];
  return t;
}

// grid (P, G): partial mean / M2 over cg*hw contiguous elements.
__global__ void gn_partials_kernel(const __nv_bfloat16* __restrict__ x, int C, int hw, int G,
                                   float* __restrict__ partials) {
  __shared__ float red[32];
  const int p = blockIdx.x, g = blockIdx.y;
  const int cg = C / G;
  const int64_t n = (int64_t)cg * hw;
  const __nv_bfloat16* base = x + ((int64_t)p * C + (int64_t)g * cg) * hw;
  const bool vec = (n % 8 == 0) && (((uintptr_t)base & 15) == 0);
  float s = 0.f;
  if (vec) {
    for (int64_t i = threadIdx.x; i < n / 8; i += blockDim.x) {
      uint4 u = __ldg(reinterpret_cast<const uint4*>(base) + i);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int k = 0; k < 4; ++k) s += __low2float(h[k]) + __high2float(h[k]);
    }
  } else {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += bf(base[i]);
  }
  const float mean = block_sum(s, red) / (float)n;
  float m2 = 0.f;
  if (vec) {
    for (int64_t i = threadIdx.x; i < n / 8; i += blockDim.x) {
      uint4 u = __ldg(reinterpret_cast<const uint4*>(base) + i);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float a = __low2float(h[k]) - mean, b = __high2float(h[k]) - mean;
        m2 += a * a + b * b;
      }
    }
  } else {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
      const float a = bf(base[i]) - mean;
      m2 += a * a;
    }
  }
  m2 = block_sum(m2, red);
  if (threadIdx.x == 0) {
    partials[((int64_t)p * G + g) * 2] = mean;
    partials[((int64_t)p * G + g) * 2 + 1] = m2;
  }
}

// grid R, block G (<=1024): Chan-combine the equal-size partials of each request.
__global__ void gn_finalize_kernel(const float* __restrict__ partials, const int32_t* __restrict__ req_off, int G,
                                   int64_t n_each, float eps, float* __restrict__ stats) {
  const int r = blockIdx.x;
  for (int g = threadIdx.x; g < G; g += blockDim.x) {
    const int p0 = req_off[r], p1 = req_off[r + 1];
    const int K = p1 - p0;
    double msum = 0.0;
    for (int p = p0; p < p1; ++p) msum += partials[((int64_t)p * G + g) * 2];
    const double mean = msum / K;
    double m2 = 0.0;
    for (int p = p0; p < p1; ++p) {
      const double d = partials[((int64_t)p * G + g) * 2] - mean;
      m2 += partials[((int64_t)p * G + g) * 2 + 1] + (double)n_each * d * d;
    }
    const double var = m2 / ((double)K * n_each);
    stats[((int64_t)r * G + g) * 2] = (float)mean;
    stats[((int64_t)r * G + g) * 2 + 1] = (float)(1.0 / sqrt(var + (double)eps));
  }
}

// NCHW -> CL over a 64-token x 64-channel tile per loop step.
// mode 0 copy, 1 group norm (stats per request/group), 2 layer norm.
constexpr int TC_TOK = 64;
__global__ void __launch_bounds__(256) to_cl_kernel(const __nv_bfloat16* __restrict__ x, int P, int C, int hw,
                                                    int Cp, int mode, const float* __restrict__ stats,
                                                    const int32_t* __restrict__ ri, int G,
                                                    const float* __restrict__ gamma, const float* __restrict__ beta,
                                                    float eps, __nv_bfloat16* __restrict__ out) {
  __shared__ float tile[64][TC_TOK + 1];
  __shared__ float ln_mean[TC_TOK], ln_rstd[TC_TOK];
  __shared__ float red[4][TC_TOK];
  const int64_t T = (int64_t)P * hw;
  const int64_t t0 = (int64_t)blockIdx.x * TC_TOK;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // 64 x 4
  const int64_t tok = t0 + tx;
  const bool tok_ok = tok < T;
  const int p = tok_ok ? (int)(tok / hw) : 0;
  const int pix = tok_ok ? (int)(tok - (int64_t)p * hw) : 0;
  const __nv_bfloat16* src = x + (int64_t)p * C * hw + pix;
  if (mode == 2) {
    float s = 0.f;
    for (int c = ty; c < C; c += 4) s += tok_ok ? bf(src[(int64_t)c * hw]) : 0.f;
    red[ty][tx] = s;
    __syncthreads();
    if (ty == 0) ln_mean[tx] = (red[0][tx] + red[1][tx] + red[2][tx] + red[3][tx]) / C;
    __syncthreads();
    const float mu = ln_mean[tx];
    float v = 0.f;
    for (int c = ty; c < C; c += 4) {
      const float d = tok_ok ? bf(src[(int64_t)c * hw]) - mu : 0.f;
      v += d * d;
    }
    red[ty][tx] = v;
    __syncthreads();
    if (ty == 0) ln_rstd[tx] = rsqrtf((red[0][tx] + red[1][tx] + red[2][tx] + red[3][tx]) / C + eps);
    __syncthreads();
  }
  const int cg = (mode == 1) ? C / G : 1;
  const int req = (mode == 1 && tok_ok) ? __ldg(ri + p) : 0;
  for (int c0 = 0; c0 < Cp; c0 += 64) {
    // load: thread (tx, ty) reads channels c0+ty, c0+ty+4, ... at token tx
    for (int cc = ty; cc < 64; cc += 4) {
      const int c = c0 + cc;
      float v = 0.f;
      if (tok_ok && c < C) {
        v = bf(src[(int64_t)c * hw]);
        if (mode == 1) {
          const int g = c / cg;
          const float mu = stats[((int64_t)req * G + g) * 2], rs = stats[((int64_t)req * G + g) * 2 + 1];
          v = (v - mu) * rs * gamma[c] + beta[c];
        } else if (mode == 2) {
          v = (v - ln_mean[tx]) * ln_rstd[tx] * gamma[c] + beta[c];
        }
      }
      tile[cc][tx] = v;
    }
    __syncthreads();
    // store: each warp writes full 128-byte channel rows of 2 tokens per pass
    for (int k = threadIdx.x; k < TC_TOK * 32; k += blockDim.x) {
      const int tk = k >> 5, cpair = k & 31;
      const int64_t t = t0 + tk;
      if (t < T)
        reinterpret_cast<uint32_t*>(out + t * Cp + c0)[cpair] = pack_bf16(tile[2 * cpair][tk], tile[2 * cpair + 1][tk]);
    }
    __syncthreads();
  }
}

// CL frames (P, ps+2, ps+2, Cp), one CTA per (patch, 64-channel chunk).
__global__ void __launch_bounds__(256) frames_cl_kernel(const __nv_bfloat16* __restrict__ x, int C, int ps, int Cp,
                                                        int mode, const float* __restrict__ stats,
                                                        const int32_t* __restrict__ ri,
                                                        const int32_t* __restrict__ nbr, int G,
                                                        const float* __restrict__ gamma,
                                                        const float* __restrict__ beta,
                                                        __nv_bfloat16* __restrict__ out) {
  extern __shared__ float fr[];  // [64][ps+3]
  const int p = blockIdx.x, c0 = blockIdx.y * 64;
  const int f = ps + 2, hw = ps * ps;
  const int ld = f + 1;
  const int cg = mode == 1 ? C / G : 1;
  const int req = __ldg(ri + p);
  int nb[8];
#pragma unroll
  for (int d = 0; d < 8; ++d) nb[d] = __ldg(nbr + (int64_t)p * 8 + d);
  for (int fy = 0; fy < f; ++fy) {
    const int ry = fy == 0 ? -1 : (fy == f - 1 ? 1 : 0);
    for (int k = threadIdx.x; k < 64 * f; k += blockDim.x) {
      const int cc = k / f, fx = k - cc * f;
      const int c = c0 + cc;
      const int rx = fx == 0 ? -1 : (fx == f - 1 ? 1 : 0);
      int q = p, sy = fy - 1, sx = fx - 1;
      if (ry != 0 || rx != 0) {
        int d;
        if (ry < 0) d = rx < 0 ? 7 : (rx > 0 ? 1 : 0);
        else if (ry > 0) d = rx < 0 ? 5 : (rx > 0 ? 3 : 4);
        else d = rx < 0 ? 6 : 2;
        q = nb[d];
        sy = ry < 0 ? ps - 1 : (ry > 0 ? 0 : fy - 1);
        sx = rx < 0 ? ps - 1 : (rx > 0 ? 0 : fx - 1);
      }
      float v = 0.f;
      if (q >= 0 && c < C) {
        v = bf(x[((int64_t)q * C + c) * hw + sy * ps + sx]);
        if (mode == 1) {
          const int g = c / cg;
          v = (v - stats[((int64_t)req * G + g) * 2]) * stats[((int64_t)req * G + g) * 2 + 1] * gamma[c] + beta[c];
        }
      }
      fr[cc * ld + fx] = v;
    }
    __syncthreads();
    __nv_bfloat16* orow = out + (((int64_t)p * f + fy) * f) * Cp + c0;
    for (int k = threadIdx.x; k < f * 32; k += blockDim.x) {
      const int fx = k >> 5, cpair = k & 31;
      reinterpret_cast<uint32_t*>(orow + (int64_t)fx * Cp)[cpair] =
          pack_bf16(fr[(2 * cpair) * ld + fx], fr[(2 * cpair + 1) * ld + fx]);
    }
    __syncthreads();
  }
}

// CL [T, Cp] -> NCHW (P, C, hw), optional + resid (NCHW).
__global__ void __launch_bounds__(256) from_cl_kernel(const __nv_bfloat16* __restrict__ xc, int P, int C, int hw,
                                                      int Cp, const __nv_bfloat16* __restrict__ resid,
                                                      __nv_bfloat16* __restrict__ out) {
  __shared__ float tile[64][65];
  const int64_t T = (int64_t)P * hw;
  const int64_t t0 = (int64_t)blockIdx.x * 64;
  const int c0 = blockIdx.y * 64;
  for (int k = threadIdx.x; k < 64 * 32; k += blockDim.x) {
    const int tk = k >> 5, cpair = k & 31;
    const int64_t t = t0 + tk;
    float a = 0.f, b = 0.f;
    if (t < T) {
      const __nv_bfloat162 v = reinterpret_cast<const __nv_bfloat162*>(xc + t * Cp + c0)[cpair];
      a = __low2float(v);
      b = __high2float(v);
    }
    tile[2 * cpair][tk] = a;
    tile[2 * cpair + 1][tk] = b;
  }
  __syncthreads();
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  const int64_t t = t0 + tx;
  if (t < T) {
    const int p = (int)(t / hw), pix = (int)(t - (int64_t)p * hw);
    for (int cc = ty; cc < 64; cc += 4) {
      const int c = c0 + cc;
      if (c >= C) break;
      const int64_t o = ((int64_t)p * C + c) * hw + pix;
      float v = tile[cc][tx];
      if (resid) v += bf(resid[o]);
      out[o] = __float2bfloat16_rn(v);
    }
  }
}

}  // namespace ps

using namespace ps;

extern "C" {

int ps_gn_partials(void* stream, const void* x, int P, int C, int ps_, int G, float* partials) {
  if (G < 1 || C % G) return set_error(PS_ERR_INPUT, "groups=%d does not divide channels=%d", G, C);
  if (P == 0) return PS_OK;
  gn_partials_kernel<<<dim3(P, G), 256, 0, (cudaStream_t)stream>>>((const __nv_bfloat16*)x, C, ps_ * ps_, G,
                                                                   partials);
  count_launch();
  return check_launch("gn_partials");
}

int ps_gn_finalize(void* stream, const float* partials, const int32_t* request_offset, int R, int G, int cg_hw,
                   float eps, float* stats) {
  if (R == 0) return PS_OK;
  gn_finalize_kernel<<<R, G < 1024 ? ((G + 31) / 32) * 32 : 1024, 0, (cudaStream_t)stream>>>(
      partials, request_offset, G, cg_hw, eps, stats);
  count_launch();
  return check_launch("gn_finalize");
}

int ps_to_cl(void* stream, const void* x, int P, int C, int ps_, int Cp, int mode, const float* stats,
             const int32_t* request_index, int G, const float* gamma, const float* beta, float eps, void* out) {
  if (Cp % 64 || Cp < C) return set_error(PS_ERR_INPUT, "to_cl: Cp must be >= C and a multiple of 64");
  if (mode == 1 && (G < 1 || C % G)) return set_error(PS_ERR_INPUT, "groups=%d does not divide channels=%d", G, C);
  const int64_t T = (int64_t)P * ps_ * ps_;
  if (T == 0) return PS_OK;
  to_cl_kernel<<<(unsigned)((T + TC_TOK - 1) / TC_TOK), 256, 0, (cudaStream_t)stream>>>(
      (const __nv_bfloat16*)x, P, C, ps_ * ps_, Cp, mode, stats, request_index, G, gamma, beta, eps,
      (__nv_bfloat16*)out);
  count_launch();
  return check_launch("to_cl");
}

int ps_frames_cl(void* stream, const void* x, int P, int C, int ps_, int Cp, int mode, const float* stats,
                 const int32_t* request_index, const int32_t* neighbors, int G, const float* gamma,
                 const float* beta, void* out) {
  if (Cp % 64 || Cp < C) return set_error(PS_ERR_INPUT, "frames_cl: Cp must be >= C and a multiple of 64");
  if (mode == 1 && (G < 1 || C % G)) return set_error(PS_ERR_INPUT, "groups=%d does not divide channels=%d", G, C);
  if (P == 0) return PS_OK;
  const int smem = 64 * (ps_ + 3) * 4;
  if (smem > 200 * 1024) return set_error(PS_ERR_INPUT, "frames_cl: patch too large");
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(frames_cl_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  frames_cl_kernel<<<dim3(P, Cp / 64), 256, smem, (cudaStream_t)stream>>>(
      (const __nv_bfloat16*)x, C, ps_, Cp, mode, stats, request_index, neighbors, G, gamma, beta,
      (__nv_bfloat16*)out);
  count_launch();
  return check_launch("frames_cl");
}

int ps_from_cl(void* stream, const void* x_cl, int P, int C, int ps_, int Cp, const void* resid, void* out) {
  const int64_t T = (int64_t)P * ps_ * ps_;
  if (T == 0) return PS_OK;
  from_cl_kernel<<<dim3((unsigned)((T + 63) / 64), (C + 63) / 64), 256, 0, (cudaStream_t)stream>>>(
      (const __nv_bfloat16*)x_cl, P, C, ps_ * ps_, Cp, (const __nv_bfloat16*)resid, (__nv_bfloat16*)out);
  count_launch();
  return check_launch("from_cl");
}

}  // extern "C"
