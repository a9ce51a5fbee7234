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
#include <stdlib.h>

#include "common.cuh"
#include "ps_internal.h"

namespace ps {

static bool getenv_flag(const char* name) {
  const char* v = getenv(name);
  return v && atoi(v) != 0;
}

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

// grid (P, G): partial mean / M2 over cg*hw contiguous elements.  The CTA's
// slice is read once into registers (up to GN_REG 16-byte vectors per thread);
// mean and then M2 are reduced from registers (two-pass numerics, one pass of HBM).
constexpr int GN_REG = 5;
// (mean, M2) of one slice of nv 16-byte vectors held in registers (nv <= GN_REG * 256);
// shared by gn_partials_kernel and the fused gn_frames_kernel (identical arithmetic)
__device__ __forceinline__ void gn_slice_regs(const __nv_bfloat16* __restrict__ base, int nv, float n, float* red,
                                              float& mean, float& m2) {
  uint4 reg[GN_REG];
#pragma unroll
  for (int i = 0; i < GN_REG; ++i) {
    const int k = threadIdx.x + i * blockDim.x;
    reg[i] = k < nv ? __ldg(reinterpret_cast<const uint4*>(base) + k) : make_uint4(0, 0, 0, 0);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < GN_REG; ++i) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&reg[i]);
#pragma unroll
    for (int k = 0; k < 4; ++k) s += __low2float(h[k]) + __high2float(h[k]);
  }
  mean = block_sum(s, red) / n;
  m2 = 0.f;
#pragma unroll
  for (int i = 0; i < GN_REG; ++i) {
    if (threadIdx.x + i * blockDim.x < nv) {
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&reg[i]);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float a = __low2float(h[k]) - mean, b = __high2float(h[k]) - mean;
        m2 += a * a + b * b;
      }
    }
  }
  m2 = block_sum(m2, red);
}

__global__ void __launch_bounds__(256, 4) gn_partials_kernel(const __nv_bfloat16* __restrict__ x, int C, int hw, int G,
                                                          const int32_t* __restrict__ plist,
                                                          const int32_t* __restrict__ n_dev,
                                                          float* __restrict__ partials) {
  pdl_wait();
  __shared__ float red[32];
  if (n_dev != nullptr && (int)blockIdx.x >= *n_dev) return;  // past the device list length
  const int p = plist ? __ldg(plist + blockIdx.x) : (int)blockIdx.x, g = blockIdx.y;
  const int cg = C / G;
  const int64_t n = (int64_t)cg * hw;
  const __nv_bfloat16* base = x + ((int64_t)p * C + (int64_t)g * cg) * hw;
  const bool vec = (n % 8 == 0) && (((uintptr_t)base & 15) == 0) && (n / 8 <= (int64_t)GN_REG * blockDim.x);
  float mean, m2 = 0.f;
  if (vec) {
    gn_slice_regs(base, (int)(n / 8), (float)n, red, mean, m2);
    if (threadIdx.x == 0) {
      partials[((int64_t)p * G + g) * 2] = mean;
      partials[((int64_t)p * G + g) * 2 + 1] = m2;
    }
    return;
  } else if ((n % 8 == 0) && (((uintptr_t)base & 15) == 0)) {
    // slice larger than the register budget: two vectorised passes (the second hits L2)
    const uint4* b4 = reinterpret_cast<const uint4*>(base);
    const int64_t nv = n / 8;
    float s = 0.f;
    for (int64_t k = threadIdx.x; k < nv; k += blockDim.x) {
      const uint4 r = __ldg(b4 + k);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
      for (int e = 0; e < 4; ++e) s += __low2float(h[e]) + __high2float(h[e]);
    }
    mean = block_sum(s, red) / (float)n;
    for (int64_t k = threadIdx.x; k < nv; k += blockDim.x) {
      const uint4 r = __ldg(b4 + k);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float a = __low2float(h[e]) - mean, b = __high2float(h[e]) - mean;
        m2 += a * a + b * b;
      }
    }
  } else {
    float s = 0.f;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += bf(base[i]);
    mean = block_sum(s, red) / (float)n;
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

// Warp-per-slice form (default): one warp streams a (patch, group) slice with 4 independent
// 32-byte non-allocating loads (LDG.256) per lane in flight, accumulating shifted moments (shift
// K = the slice's first element) in fp32: a single pass, no block reductions.
// mean = K + S1/n, M2 = S2 - S1^2/n.  Two warps per CTA: 1856 small CTAs fill every SM evenly
// in one wave (one-CTA-per-slice two-pass kernel: 6.3 waves of short CTAs, 22.6 us in ncu;
// 8-warp CTAs: 464 CTAs left SMs with 4 vs 3 of them, 17.4 us; four warps per slice with the
// quarters' sums added: 19.3 us; a persistent bulk-copy ring reduced by whole CTAs: 24 us).
// (The parts machinery below adds GNW_PARTS warps' sums of one slice in a fixed order.)
__device__ __forceinline__ void acc8(const uint4& r, float K, float& s1, float& s2) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
  float a = 0.f, b = 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float d0 = __low2float(h[k]) - K, d1 = __high2float(h[k]) - K;
    a += d0 + d1;
    b = fmaf(d0, d0, fmaf(d1, d1, b));
  }
  s1 += a;
  s2 += b;
}
template <int GNW_WARPS, int GNW_PARTS, int GNW_UNROLL>
__global__ void __launch_bounds__(GNW_WARPS * 32) gn_partials_warp_kernel(
    const __nv_bfloat16* __restrict__ x, int C, int hw, int G, const int32_t* __restrict__ plist,
    const int32_t* __restrict__ n_dev, int n_host, float* __restrict__ partials) {
  constexpr int GNW_SLICES = GNW_WARPS / GNW_PARTS;  // slices per CTA
  __shared__ float2 red[GNW_WARPS];
  pdl_wait();
  const int n_items = (n_dev != nullptr ? min(*n_dev, n_host) : n_host) * G;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int item = blockIdx.x * GNW_SLICES + warp / GNW_PARTS, part = warp % GNW_PARTS;
  const bool live = item < n_items;
  int p = 0, g = 0;
  const int cg = C / G;
  float t1 = 0.f, t2 = 0.f;
  if (live) {
    const int q = item / G;
    g = item - q * G;
    p = plist ? __ldg(plist + q) : q;
    const __nv_bfloat16* base = x + ((int64_t)p * C + (int64_t)g * cg) * hw;
    const int nv = cg * hw / 16;  // 32-byte vectors
    const int per = (nv + GNW_PARTS - 1) / GNW_PARTS;
    const int v0 = part * per, v1 = min(nv, v0 + per);
    const float K = __bfloat162float(base[0]);  // the slice's shift, the same for its parts
    float s1[2] = {0.f, 0.f}, s2[2] = {0.f, 0.f};
    for (int k0 = v0; k0 < v1; k0 += 32 * GNW_UNROLL) {
      uint4 r[GNW_UNROLL][2];
#pragma unroll
      for (int i = 0; i < GNW_UNROLL; ++i) {
        const int k = k0 + i * 32 + lane;
        if (k < v1) ld_global_nc_v8(base + (int64_t)k * 16, *reinterpret_cast<uint32_t(*)[8]>(&r[i][0]));
      }
#pragma unroll
      for (int i = 0; i < GNW_UNROLL; ++i)
        if (k0 + i * 32 + lane < v1) {
          acc8(r[i][0], K, s1[0], s2[0]);
          acc8(r[i][1], K, s1[1], s2[1]);
        }
    }
    t1 = s1[0] + s1[1];
    t2 = s2[0] + s2[1];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      t1 += __shfl_xor_sync(0xffffffffu, t1, o);
      t2 += __shfl_xor_sync(0xffffffffu, t2, o);
    }
    if (lane == 0) red[warp] = make_float2(t1, t2);
  }
  __syncthreads();
  if (live && part == 0 && lane == 0) {
    // the parts share the shift, so their moments add (fixed order: deterministic)
    float u1 = red[warp].x, u2 = red[warp].y;
#pragma unroll
    for (int k = 1; k < GNW_PARTS; ++k) {
      u1 += red[warp + k].x;
      u2 += red[warp + k].y;
    }
    const float n = (float)(cg * hw);
    const float K = __bfloat162float(x[((int64_t)p * C + (int64_t)g * cg) * hw]);
    partials[((int64_t)p * G + g) * 2] = K + u1 / n;
    partials[((int64_t)p * G + g) * 2 + 1] = fmaxf(u2 - u1 * (u1 / n), 0.f);
  }
}

// host: one CTA per (patch, group) slice.  (Persistent software-pipelined and bulk-copy staged
// variants measured 21-26 us against 20-21 us; a group-pair kernel -- one CTA per two adjacent
// groups, all ten 16-byte loads per thread issued first, one shifted-sum block reduction --
// measured 26.2 vs 21.6 us (ncu, round 2).  All removed.)
static void launch_gn_partials(cudaStream_t st, const void* x, int P, int C, int hw, int G, const int32_t* plist,
                               int n, float* partials, const int32_t* n_dev = nullptr) {
  (void)P;
  (void)C;
  const auto xb = (const __nv_bfloat16*)x;
  const int64_t slice = (int64_t)(C / G) * hw * 2;
  static const bool warp_off = getenv_flag("PS_GN_WARP_OFF");
  if (!warp_off && n > 0 && C % G == 0 && slice % 32 == 0 && ((uintptr_t)x & 31) == 0) {
    const int items = n * G;
    // (warps per CTA, warps per slice, 32-byte loads per lane in flight) = (2, 1, 4).  Round-2
    // sweep (tools/gn_sweep.py, L2 flushed, CUDA events): (2,1,4) 18.4 us, (1,1,4) 18.5, (4,1,4)
    // 18.4, (2,1,8) 21.9, (2,1,10) 20.5, (4,2,5) 20.5, (2,2,5) 20.5 -- a plain read-reduction of the
    // same 76 MB (torch.sum) takes 24.6 us: read-only launches of this size stop well short of
    // the copy bandwidth the roofline uses (profiles/r2_read_floor.jsonl).
#define PS_GNW(W, PT, U)                                                                                      \
  launch_pdl(gn_partials_warp_kernel<W, PT, U>, dim3((items + W / PT - 1) / (W / PT)), dim3(W * 32), 0, st, xb, C, \
             hw, G, plist, n_dev, n, partials)
    // ps = 64 slices (C/G * 4096 bf16 = 80 KB at C = 320): four warps per slice, their shifted
    // sums added in a fixed order -- a warp streaming 80 KB alone is 20 dependent round trips, and
    // a rank of a split image has only ~100 slices (config 5, 8 ranks: 19.6 us for 8 MB).  Chosen by
    // slice size only, so a split-image rank and the single-GPU batch round identically.
    if (slice >= 64 * 1024)
      PS_GNW(8, 4, 4);
    else
      PS_GNW(2, 1, 4);
#undef PS_GNW
    return;
  }
  launch_pdl(gn_partials_kernel, dim3(n, G), dim3(256), 0, st, xb, C, hw, G, plist, n_dev, partials);
}

// Chan-combine the equal-size partials of patches [p0, p1) for group g -> (mean, rstd).
// COHERENT: the partials were written by other CTAs of the same launch (L2 loads).
template <bool COHERENT>
__device__ __forceinline__ void gn_finalize_group(const float* partials, int p0, int p1, int G, int g, int64_t n_each,
                                                  float eps, float* out) {
  auto ld = [&](int64_t i) { return COHERENT ? __ldcg(partials + i) : partials[i]; };
  const int K = p1 - p0;
  double msum = 0.0;
  for (int p = p0; p < p1; ++p) msum += ld(((int64_t)p * G + g) * 2);
  const double mean = msum / K;
  double m2 = 0.0;
  for (int p = p0; p < p1; ++p) {
    const double d = ld(((int64_t)p * G + g) * 2) - mean;
    m2 += ld(((int64_t)p * G + g) * 2 + 1) + (double)n_each * d * d;
  }
  const double var = m2 / ((double)K * n_each);
  out[0] = (float)mean;
  out[1] = (float)(1.0 / sqrt(var + (double)eps));
}

// grid R, block G (<=1024): Chan-combine the equal-size partials of each request.
__global__ void gn_finalize_kernel(const float* __restrict__ partials, const int32_t* __restrict__ req_off, int G,
                                   int64_t n_each, float eps, float* __restrict__ stats) {
  pdl_wait();
  const int r = blockIdx.x;
  for (int g = threadIdx.x; g < G; g += blockDim.x)
    gn_finalize_group<false>(partials, req_off[r], req_off[r + 1], G, g, n_each, eps, stats + ((int64_t)r * G + g) * 2);
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

// Vectorised NCHW -> CL transpose with optional GroupNorm, R frame rows per CTA.
// FRAMES: output (P, ps+2, ps+2, Cp) with the 1-pixel neighbour ring (zero
// outside the image); else output (P*ps*ps, Cp) tokens.  smem tile
// [R][W][64] bf16 with the channel index XOR-swizzled by the pixel so both the
// scattered stores (phase 1) and the 16-byte channel-run reads (phase 2) are
// bank-conflict free.
template <bool FRAMES, int VEC>
__global__ void __launch_bounds__(256) frames_vec_kernel(const __nv_bfloat16* __restrict__ x, int C, int ps, int Cp,
                                                         int mode, const float* __restrict__ stats,
                                                         const int32_t* __restrict__ ri,
                                                         const int32_t* __restrict__ nbr, int G,
                                                         const float* __restrict__ gamma,
                                                         const float* __restrict__ beta, int R,
                                                         const int32_t* __restrict__ plist,
                                                         __nv_bfloat16* __restrict__ out) {
  extern __shared__ __align__(16) __nv_bfloat16 tile[];
  const int p = plist ? __ldg(plist + blockIdx.x) : (int)blockIdx.x, c0 = blockIdx.y * 64;
  const int F = FRAMES ? ps + 2 : ps;    // output side
  const int off = FRAMES ? 1 : 0;        // interior offset in the output row
  const int r0 = blockIdx.z * R;
  const int rows = min(R, F - r0);
  const int hw = ps * ps;
  const int req = mode == 1 ? __ldg(ri + p) : 0;
  auto sw = [](int fx) { return (fx & 7) << 3; };
  // per-channel affine of this CTA's 64 channels: y = x * a + b (GroupNorm) or identity
  __shared__ float ch_a[64], ch_b[64];
  if (threadIdx.x < 64) {
    const int c = c0 + threadIdx.x;
    float a = 1.f, b = 0.f;
    if (mode == 1 && c < C) {
      const int g = c / (C / G);
      const float mu = __ldg(stats + ((int64_t)req * G + g) * 2), rs = __ldg(stats + ((int64_t)req * G + g) * 2 + 1);
      a = rs * __ldg(gamma + c);
      b = __ldg(beta + c) - mu * a;
    }
    ch_a[threadIdx.x] = a;
    ch_b[threadIdx.x] = b;
  }
  __syncthreads();
  auto norm = [&](float v, int cc) { return fmaf(v, ch_a[cc], ch_b[cc]); };
  // phase 1: interior columns, VEC pixels per load, UNR independent loads in flight per thread
  constexpr int UNR = VEC == 8 ? 4 : 2;
  const int nvec = ps / VEC;
  const int work = rows * 64 * nvec;
  for (int base = threadIdx.x; base < work; base += blockDim.x * UNR) {
    uint4 raw[UNR];
    int kk[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int k = base + u * blockDim.x;
      kk[u] = k;
      raw[u] = make_uint4(0, 0, 0, 0);
      if (k < work) {
        const int j = k % nvec;
        const int c = (k / nvec) % 64 + c0;
        const int fy = r0 + k / (nvec * 64);
        int q = p, sy = fy - off;
        if (FRAMES) {
          if (fy == 0) { q = __ldg(nbr + (int64_t)p * 8 + 0); sy = ps - 1; }
          else if (fy == F - 1) { q = __ldg(nbr + (int64_t)p * 8 + 4); sy = 0; }
        }
        if (q >= 0 && c < C) {
          const __nv_bfloat16* src = x + ((int64_t)q * C + c) * hw + sy * ps + j * VEC;
          if constexpr (VEC == 8) {
            raw[u] = __ldg(reinterpret_cast<const uint4*>(src));
          } else if constexpr (VEC == 4) {
            const uint2 t2 = __ldg(reinterpret_cast<const uint2*>(src));
            raw[u].x = t2.x; raw[u].y = t2.y;
          } else {
            raw[u].x = (uint32_t)__bfloat16_as_ushort(src[0]);
          }
        } else {
          kk[u] = -1 - k;  // zero halo / padding channel: write zeros
        }
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      int k = kk[u];
      const bool zero = k < 0;
      if (zero) k = -1 - k;
      if (k >= work) continue;
      const int j = k % nvec;
      const int cc = (k / nvec) % 64;
      const int r = k / (nvec * 64);
      float v[VEC];
      if constexpr (VEC == 1) {
        v[0] = __uint_as_float(raw[u].x << 16);
      } else {
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw[u]);
#pragma unroll
        for (int i = 0; i < VEC / 2; ++i) { v[2 * i] = __low2float(h[i]); v[2 * i + 1] = __high2float(h[i]); }
      }
#pragma unroll
      for (int i = 0; i < VEC; ++i) {
        const int fx = off + j * VEC + i;
        tile[((r * F) + fx) * 64 + (cc ^ sw(fx))] = __float2bfloat16_rn(zero ? 0.f : norm(v[i], cc));
      }
    }
  }
  // phase 1b: ring columns (frames only)
  if (FRAMES) {
    for (int k = threadIdx.x; k < rows * 64 * 2; k += blockDim.x) {
      const int side = k & 1;  // 0 = west, 1 = east
      const int c = (k >> 1) % 64 + c0;
      const int r = k / 128;
      const int fy = r0 + r;
      const int ry = fy == 0 ? -1 : (fy == F - 1 ? 1 : 0);
      const int d = side == 0 ? (ry < 0 ? 7 : (ry > 0 ? 5 : 6)) : (ry < 0 ? 1 : (ry > 0 ? 3 : 2));
      const int q = __ldg(nbr + (int64_t)p * 8 + d);
      const int sy = ry < 0 ? ps - 1 : (ry > 0 ? 0 : fy - 1);
      const int sx = side == 0 ? ps - 1 : 0;
      float v = 0.f;
      if (q >= 0 && c < C) v = norm(bf(x[((int64_t)q * C + c) * hw + sy * ps + sx]), c - c0);
      const int fx = side == 0 ? 0 : F - 1;
      tile[((r * F) + fx) * 64 + ((c - c0) ^ sw(fx))] = __float2bfloat16_rn(v);
    }
  }
  __syncthreads();
  // phase 2: 16-byte channel runs, consecutive threads -> consecutive 16B of one pixel row
  const int nout = rows * F * 8;
  for (int k = threadIdx.x; k < nout; k += blockDim.x) {
    const int g8 = k & 7;
    const int fx = (k >> 3) % F;
    const int r = (k >> 3) / F;
    const uint4 u = *reinterpret_cast<const uint4*>(tile + ((r * F) + fx) * 64 + ((g8 * 8) ^ sw(fx)));
    const int64_t pixel = ((int64_t)p * F + r0 + r) * F + fx;
    *reinterpret_cast<uint4*>(out + pixel * Cp + c0 + g8 * 8) = u;
  }
}

// Register-transposing NCHW -> CL copy with optional GroupNorm (C % 8 == 0, ps % 8 == 0).
// One thread = 8 channels x 8 consecutive pixels of one output row: eight 16-byte loads
// (one per channel row; 4-8 consecutive threads cover a 64-128 B channel row segment),
// an 8x8 bf16 transpose in registers with the per-channel affine applied in fp32, and
// eight 16-byte stores (one per pixel; 8 consecutive channel groups = 128 B of a pixel).
// No shared memory and no per-element index math: the kernel is a streaming copy.
// FRAMES adds the 1-pixel neighbour ring of patched.py:64-88 (zero outside the image):
// rows 0 / F-1 read the N / S neighbour's edge row through the same vector path, and
// the border columns are gathered per pixel (8 channels per thread).
// One 8-pixel x 8-channel unit u of patch p of the (framed) channels-last output; the
// units of a patch are [0, n_int) interior rows and [n_int, n_int + n_brd) frame columns.
// PUSH (every patch's frame is written in the same launch): no frame-column units -- the
// units holding column 0 / ps-1 of a row also store that pixel into the west / east
// neighbour's frame (the same value the neighbour's pull unit would compute: same image,
// same statistics), or zero their own frame column when that neighbour does not exist.
// The pull units gathered one pixel of 8 channel planes per thread (2 useful bytes per
// 32-byte sector, a third of the units).
// GroupNorm affine of request ri[p] for every channel: sab[c] = rstd * gamma[c],
// sab[Cp + c] = beta[c] - mean * sab[c] (the expressions of the other stitcher kernels).
__device__ __forceinline__ void frames_affine(const float* __restrict__ stats, const int32_t* __restrict__ ri,
                                              const float* __restrict__ gamma, const float* __restrict__ beta,
                                              int C, int Cp, int G, int p, float* sab) {
  const int req = __ldg(ri + p), cg = C / G;
  for (int c = threadIdx.x; c < C; c += blockDim.x) {
    const float* sp = stats + ((int64_t)req * G + c / cg) * 2;
    const float mu = __ldg(sp), rs = __ldg(sp + 1);
    const float a = rs * __ldg(gamma + c);
    sab[c] = a;
    sab[Cp + c] = __ldg(beta + c) - mu * a;
  }
  __syncthreads();
}

template <bool FRAMES, bool PUSH>
__device__ __forceinline__ void frames_t8_unit(const __nv_bfloat16* __restrict__ x, int C, int ps, int Cp, int mode,
                                               const float* sab, const int32_t* __restrict__ nbr, int p, int u,
                                               __nv_bfloat16* __restrict__ out) {
  const int F = FRAMES ? ps + 2 : ps, off = FRAMES ? 1 : 0;
  const int nPB = ps >> 3, nCG = Cp >> 3;
  const int hw = ps * ps;
  const int n_int = F * nPB * nCG;
  const int n_brd = FRAMES && !PUSH ? F * 2 * nCG : 0;
  if (u >= n_int + n_brd) return;
  int cg, fy, q, sy, pb = 0, side = 0, sx = 0;
  if (u < n_int) {
    // 4-8 consecutive lanes: the pixel blocks of one row (a 64-128 B run of each channel
    // plane); 8 consecutive channel groups: one 128 B run of each output pixel
    pb = u % nPB;
    cg = (u / nPB) % nCG;
    fy = u / (nPB * nCG);
    q = p;
    sy = fy - off;
    if (FRAMES) {
      if (fy == 0) { q = __ldg(nbr + (int64_t)p * 8 + 0); sy = ps - 1; }
      else if (fy == F - 1) { q = __ldg(nbr + (int64_t)p * 8 + 4); sy = 0; }
    }
  } else {
    const int v = u - n_int;
    side = v & 1;
    cg = (v >> 1) % nCG;
    fy = (v >> 1) / nCG;
    const int ry = fy == 0 ? -1 : (fy == F - 1 ? 1 : 0);
    const int d = side == 0 ? (ry < 0 ? 7 : (ry > 0 ? 5 : 6)) : (ry < 0 ? 1 : (ry > 0 ? 3 : 2));
    q = __ldg(nbr + (int64_t)p * 8 + d);
    sy = ry < 0 ? ps - 1 : (ry > 0 ? 0 : fy - 1);
    sx = side == 0 ? ps - 1 : 0;
  }
  const int c0 = cg * 8;
  const int64_t obase = ((int64_t)p * F + fy) * F;
  // PUSH: the row's column 0 / ps-1 pixel goes to the west / east neighbour's frame
  auto push_w = [&](uint4 v) {
    if (pb == 0) {
      const int wq = __ldg(nbr + (int64_t)p * 8 + 6);
      if (wq >= 0) *reinterpret_cast<uint4*>(out + (((int64_t)wq * F + fy) * F + F - 1) * Cp + c0) = v;
      else *reinterpret_cast<uint4*>(out + obase * Cp + c0) = make_uint4(0, 0, 0, 0);
    }
  };
  auto push_e = [&](uint4 v) {
    if (pb == nPB - 1) {
      const int eq = __ldg(nbr + (int64_t)p * 8 + 2);
      if (eq >= 0) *reinterpret_cast<uint4*>(out + ((int64_t)eq * F + fy) * F * Cp + c0) = v;
      else *reinterpret_cast<uint4*>(out + (obase + F - 1) * Cp + c0) = make_uint4(0, 0, 0, 0);
    }
  };
  if (q < 0 || c0 >= C) {  // outside the image (zero halo) or padding channels
    const uint4 z = make_uint4(0, 0, 0, 0);
    if (u < n_int) {
#pragma unroll
      for (int i = 0; i < 8; ++i) *reinterpret_cast<uint4*>(out + (obase + off + pb * 8 + i) * Cp + c0) = z;
      if (PUSH) {
        push_w(z);
        push_e(z);
      }
    } else {
      *reinterpret_cast<uint4*>(out + (obase + (side ? F - 1 : 0)) * Cp + c0) = z;
    }
    return;
  }
  float a[8], b[8];
  if (mode == 1) {  // the patch's per-channel affine, staged once per CTA (frames_affine)
    const float4* a4 = reinterpret_cast<const float4*>(sab + c0);
    const float4* b4 = reinterpret_cast<const float4*>(sab + Cp + c0);
    const float4 a0 = a4[0], a1 = a4[1], b0 = b4[0], b1 = b4[1];
    a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w; a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
    b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w; b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      a[j] = 1.f;
      b[j] = 0.f;
    }
  }
  const __nv_bfloat16* src = x + ((int64_t)q * C + c0) * hw + sy * ps;
  if (u < n_int) {
    uint4 raw[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) raw[j] = __ldg(reinterpret_cast<const uint4*>(src + (int64_t)j * hw + pb * 8));
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t w[4];
#pragma unroll
      for (int j2 = 0; j2 < 4; ++j2) {
        float v2[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int j = 2 * j2 + h;
          const uint32_t word = (&raw[j].x)[i >> 1];
          const float f = __uint_as_float((i & 1) ? (word & 0xFFFF0000u) : (word << 16));
          v2[h] = fmaf(f, a[j], b[j]);
        }
        w[j2] = pack_bf16(v2[0], v2[1]);
      }
      const uint4 wv = make_uint4(w[0], w[1], w[2], w[3]);
      *reinterpret_cast<uint4*>(out + (obase + off + pb * 8 + i) * Cp + c0) = wv;
      if (PUSH && i == 0) push_w(wv);
      if (PUSH && i == 7) push_e(wv);
    }
  } else {
    uint32_t w[4];
#pragma unroll
    for (int j2 = 0; j2 < 4; ++j2) {
      const float f0 = bf(src[(int64_t)(2 * j2) * hw + sx]), f1 = bf(src[(int64_t)(2 * j2 + 1) * hw + sx]);
      w[j2] = pack_bf16(fmaf(f0, a[2 * j2], b[2 * j2]), fmaf(f1, a[2 * j2 + 1], b[2 * j2 + 1]));
    }
    *reinterpret_cast<uint4*>(out + (obase + (side ? F - 1 : 0)) * Cp + c0) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

template <bool FRAMES, bool PUSH>
__global__ void __launch_bounds__(256, 3) frames_t8_kernel(const __nv_bfloat16* __restrict__ x, int C, int ps, int Cp,
                                                        int mode, const float* __restrict__ stats,
                                                        const int32_t* __restrict__ ri,
                                                        const int32_t* __restrict__ nbr, int G,
                                                        const float* __restrict__ gamma,
                                                        const float* __restrict__ beta,
                                                        const int32_t* __restrict__ plist,
                                                        const int32_t* __restrict__ n_dev,
                                                        __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  extern __shared__ __align__(16) float sab[];  // [2][Cp] (mode 1)
  if (n_dev != nullptr && (int)blockIdx.y >= *n_dev) return;  // past the device list length
  const int p = plist ? __ldg(plist + blockIdx.y) : (int)blockIdx.y;
  if (mode == 1) frames_affine(stats, ri, gamma, beta, C, Cp, G, p, sab);
  frames_t8_unit<FRAMES, PUSH>(x, C, ps, Cp, mode, sab, nbr, p, blockIdx.x * blockDim.x + threadIdx.x, out);
}

template <bool FRAMES>
static int launch_frames_vec(cudaStream_t st, const void* x, int P, int C, int ps, int Cp, int mode,
                             const float* stats, const int32_t* ri, const int32_t* nbr, int G, const float* gamma,
                             const float* beta, void* out, const int32_t* plist = nullptr, int n_list = 0,
                             const int32_t* n_dev = nullptr) {
  const int F = FRAMES ? ps + 2 : ps;
  if (n_dev && (ps % 8 || C % 8))
    return set_error(PS_ERR_INPUT, "frames: a device patch count needs ps %% 8 == 0 and C %% 8 == 0");
  if (ps % 8 == 0 && C % 8 == 0 && (!getenv_flag("PS_FRAMES_SMEM") || n_dev)) {
    // full launches push the frame columns; patch lists (split path: neighbours may be
    // ghosts nobody frames here) pull them
    static const bool pull = getenv_flag("PS_FRAMES_PULL");
    const bool push = FRAMES && plist == nullptr && !pull;
    const int units = F * (ps / 8) * (Cp / 8) + (FRAMES && !push ? F * 2 * (Cp / 8) : 0);
    dim3 g2((units + 255) / 256, plist ? n_list : P);
    const size_t sab_bytes = mode == 1 ? 2 * Cp * sizeof(float) : 0;  // <= 48 KB for Cp <= 6144
    if constexpr (FRAMES) {
      if (push) {
        launch_pdl(frames_t8_kernel<true, true>, g2, dim3(256), sab_bytes, st, (const __nv_bfloat16*)x, C, ps, Cp,
                   mode, stats, ri, nbr, G, gamma, beta, plist, n_dev, (__nv_bfloat16*)out);
        count_launch();
        return check_launch("frames_cl");
      }
    }
    launch_pdl(frames_t8_kernel<FRAMES, false>, g2, dim3(256), sab_bytes, st, (const __nv_bfloat16*)x, C, ps, Cp,
               mode, stats, ri, nbr, G, gamma, beta, plist, n_dev, (__nv_bfloat16*)out);
    count_launch();
    return check_launch(FRAMES ? "frames_cl" : "to_cl");
  }
  int R = 8;
  while (R > 1 && R * F * 64 * 2 > 96 * 1024) R >>= 1;
  const int smem = R * F * 64 * 2;
  dim3 grid(plist ? n_list : P, Cp / 64, (F + R - 1) / R);
  auto xb = (const __nv_bfloat16*)x;
  auto ob = (__nv_bfloat16*)out;
#define PS_FRAMES_LAUNCH(V)                                                                                      \
  {                                                                                                              \
    static bool attr = false;                                                                                    \
    if (!attr) {                                                                                                 \
      cudaFuncSetAttribute(frames_vec_kernel<FRAMES, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024); \
      attr = true;                                                                                               \
    }                                                                                                            \
    frames_vec_kernel<FRAMES, V><<<grid, 256, smem, st>>>(xb, C, ps, Cp, mode, stats, ri, nbr, G, gamma, beta, R, plist, ob); \
  }
  if (ps % 8 == 0) PS_FRAMES_LAUNCH(8)
  else if (ps % 4 == 0) PS_FRAMES_LAUNCH(4)
  else PS_FRAMES_LAUNCH(1)
#undef PS_FRAMES_LAUNCH
  count_launch();
  return check_launch(FRAMES ? "frames_cl" : "to_cl");
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
  launch_gn_partials((cudaStream_t)stream, x, P, C, ps_ * ps_, G, nullptr, P, partials);
  count_launch();
  return check_launch("gn_partials");
}

int ps_gn_partials_sub(void* stream, const void* x, int P, int C, int ps_, int G, const int32_t* patches, int n,
                       float* partials, const int32_t* n_dev) {
  if (G < 1 || C % G) return set_error(PS_ERR_INPUT, "groups=%d does not divide channels=%d", G, C);
  if (n < 0 || n > P) return set_error(PS_ERR_INPUT, "gn_partials_sub: %d patches listed for P=%d", n, P);
  if (n == 0) return PS_OK;
  launch_gn_partials((cudaStream_t)stream, x, P, C, ps_ * ps_, G, patches, n, partials, n_dev);
  count_launch();
  return check_launch("gn_partials_sub");
}

int ps_gn_finalize(void* stream, const float* partials, const int32_t* request_offset, int R, int G, int cg_hw,
                   float eps, float* stats) {
  if (R == 0) return PS_OK;
  launch_pdl(gn_finalize_kernel, dim3(R), dim3(G < 1024 ? ((G + 31) / 32) * 32 : 1024), 0, (cudaStream_t)stream,
             partials, request_offset, G, (int64_t)cg_hw, eps, stats);
  count_launch();
  return check_launch("gn_finalize");
}

int ps_to_cl(void* stream, const void* x, int P, int C, int ps_, int Cp, int mode, const float* stats,
             const int32_t* request_index, int G, const float* gamma, const float* beta, float eps, void* out) {
  if (Cp % 64 || Cp < C) return set_error(PS_ERR_INPUT, "to_cl: Cp must be >= C and a multiple of 64");
  if (mode == 1 && (G < 1 || C % G)) return set_error(PS_ERR_INPUT, "groups=%d does not divide channels=%d", G, C);
  const int64_t T = (int64_t)P * ps_ * ps_;
  if (T == 0) return PS_OK;
  if (mode != 2)
    return launch_frames_vec<false>((cudaStream_t)stream, x, P, C, ps_, Cp, mode, stats, request_index, nullptr, G,
                                    gamma, beta, out);
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
  return launch_frames_vec<true>((cudaStream_t)stream, x, P, C, ps_, Cp, mode, stats, request_index, neighbors, G,
                                 gamma, beta, out);
}

int ps_frames_cl_sub(void* stream, const void* x, int P, int C, int ps_, int Cp, int mode, const float* stats,
                     const int32_t* request_index, const int32_t* neighbors, int G, const float* gamma,
                     const float* beta, const int32_t* patches, int n, void* out, const int32_t* n_dev) {
  if (Cp % 64 || Cp < C) return set_error(PS_ERR_INPUT, "frames_cl: Cp must be >= C and a multiple of 64");
  if (mode == 1 && (G < 1 || C % G)) return set_error(PS_ERR_INPUT, "groups=%d does not divide channels=%d", G, C);
  if (n < 0 || n > P) return set_error(PS_ERR_INPUT, "frames_cl_sub: %d patches listed for P=%d", n, P);
  if (n == 0) return PS_OK;
  return launch_frames_vec<true>((cudaStream_t)stream, x, P, C, ps_, Cp, mode, stats, request_index, neighbors, G,
                                 gamma, beta, out, patches, n, n_dev);
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
