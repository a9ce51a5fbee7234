// Per-image self-attention over the heterogeneous CSP patch batch (K7).
//
// Reference: patched_self_attention (patched.py:154-176) stitches every image
// and calls attend_tokens / _attend_single (kernels.py:230-267): single head,
// D = C, softmax(q k^T / sqrt(D)) v in 256-row chunks.  Attention is
// permutation-equivariant in the tokens of one image, so this kernel works
// directly in CSP (patch-major) token order — no stitching — and restricts
// keys to the query tile's image via `img_tok0`.
//
// One CTA = one (image, 128-query) tile; keys stream in 128-token blocks.
//   S_j = Q K_j^T   : tcgen05 SS, M=128 N=128 K=Dp -> TMEM cols [S_COL, +128)
//   P_j = exp2(S_j*scale_log2 - m)   (softmax warps, fp32) -> bf16 into TMEM
//                                      cols [P_COL, +64) with tcgen05.st
//   O  += P_j V_j   : tcgen05 TS (A = P from TMEM), M=128 N=Dp K=128 -> O cols
// TMEM: O (Dp) + S (128) + P (64) <= 512 columns.  Keeping P in TMEM removes
// the P round trip through shared memory, and 128-key blocks halve the Q
// re-reads of the S MMAs: shared-memory bandwidth, not the tensor pipe, was the
// limit of the 64-key SS design.
// K streams in 16 KB (128 keys x 64 dims) chunks through one ring, V^T in
// (Dp x 64 keys) pieces through another.
// Online-softmax rescaling of O is lazy (only when the running max grows by
// more than 2^8).  Warp roles: w0 TMA producer, w1 S issuer, w2 TMEM
// allocator, w3 PV issuer, w4..w7 softmax + epilogue (thread = query row = TMEM lane).
#include "common.cuh"
#include "ps_internal.h"

namespace ps {

constexpr int AT_BM = 128;
constexpr int AT_BN = 128;
constexpr int AT_THREADS = 256;

template <int DP>
struct AttnCfg {
  static constexpr int KB = DP / 64;                 // 64-wide chunks of the head dim
  static constexpr int Q_BYTES = KB * AT_BM * 128;   // Q tile: KB swizzle columns of 128 rows
  static constexpr int K_SLOT = AT_BN * 128;         // 128 keys x 64 dims
  static constexpr int V_SLOT = DP * 128;            // DP dims x 64 keys (V^T piece)
  static constexpr int NV = 2;
  static constexpr int BUDGET = 227 * 1024 - Q_BYTES - NV * V_SLOT - 1024 - 512;
  static constexpr int NK = BUDGET / K_SLOT > 6 ? 6 : BUDGET / K_SLOT;
  static constexpr int PV_N = DP <= 256 ? DP : DP / 2;  // MMA N for O += P V
  static constexpr int PV_MMAS = DP / PV_N;
  static constexpr int O_COL = 0;
  static constexpr int S_COL = DP;                   // 128 fp32 columns
  static constexpr int P_COL = DP + 128;             // 64 columns of packed bf16 pairs
  static constexpr int TMEM_COLS = (P_COL + 64) <= 256 ? 256 : 512;
  static constexpr int SMEM = Q_BYTES + NK * K_SLOT + NV * V_SLOT + 1024 + 512;
  static_assert(NK >= 2, "not enough shared memory for the K ring");
  static_assert(P_COL + 64 <= 512, "TMEM budget");
  static_assert(PV_N % 16 == 0 && PV_N <= 256, "bad PV N");
};

// D[tmem] (+)= A[tmem] * B[smem]^T (A = P, bf16 packed in TMEM).
PS_DEV void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// warp-wide variant (elect.sync in the asm), as mma_bf16_ts_2sm_w
PS_DEV void mma_bf16_ts_w(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int DP>
__global__ void __launch_bounds__(AT_THREADS, 1)
    attn_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using Cfg = AttnCfg<DP>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned, derived from smem_raw by an integer offset so the compiler keeps the
  // shared address space (uintptr_t arithmetic made every access through it a generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + Cfg::Q_BYTES;
  uint8_t* sV = sK + Cfg::NK * Cfg::K_SLOT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + Cfg::NV * Cfg::V_SLOT);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = k_full + Cfg::NK;
  uint64_t* v_full = k_empty + Cfg::NK;
  uint64_t* v_empty = v_full + Cfg::NV;
  uint64_t* s_full = v_empty + Cfg::NV;
  uint64_t* s_free = s_full + 1;
  uint64_t* p_full = s_free + 1;
  uint64_t* p_free = p_full + 1;
  uint64_t* o_full = p_free + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = blockIdx.x;
  const int q0 = p.tile_q0[tile];
  const int img = p.tile_img[tile];
  const int k_img = p.img_tok0[img], k_end = p.img_tok0[img + 1];
  // split-KV: this tile's key blocks start at tile_kb0 (k_begin is its first key)
  const int kb0 = p.tile_kb0 ? p.tile_kb0[tile] : 0;
  const int k_begin = k_img + kb0 * AT_BN;
  const int n_kb = p.tile_nkb ? p.tile_nkb[tile] : (k_end - k_img + AT_BN - 1) / AT_BN;
  const int slot = p.tile_slot ? p.tile_slot[tile] : -1;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < Cfg::NK; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < Cfg::NV; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 128);
    mbar_init(p_full, 128);
    mbar_init(p_free, 1);
    mbar_init(o_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // profiling (p.dbg): cycles blocked per barrier class
  unsigned long long w_a = 0, w_b = 0, w_c = 0;
  const long long t_start = clock64();
  auto twait = [&](uint64_t* bar, uint32_t par, unsigned long long& acc) {
    if (p.dbg) {
      const long long t0 = clock64();
      mbar_wait(bar, par);
      acc += clock64() - t0;
    } else {
      mbar_wait(bar, par);
    }
  };
  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, Cfg::Q_BYTES);
      for (int kc = 0; kc < Cfg::KB; ++kc) tma_load_2d(sQ + kc * AT_BM * 128, &tmQ, q_full, kc * 64, q0);
      int ks = 0, vs = 0;
      uint32_t kph = 0, vph = 0;
      // key block j lives here or, for a split image, possibly in a peer GPU's buffers
      // (read over NVLink by TMA through that peer's tensor maps -- no gather copy)
      auto src_of = [&](int j, const CUtensorMap*& mk, const CUtensorMap*& mv, int& row) {
        const int tok = k_begin + j * AT_BN;
        mk = &tmK;
        mv = &tmV;
        row = tok;
        if (p.kb_src != nullptr) {
          const int s = __ldg(p.kb_src + tok / AT_BN);
          if (s >= 0) {
            mk = p.peer_maps + 2 * s;
            mv = p.peer_maps + 2 * s + 1;
            row = __ldg(p.kb_row + tok / AT_BN);
          }
        }
      };
      auto load_k = [&](int j) {
        const CUtensorMap *mk, *mv;
        int row;
        src_of(j, mk, mv, row);
        for (int kc = 0; kc < Cfg::KB; ++kc) {
          mbar_wait(&k_empty[ks], kph ^ 1);
          mbar_arrive_expect_tx(&k_full[ks], Cfg::K_SLOT);
          tma_load_2d(sK + ks * Cfg::K_SLOT, mk, &k_full[ks], kc * 64, row);
          if (++ks == Cfg::NK) { ks = 0; kph ^= 1; }
        }
      };
      auto load_v = [&](int j) {
        const CUtensorMap *mk, *mv;
        int row;
        src_of(j, mk, mv, row);
        for (int ka = 0; ka < 2; ++ka) {
          mbar_wait(&v_empty[vs], vph ^ 1);
          mbar_arrive_expect_tx(&v_full[vs], Cfg::V_SLOT);
          uint8_t* dst = sV + vs * Cfg::V_SLOT;
          for (int dc = 0; dc < Cfg::KB; ++dc)
            tma_load_2d(dst + dc * 64 * 128, mv, &v_full[vs], row + ka * 64, dc * 64);
          if (++vs == Cfg::NV) { vs = 0; vph ^= 1; }
        }
      };
      // consumption order of the MMA warp: S0, then (S_{j+1}, PV_j) per block
      load_k(0);
      for (int j = 0; j < n_kb; ++j) {
        if (j + 1 < n_kb) load_k(j + 1);
        load_v(j);
      }
    }
  } else if (warp == 1 || warp == 3) {
    // ---------------------------------------------------------- MMA issuers
    // w1 issues S_j = Q K_j^T, w3 issues O += P_j V_j.  Two issuing threads keep
    // the tensor pipe fed while either one waits on a barrier: a wait costs the
    // issuer ~76 clk even when the phase already completed, and the MMA queue
    // of one thread is too shallow to cover it (tools/micro/mma_contention.cu:
    // one issuer with a wait per 4 N128 MMAs -> 77% of peak, two issuers -> 100%).
    constexpr uint32_t idesc_s = idesc_bf16_f32(AT_BM, AT_BN);
    constexpr uint32_t idesc_o = idesc_bf16_f32(AT_BM, Cfg::PV_N);
    mbar_wait(q_full, 0);
    if (warp == 1) {
      int ks = 0;
      uint32_t kph = 0;
      for (int j = 0; j < n_kb; ++j) {
        // S buffer is free once the softmax warps loaded S_{j-1}
        if (j >= 1) twait(s_free, (j - 1) & 1, w_a);
        tc_fence_after();
        for (int kc = 0; kc < Cfg::KB; ++kc) {
          twait(&k_full[ks], kph, w_c);
          tc_fence_after();
          {  // the converged warp issues (elect.sync in the asm; see attention2.cu)
            const uint64_t dq = sdesc_sw128(sQ + kc * AT_BM * 128), dk = sdesc_sw128(sK + ks * Cfg::K_SLOT);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_bf16_ss_w(tmem + Cfg::S_COL, dq + (uint64_t)(k * 2), dk + (uint64_t)(k * 2), idesc_s, (kc | k) != 0);
            mma_commit_w(&k_empty[ks]);
            if (kc == Cfg::KB - 1) mma_commit_w(s_full);
          }
          if (++ks == Cfg::NK) { ks = 0; kph ^= 1; }
        }
      }
    } else {
      int vs = 0;
      uint32_t vph = 0;
      for (int j = 0; j < n_kb; ++j) {
        twait(p_full, j & 1, w_b);
        tc_fence_after();
        for (int ka = 0; ka < 2; ++ka) {
          twait(&v_full[vs], vph, w_c);
          tc_fence_after();
          {
            const uint64_t dv = sdesc_sw128(sV + vs * Cfg::V_SLOT);
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
              for (int n = 0; n < Cfg::PV_MMAS; ++n)
                mma_bf16_ts_w(tmem + Cfg::O_COL + n * Cfg::PV_N, tmem + Cfg::P_COL + ka * 32 + k * 8,
                              dv + (uint64_t)((n * Cfg::PV_N * 128 + k * 32) >> 4), idesc_o, (j | ka | k) != 0);
            mma_commit_w(&v_empty[vs]);
            if (ka == 1) {
              mma_commit_w(p_free);
              if (j == n_kb - 1) mma_commit_w(o_full);
            }
          }
          if (++vs == Cfg::NV) { vs = 0; vph ^= 1; }
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ softmax + epilogue
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < n_kb; ++j) {
      twait(s_full, j & 1, w_a);
      tc_fence_after();
      uint32_t sr[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) PS_TMEM_LD32(tmem + lane_base + Cfg::S_COL + 32 * c, (sr + 32 * c));
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(s_free);
      const int kvalid = k_end - (k_begin + j * AT_BN);  // keys valid in this block
      if (kvalid < AT_BN) {  // only the last block of an image can be ragged
#pragma unroll
        for (int i = 0; i < 128; ++i)
          if (i >= kvalid) sr[i] = __float_as_uint(-INFINITY);
      }
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int i = 0; i < 128; i += 4) {
        mx0 = fmaxf(mx0, fmaxf(__uint_as_float(sr[i]), __uint_as_float(sr[i + 1])));
        mx1 = fmaxf(mx1, fmaxf(__uint_as_float(sr[i + 2]), __uint_as_float(sr[i + 3])));
      }
      const float mx = fmaxf(mx0, mx1) * p.scale_log2;  // scale_log2 > 0
      // lazy rescale: keep the stale max unless it grew by more than 8 (log2 units)
      float m_use = m_run;
      const bool need = (m_run == -INFINITY) || (mx > m_run + 8.0f);
      if (need) m_use = fmaxf(mx, m_run);
      const float alpha = (m_run == -INFINITY) ? 0.f : ex2_approx(m_run - m_use);
      const float neg = -m_use;
      float sum0 = 0.f, sum1 = 0.f;
#pragma unroll
      for (int i = 0; i < 64; ++i) {
        const float a = ex2_approx(fmaf(__uint_as_float(sr[2 * i]), p.scale_log2, neg));
        const float b = ex2_approx(fmaf(__uint_as_float(sr[2 * i + 1]), p.scale_log2, neg));
        sum0 += a;
        sum1 += b;
        sr[i] = pack_bf16(a, b);  // packed P overwrites the consumed half of sr
      }
      l_run = l_run * alpha + (sum0 + sum1);
      // P columns and O are owned by the MMAs of block j-1 until they complete
      if (j >= 1) twait(p_free, (j - 1) & 1, w_b);
      tc_fence_after();
      const bool warp_rescale = __any_sync(0xffffffffu, need && j >= 1 && alpha != 1.f);
      if (warp_rescale) {
        const float sc = (need && j >= 1) ? alpha : 1.f;
#pragma unroll 1
        for (int c = 0; c < DP; c += 16) {
          uint32_t o[16];
          PS_TMEM_LD16(tmem + lane_base + Cfg::O_COL + c, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * sc);
          PS_TMEM_ST16(tmem + lane_base + Cfg::O_COL + c, o);
        }
      }
      m_run = m_use;
#pragma unroll
      for (int c = 0; c < 4; ++c) PS_TMEM_ST16(tmem + lane_base + Cfg::P_COL + 16 * c, (sr + 16 * c));
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    // epilogue: O / l -> bf16 channels-last (or the unnormalised split-KV partial)
    mbar_wait(o_full, 0);
    tc_fence_after();
    const int q = q0 + row;
    const bool ok = q < k_end;
    if (slot >= 0) {
      float* po = p.part_o + ((size_t)slot * AT_BM + row) * DP;
      if (row < AT_BM) {
        p.part_ml[((size_t)slot * AT_BM + row) * 2] = m_run;
        p.part_ml[((size_t)slot * AT_BM + row) * 2 + 1] = l_run;
      }
#pragma unroll 1
      for (int c = 0; c < DP; c += 32) {
        uint32_t o[32];
        PS_TMEM_LD32(tmem + lane_base + Cfg::O_COL + c, o);
        tmem_ld_wait();
        float4* d4 = reinterpret_cast<float4*>(po + c);
#pragma unroll
        for (int v = 0; v < 8; ++v)
          d4[v] = make_float4(__uint_as_float(o[4 * v]), __uint_as_float(o[4 * v + 1]), __uint_as_float(o[4 * v + 2]),
                              __uint_as_float(o[4 * v + 3]));
      }
    } else {
    const float inv = 1.f / l_run;
    __nv_bfloat16* dst = p.out + (size_t)q * p.Dp;
#pragma unroll 1
    for (int c = 0; c < DP; c += 32) {
      uint32_t o[32];
      PS_TMEM_LD32(tmem + lane_base + Cfg::O_COL + c, o);
      tmem_ld_wait();
      if (ok) {
        uint4* d4 = reinterpret_cast<uint4*>(dst + c);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(o[8 * v + 0]) * inv, __uint_as_float(o[8 * v + 1]) * inv);
          w.y = pack_bf16(__uint_as_float(o[8 * v + 2]) * inv, __uint_as_float(o[8 * v + 3]) * inv);
          w.z = pack_bf16(__uint_as_float(o[8 * v + 4]) * inv, __uint_as_float(o[8 * v + 5]) * inv);
          w.w = pack_bf16(__uint_as_float(o[8 * v + 6]) * inv, __uint_as_float(o[8 * v + 7]) * inv);
          d4[v] = w;
        }
      }
    }
    }
  }
  if (p.dbg && lane == 0) {
    const unsigned long long tot = clock64() - t_start;
    // [0] mma:s_free [1] mma:p_full [2] mma:k/v_full [3] mma total [4] softmax:s_full [5] softmax:p_free [6] sm total
    if (warp == 1) { atomicAdd(p.dbg + 0, w_a); atomicAdd(p.dbg + 2, w_c); atomicAdd(p.dbg + 3, tot); }
    if (warp == 3) { atomicAdd(p.dbg + 1, w_b); atomicAdd(p.dbg + 2, w_c); }
    if (warp == 4) { atomicAdd(p.dbg + 4, w_a); atomicAdd(p.dbg + 5, w_b); atomicAdd(p.dbg + 6, tot); }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, Cfg::TMEM_COLS);
}

template <int DP>
static int launch_dp(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v, const AttnParams& p,
                     cudaStream_t st) {
  using Cfg = AttnCfg<DP>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_kernel<DP>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    attr = true;
  }
  attn_kernel<DP><<<p.n_tiles, AT_THREADS, Cfg::SMEM, st>>>(q, k, v, p);
  count_launch();
  return check_launch("attention");
}

// Split-KV combine: query tile i has partials in slots [slot0[i], slot0[i] + nsplit[i]);
// O = sum_s 2^(m_s - M) O_s / sum_s 2^(m_s - M) l_s, M = max_s m_s (m in log2 units).
// grid = (tiles, AT_BM / CMB_ROWS), 256 threads; thread = (row, 8 columns).  (One CTA per tile
// left 96 CTAs streaming ~1 MB of partials each at config 5 / 8 ranks: 110 us per launch.)
constexpr int CMB_ROWS = 16;
__global__ void __launch_bounds__(256) attn_combine_kernel(const float* __restrict__ part_o,
                                                           const float* __restrict__ part_ml,
                                                           const int* __restrict__ q0s, const int* __restrict__ slot0,
                                                           const int* __restrict__ nsplit,
                                                           const int* __restrict__ img_of, const int* __restrict__ img_tok0,
                                                           int Dp, __nv_bfloat16* __restrict__ out) {
  const int i = blockIdx.x;
  const int q0 = __ldg(q0s + i), s0 = __ldg(slot0 + i), ns = __ldg(nsplit + i);
  const int k_end = __ldg(img_tok0 + __ldg(img_of + i) + 1);
  const int groups = Dp / 8;
  for (int w = threadIdx.x; w < CMB_ROWS * groups; w += blockDim.x) {
    const int row = blockIdx.y * CMB_ROWS + w / groups, c = (w % groups) * 8;
    if (q0 + row >= k_end) continue;
    float M = -INFINITY;
    for (int s = 0; s < ns; ++s) M = fmaxf(M, __ldg(part_ml + ((size_t)(s0 + s) * AT_BM + row) * 2));
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    float L = 0.f;
    for (int s = 0; s < ns; ++s) {
      const size_t r = (size_t)(s0 + s) * AT_BM + row;
      const float m = __ldg(part_ml + r * 2), l = __ldg(part_ml + r * 2 + 1);
      const float wgt = m == -INFINITY ? 0.f : exp2f(m - M);
      L += wgt * l;
      const float4* src = reinterpret_cast<const float4*>(part_o + r * Dp + c);
      const float4 a = __ldg(src), b = __ldg(src + 1);
      acc[0] += wgt * a.x; acc[1] += wgt * a.y; acc[2] += wgt * a.z; acc[3] += wgt * a.w;
      acc[4] += wgt * b.x; acc[5] += wgt * b.y; acc[6] += wgt * b.z; acc[7] += wgt * b.w;
    }
    const float inv = 1.f / L;
    uint4 o;
    o.x = pack_bf16(acc[0] * inv, acc[1] * inv);
    o.y = pack_bf16(acc[2] * inv, acc[3] * inv);
    o.z = pack_bf16(acc[4] * inv, acc[5] * inv);
    o.w = pack_bf16(acc[6] * inv, acc[7] * inv);
    *reinterpret_cast<uint4*>(out + (size_t)(q0 + row) * Dp + c) = o;
  }
}

int attention_combine_launch(const float* part_o, const float* part_ml, const int* q0s, const int* slot0,
                             const int* nsplit, const int* img_of, const int* img_tok0, int n, int Dp,
                             __nv_bfloat16* out, cudaStream_t st) {
  if (n == 0) return PS_OK;
  attn_combine_kernel<<<dim3(n, AT_BM / CMB_ROWS), 256, 0, st>>>(part_o, part_ml, q0s, slot0, nsplit, img_of, img_tok0, Dp, out);
  count_launch();
  return check_launch("attention_combine");
}

int attention_launch(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& vt, const AttnParams& p, int dp,
                     cudaStream_t st) {
  switch (dp) {
    case 64: return launch_dp<64>(q, k, vt, p, st);
    case 128: return launch_dp<128>(q, k, vt, p, st);
    case 192: return launch_dp<192>(q, k, vt, p, st);
    case 256: return launch_dp<256>(q, k, vt, p, st);
    case 320: return launch_dp<320>(q, k, vt, p, st);
    default: return set_error(PS_ERR_INPUT, "attention: unsupported head dim %d", dp);
  }
}

}  // namespace ps
