// Per-image self-attention on CTA pairs (cta_group::2) -- the default attention path
// (PS_ATTN_PAIRS=0 selects the single-CTA kernel in attention.cu).  attn2p_kernel (persistent,
// tiles from an atomic ticket) is the production kernel; attn2_kernel (one tile per CTA pair,
// PS_ATTN_PERSIST=0) is kept as the A/B baseline.
//
// Same math as attention.cu (reference patched.py:154-176 -> kernels.py:230-267,
// one head, D = C, keys restricted to the query tile's image), but each cluster of
// two CTAs on one TPC owns 256 queries and issues M=256 tcgen05 MMAs:
//   * CTA r holds its own 128 query rows (Q in smem, S/P/O in its TMEM lanes);
//   * every 128-key block is split between the pair: CTA r loads keys
//     [64r, 64r+64) of K and half of the V^T rows of each PV MMA;
//   * the leader (rank 0) issues all MMAs; TMA loads of both CTAs complete on the
//     leader's barriers; MMA completions are multicast to both CTAs.
// Per SM this halves the K/V bytes loaded and read by the tensor core (shared-memory
// operand bandwidth is what limits the single-CTA kernel).
#include <stdlib.h>

#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "ps_internal.h"

namespace ps {

constexpr int A2_BM = 128;  // query rows per CTA (256 per pair)
constexpr int A2_BN = 128;  // keys per block (64 per CTA)
constexpr int A2_THREADS = 256;
#ifndef A2_WARP_ISSUE  // MMA issue by the converged warp (elect.sync in the asm) instead of lane 0
#define A2_WARP_ISSUE 1
#endif
#ifndef A2_KWAIT
#define A2_KWAIT 5  // K chunks the persistent kernel's S issuer waits for before issuing their MMAs
#endif

template <int DP, int NV_ = 4>
struct Attn2Cfg {
  static constexpr int KB = DP / 64;
  static constexpr int Q_BYTES = KB * A2_BM * 128;
  static constexpr int K_SLOT = (A2_BN / 2) * 128;          // 64 keys x 64 dims, this CTA's half
  static constexpr int PV_N = DP <= 256 ? DP : DP / 2;       // N of one PV MMA
  static constexpr int PV_MMAS = DP / PV_N;
  static constexpr int V_ROWS = PV_N / 2;                   // V^T rows per CTA per PV MMA
  static constexpr int V_SLOT = PV_MMAS * V_ROWS * 128;     // one 64-key atom, this CTA's rows
  static constexpr int NV = NV_;  // V ring (64-key slots); 3 leaves room for 10 K slots (2 key blocks)
  static constexpr int BUDGET = 227 * 1024 - Q_BYTES - NV * V_SLOT - 1024 - 512 - 2048;
  static constexpr int NK = BUDGET / K_SLOT > 10 ? 10 : BUDGET / K_SLOT;
  static constexpr int O_COL = 0;
  static constexpr int S_COL = DP;
  static constexpr int P_COL = DP + 128;
  static constexpr int TMEM_COLS = (P_COL + 64) <= 256 ? 256 : 512;
  static constexpr int SMEM = Q_BYTES + NK * K_SLOT + NV * V_SLOT + 1024 + 512 + 2048;
  static_assert(NK >= 4, "K ring too small");
  static_assert(V_ROWS % 8 == 0, "V^T half rows must be whole swizzle atoms");
};

// trace events (profiling): [ev * 64 + block], block < 64, first pair's leader CTA only
#define A2_TRACE(ev, j)                                                                  \
  if (p.trace != nullptr && blockIdx.x == 0 && (j) < 64) p.trace[(ev) * 64 + (j)] = clock64();

template <int DP, int NV_>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(A2_THREADS, 1)
    attn2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                 const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                 const AttnParams p) {
  if (threadIdx.x == 0) { A2_TRACE(11, 0) }  // kernel entry (profiling)
  pdl_wait();
  using Cfg = Attn2Cfg<DP, NV_>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned, derived from smem_raw by an integer offset so the compiler keeps the
  // shared address space (uintptr_t arithmetic made every access through it a generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + Cfg::Q_BYTES;
  uint8_t* sV = sK + Cfg::NK * Cfg::K_SLOT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + Cfg::NV * Cfg::V_SLOT);
  uint64_t* q_full = bars;                    // leader
  uint64_t* k_full = bars + 1;                // leader
  uint64_t* k_empty = k_full + Cfg::NK;       // both (multicast commit)
  uint64_t* v_full = k_empty + Cfg::NK;       // leader
  uint64_t* v_empty = v_full + Cfg::NV;       // both
  uint64_t* s_full = v_empty + Cfg::NV;       // both
  uint64_t* s_free = s_full + 1;              // leader, 256 arrivals
  uint64_t* p_full = s_free + 1;              // leader, 256 arrivals
  uint64_t* p_free = p_full + 1;              // both
  uint64_t* o_full = p_free + 1;              // both
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1;
  if (p.n_dev != nullptr && pair >= *p.n_dev) return;  // past the device tile count (both CTAs)
  const int q0 = p.tile_q0[pair] + (int)rank * A2_BM;
  const int img = p.tile_img[pair];
  const int k_begin = p.img_tok0[img], k_end = p.img_tok0[img + 1];
  const int n_kb = (k_end - k_begin + A2_BN - 1) / A2_BN;

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
    mbar_init(s_free, 2 * 128);
    mbar_init(p_full, 2 * 128);
    mbar_init(p_free, 1);
    mbar_init(o_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_2sm(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

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
    // -------------------------------------------------- producer (both CTAs)
    if (lane == 0) {
      const uint32_t lq = mapa_shared(q_full, 0);
      if (leader) mbar_arrive_expect_tx(q_full, 2 * Cfg::Q_BYTES);
      for (int kc = 0; kc < Cfg::KB; ++kc) tma_load_2d_2sm(sQ + kc * A2_BM * 128, &tmQ, lq, kc * 64, q0);
      int ks = 0, vs = 0;
      uint32_t kph = 0, vph = 0;
      auto load_k = [&](int j) {
        for (int kc = 0; kc < Cfg::KB; ++kc) {
          mbar_wait(&k_empty[ks], kph ^ 1);
#ifdef A2_NOLOAD  // profiling only: K slots keep stale data (no TMA traffic)
          if (leader) mbar_arrive(&k_full[ks]);
#else
          if (leader) mbar_arrive_expect_tx(&k_full[ks], 2 * Cfg::K_SLOT);
          tma_load_2d_2sm(sK + ks * Cfg::K_SLOT, &tmK, mapa_shared(&k_full[ks], 0), kc * 64,
                          k_begin + j * A2_BN + (int)rank * (A2_BN / 2));
#endif
          if (++ks == Cfg::NK) { ks = 0; kph ^= 1; }
        }
      };
      auto load_v = [&](int j) {
        for (int ka = 0; ka < 2; ++ka) {
          mbar_wait(&v_empty[vs], vph ^ 1);
#ifdef A2_NOLOAD
          if (leader) mbar_arrive(&v_full[vs]);
#else
          if (leader) mbar_arrive_expect_tx(&v_full[vs], 2 * Cfg::V_SLOT);
          const uint32_t lb = mapa_shared(&v_full[vs], 0);
          uint8_t* dst = sV + vs * Cfg::V_SLOT;
          for (int n = 0; n < Cfg::PV_MMAS; ++n)
            tma_load_2d_2sm(dst + n * Cfg::V_ROWS * 128, &tmV, lb, k_begin + j * A2_BN + ka * 64,
                            n * Cfg::PV_N + (int)rank * Cfg::V_ROWS);
#endif
          if (++vs == Cfg::NV) { vs = 0; vph ^= 1; }
        }
      };
      load_k(0);
      for (int j = 0; j < n_kb; ++j) {
        if (j + 1 < n_kb) load_k(j + 1);
        load_v(j);
      }
    }
  } else if (warp == 1 || warp == 3) {
    // ------------------------------- MMA issuers (leader only): w1 S = Q K^T, w3 O += P V
    // Two issuing threads keep the pair's tensor pipes fed while either waits on a
    // barrier (as in attention.cu).
    if (leader) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(2 * A2_BM, A2_BN);
      constexpr uint32_t idesc_o = idesc_bf16_f32(2 * A2_BM, Cfg::PV_N);
      // descriptor bases: the start-address field is (smem address >> 4) in the low bits, so an
      // operand offset is a plain add (no carry: smem < 256 KB); fewer dependent ops per issue
      const uint64_t dq0 = sdesc_sw128(sQ), dk0 = sdesc_sw128(sK), dv0 = sdesc_sw128(sV);
      mbar_wait(q_full, 0);
      if (warp == 1) {
        int ks = 0;
        uint32_t kph = 0;
        for (int j = 0; j < n_kb; ++j) {
          if (j >= 1) twait(s_free, (j - 1) & 1, w_a);
          tc_fence_after();
          if (lane == 0) { A2_TRACE(0, j) }
          long long kw = 0;
          {  // the block's K chunks first, then its MMAs back to back (as attn2p_kernel)
            const long long tk0 = p.trace ? clock64() : 0;
            int k2 = ks;
            uint32_t p2 = kph;
            for (int kc = 0; kc < Cfg::KB; ++kc) {
              twait(&k_full[k2], p2, w_c);
              if (++k2 == Cfg::NK) { k2 = 0; p2 ^= 1; }
            }
            if (p.trace) kw += clock64() - tk0;
            tc_fence_after();
          }
          for (int kc = 0; kc < Cfg::KB; ++kc) {
            const uint64_t dq = dq0 + (uint64_t)((kc * A2_BM * 128) >> 4);
            const uint64_t dk = dk0 + (uint64_t)((ks * Cfg::K_SLOT) >> 4);
#if A2_WARP_ISSUE
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_bf16_ss_2sm_w(tmem + Cfg::S_COL, dq + (uint64_t)(k * 2), dk + (uint64_t)(k * 2), idesc_s,
                                (kc | k) != 0);
            mma_commit_2sm_w(&k_empty[ks], 0x3);
            if (kc == Cfg::KB - 1) mma_commit_2sm_w(s_full, 0x3);
#else
            if (lane == 0) {
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_bf16_ss_2sm(tmem + Cfg::S_COL, dq + (uint64_t)(k * 2), dk + (uint64_t)(k * 2), idesc_s,
                                (kc | k) != 0);
              mma_commit_2sm(&k_empty[ks], 0x3);
              if (kc == Cfg::KB - 1) mma_commit_2sm(s_full, 0x3);
            }
            __syncwarp();
#endif
            if (++ks == Cfg::NK) { ks = 0; kph ^= 1; }
          }
          if (lane == 0) { A2_TRACE(1, j) }
          if (lane == 0 && p.trace != nullptr && blockIdx.x == 0 && j < 64) p.trace[9 * 64 + j] = kw;
        }
      } else {
        int vs = 0;
        uint32_t vph = 0;
        for (int j = 0; j < n_kb; ++j) {
          twait(p_full, j & 1, w_b);
          tc_fence_after();
          if (lane == 0) { A2_TRACE(2, j) }
          long long vw = 0;
          for (int ka = 0; ka < 2; ++ka) {
            const long long tv0 = p.trace ? clock64() : 0;
            twait(&v_full[vs], vph, w_c);
            if (p.trace) vw += clock64() - tv0;
            tc_fence_after();
            const uint64_t dv = dv0 + (uint64_t)((vs * Cfg::V_SLOT) >> 4);
#if A2_WARP_ISSUE
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
              for (int n = 0; n < Cfg::PV_MMAS; ++n)
                mma_bf16_ts_2sm_w(tmem + Cfg::O_COL + n * Cfg::PV_N, tmem + Cfg::P_COL + ka * 32 + k * 8,
                                  dv + (uint64_t)((n * Cfg::V_ROWS * 128 + k * 32) >> 4), idesc_o,
                                  (j | ka | k) != 0);
            mma_commit_2sm_w(&v_empty[vs], 0x3);
            if (ka == 1) {
              mma_commit_2sm_w(p_free, 0x3);
              if (j == n_kb - 1) mma_commit_2sm_w(o_full, 0x3);
            }
#else
            if (lane == 0) {
#pragma unroll
              for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int n = 0; n < Cfg::PV_MMAS; ++n)
                  mma_bf16_ts_2sm(tmem + Cfg::O_COL + n * Cfg::PV_N, tmem + Cfg::P_COL + ka * 32 + k * 8,
                                  dv + (uint64_t)((n * Cfg::V_ROWS * 128 + k * 32) >> 4), idesc_o,
                                  (j | ka | k) != 0);
              mma_commit_2sm(&v_empty[vs], 0x3);
              if (ka == 1) {
                mma_commit_2sm(p_free, 0x3);
                if (j == n_kb - 1) mma_commit_2sm(o_full, 0x3);
              }
            }
            __syncwarp();
#endif
            if (++vs == Cfg::NV) { vs = 0; vph ^= 1; }
          }
          if (lane == 0) { A2_TRACE(3, j) }
          if (lane == 0 && p.trace != nullptr && blockIdx.x == 0 && j < 64) p.trace[10 * 64 + j] = vw;
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ softmax + epilogue
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const uint32_t s_free_l = mapa_shared(s_free, 0);
    const uint32_t p_full_l = mapa_shared(p_full, 0);
    float m_run = -INFINITY, l_run = 0.f;
    for (int j = 0; j < n_kb; ++j) {
      twait(s_full, j & 1, w_a);
      tc_fence_after();
      if (threadIdx.x == 128) { A2_TRACE(4, j) }
      uint32_t sr[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) PS_TMEM_LD32(tmem + lane_base + Cfg::S_COL + 32 * c, (sr + 32 * c));
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive_cluster(s_free_l);
      if (threadIdx.x == 128) { A2_TRACE(5, j) }
      const int kvalid = k_end - (k_begin + j * A2_BN);  // keys valid in this block
      if (kvalid < A2_BN) {  // only the last block of an image can be ragged
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
#ifdef A2_EXP_OFF  // profiling only: no exponentials
        const float a = fmaf(__uint_as_float(sr[2 * i]), p.scale_log2, neg);
        const float b = fmaf(__uint_as_float(sr[2 * i + 1]), p.scale_log2, neg);
#else
        const float a = ex2_approx(fmaf(__uint_as_float(sr[2 * i]), p.scale_log2, neg));
        const float b = ex2_approx(fmaf(__uint_as_float(sr[2 * i + 1]), p.scale_log2, neg));
#endif
        sum0 += a;
        sum1 += b;
        sr[i] = pack_bf16(a, b);  // packed P overwrites the consumed half of sr
      }
      l_run = l_run * alpha + (sum0 + sum1);
      if (threadIdx.x == 128) { A2_TRACE(6, j) }
      // P columns and O are owned by the MMAs of block j-1 until they complete
      if (j >= 1) twait(p_free, (j - 1) & 1, w_b);
      tc_fence_after();
      if (threadIdx.x == 128) { A2_TRACE(7, j) }
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
      mbar_arrive_cluster(p_full_l);
      if (threadIdx.x == 128) { A2_TRACE(8, j) }
    }
    // epilogue: O / l -> bf16 channels-last
    mbar_wait(o_full, 0);
    tc_fence_after();
    if (threadIdx.x == 128) { A2_TRACE(12, 0) }
    const int q = q0 + row;
    const bool ok = q < k_end;
    const float inv = 1.f / l_run;
    // up to EPI_G TMEM loads of 32 columns in flight per wait
    constexpr int EPI_G = (DP / 32) % 5 == 0 ? 5 : (DP / 32) % 4 == 0 ? 4 : (DP / 32) % 3 == 0 ? 3 : (DP / 32) % 2 == 0 ? 2 : 1;
    if (p.epi_tma && q0 + A2_BM <= k_end) {
      // whole tile: stage O (bf16) in the Q buffer -- free once the last S MMA completed, and
      // already laid out as the TMA boxes [64 columns][128 rows] with 128-byte swizzle -- and
      // leave through TMA stores: per-thread 16-byte row stores (32 rows 640 B apart per
      // warp instruction) made the epilogue ~8k cycles per tile
      uint8_t* srow = sQ + row * 128;
#pragma unroll 1
      for (int c0 = 0; c0 < DP; c0 += 32 * EPI_G) {
        uint32_t o[EPI_G][32];
#pragma unroll
        for (int g = 0; g < EPI_G; ++g) PS_TMEM_LD32(tmem + lane_base + Cfg::O_COL + c0 + 32 * g, o[g]);
        tmem_ld_wait();
#pragma unroll
        for (int g = 0; g < EPI_G; ++g) {
          reg_fence32(o[g]);
          const int col = c0 + 32 * g;
          uint8_t* box = srow + (col >> 6) * (A2_BM * 128);
          const int j0 = (col & 63) >> 3;
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            uint4 w;
            w.x = pack_bf16(__uint_as_float(o[g][8 * v + 0]) * inv, __uint_as_float(o[g][8 * v + 1]) * inv);
            w.y = pack_bf16(__uint_as_float(o[g][8 * v + 2]) * inv, __uint_as_float(o[g][8 * v + 3]) * inv);
            w.z = pack_bf16(__uint_as_float(o[g][8 * v + 4]) * inv, __uint_as_float(o[g][8 * v + 5]) * inv);
            w.w = pack_bf16(__uint_as_float(o[g][8 * v + 6]) * inv, __uint_as_float(o[g][8 * v + 7]) * inv);
            *reinterpret_cast<uint4*>(box + (((j0 + v) ^ (row & 7)) << 4)) = w;
          }
        }
      }
      fence_proxy_async();
      named_bar_sync(1, 128);
      if (threadIdx.x == 128) {
        for (int kc = 0; kc < Cfg::KB; ++kc) tma_store_2d(&tmO, sQ + kc * A2_BM * 128, kc * 64, q0);
        bulk_commit();
        bulk_wait_read<0>();  // the Q buffer is read by the TMA engine before the CTA exits
      }
    } else {
      __nv_bfloat16* dst = p.out + (size_t)q * p.Dp;
#pragma unroll 1
      for (int c0 = 0; c0 < DP; c0 += 32 * EPI_G) {
        uint32_t o[EPI_G][32];
#pragma unroll
        for (int g = 0; g < EPI_G; ++g) PS_TMEM_LD32(tmem + lane_base + Cfg::O_COL + c0 + 32 * g, o[g]);
        tmem_ld_wait();
#pragma unroll
        for (int g = 0; g < EPI_G; ++g) reg_fence32(o[g]);
        if (ok) {
#pragma unroll
          for (int g = 0; g < EPI_G; ++g) {
            uint4* d4 = reinterpret_cast<uint4*>(dst + c0 + 32 * g);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              uint4 w;
              w.x = pack_bf16(__uint_as_float(o[g][8 * v + 0]) * inv, __uint_as_float(o[g][8 * v + 1]) * inv);
              w.y = pack_bf16(__uint_as_float(o[g][8 * v + 2]) * inv, __uint_as_float(o[g][8 * v + 3]) * inv);
              w.z = pack_bf16(__uint_as_float(o[g][8 * v + 4]) * inv, __uint_as_float(o[g][8 * v + 5]) * inv);
              w.w = pack_bf16(__uint_as_float(o[g][8 * v + 6]) * inv, __uint_as_float(o[g][8 * v + 7]) * inv);
              d4[v] = w;
            }
          }
        }
      }
    }
  }
  if (threadIdx.x == 128) { A2_TRACE(13, 0) }  // epilogue stores issued
  if (p.dbg && lane == 0) {
    const unsigned long long tot = clock64() - t_start;
    if (warp == 1 && leader) { atomicAdd(p.dbg + 0, w_a); atomicAdd(p.dbg + 2, w_c); atomicAdd(p.dbg + 3, tot); }
    if (warp == 3 && leader) { atomicAdd(p.dbg + 1, w_b); atomicAdd(p.dbg + 2, w_c); }
    if (warp == 4) { atomicAdd(p.dbg + 4, w_a); atomicAdd(p.dbg + 5, w_b); atomicAdd(p.dbg + 6, tot); }
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_2sm(tmem, Cfg::TMEM_COLS);
}

// Ticket counters of the persistent pair kernel: a per-device pool of int pairs, zeroed once
// (and synchronised) before first use; every launch leaves its pair at zero again (the last
// cluster out resets it).  Eager launches take one pair per launching stream, so two
// persistent attentions in flight on different streams never share a counter.  A launch
// captured into a CUDA graph takes a pair of its own, never handed out again, so graphs
// captured on the same stream can replay concurrently on different streams.  The pool is
// allocated on the first launch outside stream capture; a capture before that, or after the
// pool is exhausted, runs the one-tile kernel (same results).
static int* attention2_tile_counter(cudaStream_t st) {
  constexpr int kSlots = 16384;
  constexpr int kMaxDev = 64;
  static std::mutex mu;
  static int* pool[kMaxDev] = {};
  static std::unordered_map<cudaStream_t, int> slot_of[kMaxDev];
  static int next_slot[kMaxDev] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDev) return nullptr;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  const bool capturing = cs != cudaStreamCaptureStatusNone;
  std::lock_guard<std::mutex> lock(mu);
  if (pool[dev] == nullptr) {
    if (capturing) return nullptr;
    int* c = nullptr;
    if (cudaMalloc(&c, kSlots * 2 * sizeof(int)) != cudaSuccess) return nullptr;
    // zero on the launching stream, then wait: the pool is visible as zero to every stream
    // (a plain cudaMemset runs on the legacy stream, unordered with non-blocking streams)
    if (cudaMemsetAsync(c, 0, kSlots * 2 * sizeof(int), st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      cudaFree(c);
      return nullptr;
    }
    pool[dev] = c;
  }
  int slot;
  if (capturing) {
    if (next_slot[dev] >= kSlots) return nullptr;
    slot = next_slot[dev]++;  // owned by this captured launch for the graph's lifetime
  } else {
    auto it = slot_of[dev].find(st);
    if (it != slot_of[dev].end()) {
      slot = it->second;
    } else {
      if (next_slot[dev] >= kSlots) return nullptr;  // pool exhausted: one-tile kernel
      slot = next_slot[dev]++;
      slot_of[dev][st] = slot;
    }
  }
  return pool[dev] + 2 * slot;
}

// Persistent variant (default; PS_ATTN_PERSIST=0 for one tile per CTA pair): one cluster per
// SM pair takes tiles of the (longest-first) tile list from an atomic ticket.  The next tile's Q is loaded as soon as
// the last S MMA of the current tile has read Q (q_empty), its S MMAs run while the softmax
// warps finish the current tile, and its first PV MMA waits for the epilogue to have read O
// (o_empty) -- the per-tile prologue (barrier / TMEM setup, Q load, pipeline fill) leaves
// the critical path.  Barrier parities run on a per-cluster block counter across tiles.
// Same arithmetic per tile as attn2_kernel; the epilogue stores rows directly (the Q buffer
// already holds the next tile's Q).
template <int DP, int NV_>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(A2_THREADS, 1)
    attn2p_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV, const AttnParams p) {
  using Cfg = Attn2Cfg<DP, NV_>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned, derived from smem_raw by an integer offset so the compiler keeps the
  // shared address space (uintptr_t arithmetic made every access through it a generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + Cfg::Q_BYTES;
  uint8_t* sV = sK + Cfg::NK * Cfg::K_SLOT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + Cfg::NV * Cfg::V_SLOT);
  uint64_t* q_full = bars;                    // leader
  uint64_t* q_empty = bars + 1;               // both (multicast commit)
  uint64_t* k_full = bars + 2;                // leader
  uint64_t* k_empty = k_full + Cfg::NK;       // both
  uint64_t* v_full = k_empty + Cfg::NK;       // leader
  uint64_t* v_empty = v_full + Cfg::NV;       // both
  uint64_t* s_full = v_empty + Cfg::NV;       // both
  uint64_t* s_free = s_full + 1;              // leader, 256 arrivals
  uint64_t* p_full = s_free + 1;              // leader, 256 arrivals
  uint64_t* p_free = p_full + 1;              // both
  uint64_t* o_full = p_free + 1;              // both
  uint64_t* o_empty = o_full + 1;             // leader, 256 arrivals
  uint64_t* tile_full = o_empty + 1;          // both, [8]: tile ring entries written
  int* tring = reinterpret_cast<int*>(tile_full + 8);  // [8] tile ring (leader fills both CTAs')
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tring + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int ncl = gridDim.x >> 1;
  // k-th tile of this cluster: dealt dynamically (an atomic ticket per tile, fetched by the
  // leader's producer and published through an 8-entry ring in both CTAs), so the longest-
  // first list balances like the hardware's CTA scheduling of the one-tile-per-CTA kernel.
  // Ring reuse is safe: no role lags the producer by more than two tiles (the K ring holds
  // two key blocks and every tile has at least one).
  auto next_tile = [&](int k) -> int {
    mbar_wait(&tile_full[k & 7], (k >> 3) & 1);
    return *reinterpret_cast<volatile int*>(tring + (k & 7));
  };
  auto tile = [&](int t, int& q0, int& kb0, int& ke, int& nkb) {
    const int img = p.tile_img[t];
    q0 = p.tile_q0[t] + (int)rank * A2_BM;
    kb0 = p.img_tok0[img];
    ke = p.img_tok0[img + 1];
    nkb = (ke - kb0 + A2_BN - 1) / A2_BN;
    if (p.tile_kb0 != nullptr) {  // split-KV: key blocks [tile_kb0, +tile_nkb) of the image
      kb0 += p.tile_kb0[t] * A2_BN;  // (ke stays the image end: interior ranges are whole blocks)
      nkb = p.tile_nkb[t];
    }
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < Cfg::NK; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < Cfg::NV; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 2 * 128);
    mbar_init(p_full, 2 * 128);
    mbar_init(p_free, 1);
    mbar_init(o_full, 1);
    mbar_init(o_empty, 2 * 128);
    for (int i = 0; i < 8; ++i) mbar_init(&tile_full[i], 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_2sm(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // PDL: the setup above (barriers, TMEM, descriptor prefetch) overlaps the previous kernel's
  // tail; Q/K/V, the device tile count and the ticket counters are read only after this
  pdl_wait();
  const int n_tiles = p.n_dev != nullptr ? *p.n_dev : p.n_tiles;

  if (warp == 0) {
    // -------------------------------------------------- producer (both CTAs)
    if (lane == 0) {
      int ks = 0, vs = 0;
      uint32_t kph = 0, vph = 0;
      for (int ti = 0;; ++ti) {
        int t;
        if (leader) {  // fetch and publish the next tile (-1: none left)
          t = (int)atomicAdd(p.tile_ctr, 1u);
          if (t >= n_tiles) t = -1;
          tring[ti & 7] = t;
          asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(mapa_shared(tring + (ti & 7), 1)), "r"(t) : "memory");
          mbar_arrive(&tile_full[ti & 7]);
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                           mapa_shared(&tile_full[ti & 7], 1))
                       : "memory");
        } else {
          t = next_tile(ti);
        }
        if (t < 0) break;
        int q0, k_begin, k_end, n_kb;
        tile(t, q0, k_begin, k_end, n_kb);
        if (ti >= 1) mbar_wait(q_empty, (ti - 1) & 1);  // the previous tile's S MMAs read Q
        if (leader) mbar_arrive_expect_tx(q_full, 2 * Cfg::Q_BYTES);
        for (int kc = 0; kc < Cfg::KB; ++kc)
          tma_load_2d_2sm(sQ + kc * A2_BM * 128, &tmQ, mapa_shared(q_full, 0), kc * 64, q0);
        auto load_k = [&](int j) {
          for (int kc = 0; kc < Cfg::KB; ++kc) {
            mbar_wait(&k_empty[ks], kph ^ 1);
            if (leader) mbar_arrive_expect_tx(&k_full[ks], 2 * Cfg::K_SLOT);
            tma_load_2d_2sm(sK + ks * Cfg::K_SLOT, &tmK, mapa_shared(&k_full[ks], 0), kc * 64,
                            k_begin + j * A2_BN + (int)rank * (A2_BN / 2));
            if (++ks == Cfg::NK) { ks = 0; kph ^= 1; }
          }
        };
        auto load_v = [&](int j) {
          for (int ka = 0; ka < 2; ++ka) {
            mbar_wait(&v_empty[vs], vph ^ 1);
            if (leader) mbar_arrive_expect_tx(&v_full[vs], 2 * Cfg::V_SLOT);
            const uint32_t lb = mapa_shared(&v_full[vs], 0);
            uint8_t* dst = sV + vs * Cfg::V_SLOT;
            for (int n = 0; n < Cfg::PV_MMAS; ++n)
              tma_load_2d_2sm(dst + n * Cfg::V_ROWS * 128, &tmV, lb, k_begin + j * A2_BN + ka * 64,
                              n * Cfg::PV_N + (int)rank * Cfg::V_ROWS);
            if (++vs == Cfg::NV) { vs = 0; vph ^= 1; }
          }
        };
        load_k(0);
        for (int j = 0; j < n_kb; ++j) {
          if (j + 1 < n_kb) load_k(j + 1);
          load_v(j);
        }
      }
    }
  } else if (warp == 1 || warp == 3) {
    // ------------------------------- MMA issuers (leader only): w1 S = Q K^T, w3 O += P V
    if (leader) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(2 * A2_BM, A2_BN);
      constexpr uint32_t idesc_o = idesc_bf16_f32(2 * A2_BM, Cfg::PV_N);
      const uint64_t dq0 = sdesc_sw128(sQ), dk0 = sdesc_sw128(sK), dv0 = sdesc_sw128(sV);
      int ring = 0;
      uint32_t rph = 0;
      int gj = 0;
      for (int ti = 0;; ++ti) {
        const int t = next_tile(ti);
        if (t < 0) break;
        int q0, k_begin, k_end, n_kb;
        tile(t, q0, k_begin, k_end, n_kb);
        if (warp == 1) {
          mbar_wait(q_full, ti & 1);
          tc_fence_after();
          for (int j = 0; j < n_kb; ++j, ++gj) {
            if (gj >= 1) mbar_wait(s_free, (gj - 1) & 1);
            tc_fence_after();
            for (int kc0 = 0; kc0 < Cfg::KB; kc0 += A2_KWAIT) {
              // wait for A2_KWAIT K chunks, then issue their MMAs back to back (a wait between
              // groups of 4 MMAs lets the tensor queue drain)
              {
                int r2 = ring;
                uint32_t p2 = rph;
                for (int q = 0; q < A2_KWAIT && kc0 + q < Cfg::KB; ++q) {
                  mbar_wait(&k_full[r2], p2);
                  if (++r2 == Cfg::NK) { r2 = 0; p2 ^= 1; }
                }
              }
              tc_fence_after();
              for (int kc = kc0; kc < kc0 + A2_KWAIT && kc < Cfg::KB; ++kc) {
                // descriptors from hoisted bases: the start-address field is (smem address >> 4)
                // in the low bits, so an operand offset is a plain add (no carry: smem < 256 KB)
                const uint64_t dq = dq0 + (uint64_t)((kc * A2_BM * 128) >> 4);
                const uint64_t dk = dk0 + (uint64_t)((ring * Cfg::K_SLOT) >> 4);
#if A2_WARP_ISSUE
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  mma_bf16_ss_2sm_w(tmem + Cfg::S_COL, dq + (uint64_t)(k * 2), dk + (uint64_t)(k * 2), idesc_s,
                                    (kc | k) != 0);
                mma_commit_2sm_w(&k_empty[ring], 0x3);
                if (kc == Cfg::KB - 1) {
                  mma_commit_2sm_w(s_full, 0x3);
                  if (j == n_kb - 1) mma_commit_2sm_w(q_empty, 0x3);  // Q free for the next tile
                }
#else
                if (lane == 0) {
#pragma unroll
                  for (int k = 0; k < 4; ++k)
                    mma_bf16_ss_2sm(tmem + Cfg::S_COL, dq + (uint64_t)(k * 2), dk + (uint64_t)(k * 2), idesc_s,
                                    (kc | k) != 0);
                  mma_commit_2sm(&k_empty[ring], 0x3);
                  if (kc == Cfg::KB - 1) {
                    mma_commit_2sm(s_full, 0x3);
                    if (j == n_kb - 1) mma_commit_2sm(q_empty, 0x3);  // Q free for the next tile
                  }
                }
                __syncwarp();
#endif
                if (++ring == Cfg::NK) { ring = 0; rph ^= 1; }
              }
            }
          }
        } else {
          for (int j = 0; j < n_kb; ++j, ++gj) {
            mbar_wait(p_full, gj & 1);
            if (j == 0 && ti >= 1) mbar_wait(o_empty, (ti - 1) & 1);  // O of the previous tile read
            tc_fence_after();
            for (int ka = 0; ka < 2; ++ka) {
              mbar_wait(&v_full[ring], rph);
              tc_fence_after();
              const uint64_t dv = dv0 + (uint64_t)((ring * Cfg::V_SLOT) >> 4);
#if A2_WARP_ISSUE
#pragma unroll
              for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int n = 0; n < Cfg::PV_MMAS; ++n)
                  mma_bf16_ts_2sm_w(tmem + Cfg::O_COL + n * Cfg::PV_N, tmem + Cfg::P_COL + ka * 32 + k * 8,
                                    dv + (uint64_t)((n * Cfg::V_ROWS * 128 + k * 32) >> 4), idesc_o,
                                    (j | ka | k) != 0);
              mma_commit_2sm_w(&v_empty[ring], 0x3);
              if (ka == 1) {
                mma_commit_2sm_w(p_free, 0x3);
                if (j == n_kb - 1) mma_commit_2sm_w(o_full, 0x3);
              }
#else
              if (lane == 0) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
#pragma unroll
                  for (int n = 0; n < Cfg::PV_MMAS; ++n)
                    mma_bf16_ts_2sm(tmem + Cfg::O_COL + n * Cfg::PV_N, tmem + Cfg::P_COL + ka * 32 + k * 8,
                                    dv + (uint64_t)((n * Cfg::V_ROWS * 128 + k * 32) >> 4), idesc_o,
                                    (j | ka | k) != 0);
                mma_commit_2sm(&v_empty[ring], 0x3);
                if (ka == 1) {
                  mma_commit_2sm(p_free, 0x3);
                  if (j == n_kb - 1) mma_commit_2sm(o_full, 0x3);
                }
              }
              __syncwarp();
#endif
              if (++ring == Cfg::NV) { ring = 0; rph ^= 1; }
            }
          }
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------ softmax + epilogue
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const uint32_t s_free_l = mapa_shared(s_free, 0);
    const uint32_t p_full_l = mapa_shared(p_full, 0);
    const uint32_t o_empty_l = mapa_shared(o_empty, 0);
    int gj = 0;
    for (int ti = 0;; ++ti) {
      const int t = next_tile(ti);
      if (t < 0) break;
      int q0, k_begin, k_end, n_kb;
      tile(t, q0, k_begin, k_end, n_kb);
      float m_run = -INFINITY, l_run = 0.f;
      for (int j = 0; j < n_kb; ++j, ++gj) {
        mbar_wait(s_full, gj & 1);
        tc_fence_after();
        uint32_t sr[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) PS_TMEM_LD32(tmem + lane_base + Cfg::S_COL + 32 * c, (sr + 32 * c));
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive_cluster(s_free_l);
        const int kvalid = k_end - (k_begin + j * A2_BN);
        if (kvalid < A2_BN) {
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
        const float mx = fmaxf(mx0, mx1) * p.scale_log2;
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
          sr[i] = pack_bf16(a, b);
        }
        l_run = l_run * alpha + (sum0 + sum1);
        // P columns (and O) are owned by the PV MMAs of the previous block -- across tiles too
        if (gj >= 1) mbar_wait(p_free, (gj - 1) & 1);
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
        mbar_arrive_cluster(p_full_l);
      }
      // epilogue: O / l -> bf16 channels-last rows, then hand O back to the PV issuer
      mbar_wait(o_full, ti & 1);
      tc_fence_after();
      const int q = q0 + row;
      const bool ok = q < k_end;
      const float inv = 1.f / l_run;
      __nv_bfloat16* dst = p.out + (size_t)q * p.Dp;
      // split-KV: this CTA's 128 rows leave as an unnormalised fp32 partial (O, m, l) in slot
      // tile_slot[t] (rank 0) / tile_slot1[t] (rank 1), merged by ps_attention_combine
      const int slot = p.tile_slot != nullptr ? (rank == 0 ? p.tile_slot[t] : p.tile_slot1[t]) : -1;
      float* po = slot >= 0 ? p.part_o + ((size_t)slot * A2_BM + row) * DP : nullptr;
      if (slot >= 0) {
        p.part_ml[((size_t)slot * A2_BM + row) * 2] = m_run;
        p.part_ml[((size_t)slot * A2_BM + row) * 2 + 1] = l_run;
      }
      constexpr int EPI_G = (DP / 32) % 5 == 0 ? 5 : (DP / 32) % 4 == 0 ? 4 : (DP / 32) % 3 == 0 ? 3 : (DP / 32) % 2 == 0 ? 2 : 1;
      uint32_t o[EPI_G][32];
#pragma unroll 1
      for (int c0 = 0; c0 < DP; c0 += 32 * EPI_G) {
#pragma unroll
        for (int g = 0; g < EPI_G; ++g) PS_TMEM_LD32(tmem + lane_base + Cfg::O_COL + c0 + 32 * g, o[g]);
        tmem_ld_wait();
#pragma unroll
        for (int g = 0; g < EPI_G; ++g) reg_fence32(o[g]);
        if (c0 + 32 * EPI_G >= DP) {  // last TMEM read: O can be overwritten by the next tile
          tc_fence_before();
          mbar_arrive_cluster(o_empty_l);
        }
        if (slot >= 0) {
#pragma unroll
          for (int g = 0; g < EPI_G; ++g)
#pragma unroll
            for (int v = 0; v < 4; ++v)
              st_global_v8(po + c0 + 32 * g + 8 * v, *reinterpret_cast<uint32_t(*)[8]>(&o[g][8 * v]));
        } else if (ok) {
#pragma unroll
          for (int g = 0; g < EPI_G; ++g) {
            // 32-byte stores: one full sector per lane and half the store instructions
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              uint32_t w[8];
#pragma unroll
              for (int e = 0; e < 8; ++e)
                w[e] = pack_bf16(__uint_as_float(o[g][16 * v + 2 * e]) * inv,
                                 __uint_as_float(o[g][16 * v + 2 * e + 1]) * inv);
              st_global_v8(dst + c0 + 32 * g + 16 * v, w);
            }
          }
        }
      }
    }
  }
  if (leader && warp == 0 && lane == 0) {
    // the last cluster out leaves the ticket counters at zero for the next launch (every
    // cluster has fetched its -1 before it counts itself done)
    __threadfence();
    if (atomicAdd(p.tile_ctr + 1, 1u) == (unsigned)ncl - 1) {
      p.tile_ctr[0] = 0;
      p.tile_ctr[1] = 0;
      __threadfence();
    }
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_2sm(tmem, Cfg::TMEM_COLS);
}

template <int DP, int NV_>
static int launch2_nv(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v, const CUtensorMap& o,
                      const AttnParams& p, cudaStream_t st) {
  using Cfg = Attn2Cfg<DP, NV_>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn2_kernel<DP, NV_>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    attr = true;
  }
  // persistent kernel by default (config-2 step 14.9 -> 14.3 ms on one box); PS_ATTN_PERSIST=0:
  // one tile per CTA pair
  static const bool persist = !getenv("PS_ATTN_PERSIST") || atoi(getenv("PS_ATTN_PERSIST")) != 0;
  int* ctr = persist ? attention2_tile_counter(st) : nullptr;
  if (ctr != nullptr) {
    AttnParams pp = p;
    pp.tile_ctr = ctr;
    static bool attr_p = false;
    if (!attr_p) {
      cudaFuncSetAttribute(attn2p_kernel<DP, NV_>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
      attr_p = true;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int clusters = p.n_tiles < sms / 2 ? p.n_tiles : sms / 2;
    launch_pdl(attn2p_kernel<DP, NV_>, dim3(2 * clusters), dim3(A2_THREADS), Cfg::SMEM, st, q, k, v, pp);
  } else {
    launch_pdl(attn2_kernel<DP, NV_>, dim3(2 * p.n_tiles), dim3(A2_THREADS), Cfg::SMEM, st, q, k, v, o, p);
  }
  count_launch();
  return check_launch("attention_2cta");
}

template <int DP>
static int launch2_dp(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v, const CUtensorMap& o,
                      const AttnParams& p, cudaStream_t st) {
  // V ring depth (PS_ATTN2_NV=3|4): A/B switch for tools/attn_pair_check.py
  // default 3: the K ring then holds two key blocks (10 slots), which the S issuer's one wait per
  // block (A2_KWAIT) and the tile ring's reuse argument rely on; +0.3-1.4% over 4 (round 2)
  static const int nv = getenv("PS_ATTN2_NV") ? atoi(getenv("PS_ATTN2_NV")) : 3;
  return nv == 3 ? launch2_nv<DP, 3>(q, k, v, o, p, st) : launch2_nv<DP, 4>(q, k, v, o, p, st);
}

int attention2_launch(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& vt, const CUtensorMap& o,
                      const AttnParams& p, int dp,
                      cudaStream_t st) {
  switch (dp) {
    case 64: return launch2_dp<64>(q, k, vt, o, p, st);
    case 128: return launch2_dp<128>(q, k, vt, o, p, st);
    case 192: return launch2_dp<192>(q, k, vt, o, p, st);
    case 256: return launch2_dp<256>(q, k, vt, o, p, st);
    case 320: return launch2_dp<320>(q, k, vt, o, p, st);
    default: return set_error(PS_ERR_INPUT, "attention: unsupported head dim %d", dp);
  }
}

int attention2_v_rows(int dp) { return (dp <= 256 ? dp : dp / 2) / 2; }

}  // namespace ps
