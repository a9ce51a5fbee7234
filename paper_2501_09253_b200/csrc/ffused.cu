// Fused feed-forward + residual on CTA pairs (K6):
//
//   out[NCHW] = W2 gelu(W1 x + b1) + b2 + resid      (kernels.py:124-127, patched.py:215-217)
//
// The 2-GEMM path writes the hidden activations (T x 1280 bf16, 304 MB at config 2)
// to HBM and reads them back.  Here a CTA pair owns 256 tokens and walks the hidden
// dimension in chunks of 128:
//   MMA1(c): H = X W1[c]^T           (M = 256, N = 128, K = Cp; A = X resident in smem)
//   epilogue: H -> +b1 -> bf16 -> GELU -> TMEM (the A operand of MMA2; shared memory with p.ts = 0)
//   MMA2(c): O += H W2[:, c]^T       (M = 256, N = Cp as two MMAs, K = 128)
// O (Cp fp32 columns), the H chunk (128) and its bf16 GELU (64) live in TMEM (<= 512);
// weights stream through one ring of 10 KB slots, each CTA loading its half of every
// MMA's B operand.  MMA1(c + 1) runs while the epilogue turns H(c) into MMA2's operand.
// Arithmetic is the 2-GEMM path's exactly (same MMA accumulation order, same bf16 GELU,
// same residual epilogue), so the output is bit-identical to it.
//
// Warp roles (512 threads): w0 TMA producer, w1 MMA issuer (leader CTA), w2 TMEM
// allocator, w4..w15 epilogue (w4..w11 also the H epilogue).
#include "common.cuh"
#include "ps_internal.h"

#ifndef FF_WARP_ISSUE  // MMA issue by the converged warp (elect.sync in the asm) instead of lane 0
#define FF_WARP_ISSUE 1  // fused FF 207 -> 186 us (p.ts branch hoisted out of the MMA loop; with it inside, 205 -> 210)
#endif
namespace ps {

constexpr int FF_BM = 128;
constexpr int FF_HC = 128;      // hidden units per chunk (2 k-blocks of MMA2)
constexpr int FF_NS = 8;        // weight ring slots
constexpr int FF_SLOT = 10240;  // bytes per slot (max of a W1 piece 8 KB and a W2 piece <= 10 KB)
constexpr int FF_THREADS = 512;
constexpr int FF_ST_LD = 36;    // row pitch (floats) of the output epilogue's transpose tiles

template <int CP>
struct FfCfg {
  static constexpr int KB = CP / 64;
  static constexpr int X_BYTES = KB * FF_BM * 128;
  static constexpr int H_BYTES = 2 * FF_BM * 128;
  static constexpr int NHALF = CP / 2;        // N of one MMA2
  static constexpr int W2_ROWS = NHALF / 2;   // this CTA's B rows of one MMA2
  static constexpr int W1_ROWS = FF_HC / 2;   // this CTA's B rows of one MMA1 (64)
  // per-warp [16][FF_ST_LD] fp32 transpose tiles of the output epilogue: rows padded 32 -> 36
  // floats so the transposed float4 reads (16 lanes on 16 rows of one column range) spread over
  // the banks -- with 32-float rows they were 16-way conflicts (77% of the kernel's shared-load
  // wavefronts, ncu round 2)
  static constexpr int STG = 12 * 16 * FF_ST_LD * 4;
  static constexpr int B1_FLOATS = 1280;  // first-layer biases staged in shared memory (hp <= 1280)
  static constexpr int SMEM = X_BYTES + H_BYTES + FF_NS * FF_SLOT + STG + (B1_FLOATS + CP) * 4 + 1024 + 512;
  // TMEM: O (Cp fp32) | H chunk (128 fp32) | GELU(H) chunk as bf16 pairs (64), MMA2's A (p.ts)
  static constexpr int O_COL = 0, H_COL = CP, HB_COL = CP + FF_HC;
  static_assert(CP % 64 == 0 && NHALF % 16 == 0 && W2_ROWS % 8 == 0 && W2_ROWS * 128 <= FF_SLOT, "Cp");
  static_assert(CP + FF_HC + FF_HC / 2 <= 512, "TMEM");
};

// PROBE: the p.dbg build (role wait counters, epilogue phase clocks) -- a separate instantiation
// so the production kernel carries no probe registers (the H epilogue sits at 128 registers)
template <int CP, bool PROBE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(FF_THREADS, 1)
    ff_pair_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW1,
                   const __grid_constant__ CUtensorMap tmW2, const FfParams p) {
  using Cfg = FfCfg<CP>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned, derived from smem_raw by an integer offset so the compiler keeps the
  // shared address space (uintptr_t arithmetic made every access through it a generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sX = smem;
  uint8_t* sH = sX + Cfg::X_BYTES;
  uint8_t* sW = sH + Cfg::H_BYTES;
  float* sStg = reinterpret_cast<float*>(sW + FF_NS * FF_SLOT);
  float* sB1 = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(sStg) + Cfg::STG);
  float* sB2 = sB1 + Cfg::B1_FLOATS;  // [CP] output biases
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB2 + CP);
  uint64_t* x_full = bars;
  uint64_t* x_empty = bars + 1;
  uint64_t* w_full = bars + 2;
  uint64_t* w_empty = w_full + FF_NS;
  uint64_t* h_full = w_empty + FF_NS;
  uint64_t* h_empty = h_full + 1;
  uint64_t* hs_full = h_empty + 1;
  uint64_t* hs_empty = hs_full + 1;
  uint64_t* o_full = hs_empty + 1;
  uint64_t* o_empty = o_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmX);
    tma_prefetch(&tmW1);
    tma_prefetch(&tmW2);
    mbar_init(x_full, 1);
    mbar_init(x_empty, 1);
    for (int s = 0; s < FF_NS; ++s) {
      mbar_init(&w_full[s], 1);
      mbar_init(&w_empty[s], 1);
    }
    mbar_init(h_full, 1);
    mbar_init(h_empty, 2 * 256);   // H epilogue warpgroups 0-1 of both CTAs
    mbar_init(hs_full, 2 * 256);
    mbar_init(hs_empty, 1);
    mbar_init(o_full, 1);
    mbar_init(o_empty, 2 * 384);   // all epilogue threads of both CTAs
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_2sm(tmem_slot, 512);
  // first-layer biases -> shared memory (the chunk epilogue's per-chunk reads were L2 loads
  // issued next to the H wait); weights are not written by the previous kernel, so this may
  // run before the PDL wait
  const bool b1_smem = p.hp <= Cfg::B1_FLOATS;
  if (b1_smem && warp >= 4)
    for (int i = threadIdx.x - 128; i < p.hp / 4; i += FF_THREADS - 128)
      reinterpret_cast<float4*>(sB1)[i] = __ldg(reinterpret_cast<const float4*>(p.b1) + i);
  if (warp >= 4)
    for (int i = threadIdx.x - 128; i < CP / 4; i += FF_THREADS - 128)
      reinterpret_cast<float4*>(sB2)[i] = __ldg(reinterpret_cast<const float4*>(p.b2) + i);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // PDL: the setup above overlaps the previous kernel's tail
  const int num_m = p.m_map ? (p.m_count_dev ? *p.m_count_dev : p.m_count) : (p.M + FF_BM - 1) / FF_BM;
  const int n_units = (num_m + 1) / 2;
  const int unit0 = blockIdx.x >> 1, unit_step = gridDim.x >> 1;
  // tail split (p.tail_split): the units of the last, partial wave become two work items
  // each, one per half of the output channels (each recomputes H; MMA2 and the epilogue do
  // half the columns) -- a 0.27 wave of full units becomes 0.54 wave of ~0.75-cost items
  const int tail = (p.tail_split && 2 * (n_units % unit_step) <= unit_step) ? n_units % unit_step : 0;
  const int n_full = n_units - tail;
  const int n_items = n_full + 2 * tail;
  auto item = [&](int w, int& u, int& half) {
    if (w < n_full) {
      u = w;
      half = -1;
    } else {
      u = n_full + ((w - n_full) >> 1);
      half = (w - n_full) & 1;
    }
  };
  const int m_oob = (p.M + FF_BM - 1) / FF_BM;
  const int NC = p.hp / FF_HC;
  auto my_m = [&](int u) {
    const int lm = 2 * u + (int)rank;
    return lm >= num_m ? -1 : p.m_map ? __ldg(p.m_map + lm) : lm;
  };

  unsigned long long cnt[4] = {0, 0, 0, 0};
  // PROBE timeline: clock64 stamps of CTA 0's first 40 chunks at dbg[64 + 8 g + k] (k: 0/1 MMA1
  // issue start/end, 2/3 MMA2 issue start/end, 4 H ready seen, 5 H released, 6 GELU done,
  // 7 Hb handed to MMA2)
#define FF_STAMP(gg, k)                                                                 \
  do {                                                                                  \
    if (PROBE && blockIdx.x == 0 && (gg) < 40) p.dbg[64 + 8 * (gg) + (k)] = clock64(); \
  } while (0)
  // epilogue phase clocks (p.dbg, warp 4): [0] H TMEM load, [1] load + GELU, [2] Hb store + arrive,
  // [3] chunks, [4] output drain per tile, [5] tiles
  __shared__ unsigned long long ph[8];
  __shared__ long long t_mma1;  // PROBE: clock when the issuer started the current chunk's MMA1
  if (PROBE && threadIdx.x < 8) ph[threadIdx.x] = 0;
  const long long t_start = PROBE ? clock64() : 0;
  auto tw = [&](uint64_t* bar, uint32_t par, int k) {
    if (PROBE) {
      const long long t0 = clock64();
      mbar_wait(bar, par);
      cnt[k] += clock64() - t0;
    } else {
      mbar_wait(bar, par);
    }
  };

  if (warp == 0) {
    // --------------------------------------------------------------- producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int li = 0;
      auto next = [&]() {
        if (++s == FF_NS) { s = 0; ph ^= 1; }
      };
      for (int w = unit0; w < n_items; w += unit_step, ++li) {
        int u, half;
        item(w, u, half);
        const int mt0 = my_m(u);
        const int mt = mt0 < 0 ? m_oob : mt0;
        tw(x_empty, (li & 1) ^ 1, 1);
        if (leader) mbar_arrive_expect_tx(x_full, 2 * Cfg::X_BYTES);
        for (int kb = 0; kb < Cfg::KB; ++kb)
          tma_load_2d_2sm(sX + kb * FF_BM * 128, &tmX, mapa_shared(x_full, 0), kb * 64, mt * FF_BM);
        auto w1 = [&](int c) {
          for (int kb = 0; kb < Cfg::KB; ++kb) {
            tw(&w_empty[s], ph ^ 1, 0);
            if (leader) mbar_arrive_expect_tx(&w_full[s], 2 * Cfg::W1_ROWS * 128);
            tma_load_2d_2sm(sW + s * FF_SLOT, &tmW1, mapa_shared(&w_full[s], 0), kb * 64,
                            c * FF_HC + (int)rank * Cfg::W1_ROWS);
            next();
          }
        };
        auto w2 = [&](int c) {
          for (int kk = 0; kk < 2; ++kk)
            for (int nn = 0; nn < 2; ++nn) {
              if (half >= 0 && nn != half) continue;
              tw(&w_empty[s], ph ^ 1, 0);
              if (leader) mbar_arrive_expect_tx(&w_full[s], 2 * Cfg::W2_ROWS * 128);
              tma_load_2d_2sm(sW + s * FF_SLOT, &tmW2, mapa_shared(&w_full[s], 0), c * FF_HC + kk * 64,
                              nn * Cfg::NHALF + (int)rank * Cfg::W2_ROWS);
              next();
            }
        };
        // the MMA issuer's consumption order: W1(0), then W1(c+1), W2(c) per chunk
        w1(0);
        for (int c = 0; c < NC; ++c) {
          if (c + 1 < NC) w1(c + 1);
          w2(c);
        }
      }
    }
  } else if (warp == 1 || warp == 3) {
    // ---------------------------------------- MMA issuers (leader CTA): w1 MMA1, w3 MMA2
    // Two issuing threads: one thread issuing all 36 MMAs + 9 commits + 11 waits of a chunk
    // was the bottleneck (issuer busy 70%, tensor pipe 33%).  Weight pieces are consumed at
    // fixed positions of the producer's sequence W1(0), [W1(c+1), W2(c)] per chunk (KB pieces
    // of W1, 4 of W2).
    if (leader) {
      constexpr uint32_t idesc1 = idesc_bf16_f32(2 * FF_BM, FF_HC);
      constexpr uint32_t idesc2 = idesc_bf16_f32(2 * FF_BM, Cfg::NHALF);
      int g = 0;  // global chunk counter
      int li = 0;
      long long base = 0;  // the item's first weight piece in the producer's sequence
      for (int w = unit0; w < n_items; w += unit_step, ++li) {
        int u, half;
        item(w, u, half);
        (void)u;
        const int PC = Cfg::KB + (half < 0 ? 4 : 2);  // weight pieces per chunk: KB of W1, 4 (2) of W2
        auto pos_w1 = [&](int c) { return c == 0 ? 0 : Cfg::KB + PC * (c - 1); };
        auto pos_w2 = [&](int c) { return c < NC - 1 ? 2 * Cfg::KB + PC * c : Cfg::KB + PC * c; };
        if (warp == 1) {
          tw(x_full, li & 1, 3);
          tc_fence_after();
        }
        for (int c = 0; c < NC; ++c, ++g) {
          if (warp == 1) {
            tw(h_empty, (g & 1) ^ 1, 1);  // the epilogue drained H(g - 1)
            if (PROBE && lane == 0) t_mma1 = clock64();
            if (lane == 0) FF_STAMP(g, 0);
            tc_fence_after();
            for (int kb = 0; kb < Cfg::KB; ++kb) {
              const long long gi = base + pos_w1(c) + kb;
              const int s = (int)(gi % FF_NS);
              tw(&w_full[s], (uint32_t)((gi / FF_NS) & 1), 0);
              tc_fence_after();
#if FF_WARP_ISSUE
              {  // the converged warp issues (elect.sync in the asm): uniform-register descriptors
                const uint64_t dx = sdesc_sw128(sX + kb * FF_BM * 128), dw = sdesc_sw128(sW + s * FF_SLOT);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  mma_bf16_ss_2sm_w(tmem + Cfg::H_COL, dx + (uint64_t)(k * 2), dw + (uint64_t)(k * 2), idesc1,
                                    (kb | k) != 0);
                mma_commit_2sm_w(&w_empty[s], 0x3);
                if (kb == Cfg::KB - 1) {
                  mma_commit_2sm_w(h_full, 0x3);
                  if (c == NC - 1) mma_commit_2sm_w(x_empty, 0x3);
                  if (lane == 0) FF_STAMP(g, 1);
                }
              }
#else
              if (lane == 0) {
                const uint8_t* wt = sW + s * FF_SLOT;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  mma_bf16_ss_2sm(tmem + Cfg::H_COL, sdesc_sw128(sX + kb * FF_BM * 128 + k * 32),
                                  sdesc_sw128(wt + k * 32), idesc1, (kb | k) != 0);
                mma_commit_2sm(&w_empty[s], 0x3);
                if (kb == Cfg::KB - 1) {
                  mma_commit_2sm(h_full, 0x3);
                  if (c == NC - 1) mma_commit_2sm(x_empty, 0x3);
                  FF_STAMP(g, 1);
                }
              }
              __syncwarp();
#endif
            }
          } else {
            tw(hs_full, g & 1, 2);  // H(c) written to shared memory
            if (c == 0) tw(o_empty, (li & 1) ^ 1, 3);  // O of the previous tile drained
            if (lane == 0) FF_STAMP(g, 2);
            tc_fence_after();
            int piece = 0;
            for (int kk = 0; kk < 2; ++kk)
              for (int nn = 0; nn < 2; ++nn) {
                if (half >= 0 && nn != half) continue;
                const long long gi = base + pos_w2(c) + piece;
                ++piece;
                const int s = (int)(gi % FF_NS);
                tw(&w_full[s], (uint32_t)((gi / FF_NS) & 1), 0);
                tc_fence_after();
#if FF_WARP_ISSUE
                {
                  const uint64_t dw = sdesc_sw128(sW + s * FF_SLOT);
                  const uint32_t dcol = tmem + Cfg::O_COL + nn * Cfg::NHALF;
                  if (p.ts) {  // one branch per piece: no runtime condition between the MMAs
                    const uint32_t acol = tmem + Cfg::HB_COL + kk * 32;
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                      mma_bf16_ts_2sm_w(dcol, acol + k * 8, dw + (uint64_t)(k * 2), idesc2, (c | kk | k) != 0);
                  } else {
                    const uint64_t dh = sdesc_sw128(sH + kk * FF_BM * 128);
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                      mma_bf16_ss_2sm_w(dcol, dh + (uint64_t)(k * 2), dw + (uint64_t)(k * 2), idesc2,
                                        (c | kk | k) != 0);
                  }
                  mma_commit_2sm_w(&w_empty[s], 0x3);
                  if (kk == 1 && (half >= 0 || nn == 1)) {  // the chunk's last W2 piece
                    mma_commit_2sm_w(hs_empty, 0x3);
                    if (c == NC - 1) mma_commit_2sm_w(o_full, 0x3);
                    if (lane == 0) FF_STAMP(g, 3);
                  }
                }
#else
                if (lane == 0) {
                  const uint8_t* wt = sW + s * FF_SLOT;
#pragma unroll
                  for (int k = 0; k < 4; ++k) {
                    if (p.ts)
                      mma_bf16_ts_2sm(tmem + Cfg::O_COL + nn * Cfg::NHALF, tmem + Cfg::HB_COL + kk * 32 + k * 8,
                                      sdesc_sw128(wt + k * 32), idesc2, (c | kk | k) != 0);
                    else
                      mma_bf16_ss_2sm(tmem + Cfg::O_COL + nn * Cfg::NHALF,
                                      sdesc_sw128(sH + kk * FF_BM * 128 + k * 32), sdesc_sw128(wt + k * 32), idesc2,
                                      (c | kk | k) != 0);
                  }
                  mma_commit_2sm(&w_empty[s], 0x3);
                  if (kk == 1 && (half >= 0 || nn == 1)) {  // the chunk's last W2 piece
                    mma_commit_2sm(hs_empty, 0x3);
                    if (c == NC - 1) mma_commit_2sm(o_full, 0x3);
                    FF_STAMP(g, 3);
                  }
                }
                __syncwarp();
#endif
              }
          }
        }
        base += (long long)PC * NC;
      }
    }
  } else if (warp >= 4) {
    // --------------------------------------------------------------- epilogue
    const int wq = warp & 3;
    const int wg = (warp - 4) >> 2;
    const int row = wq * 32 + lane;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    const uint32_t h_empty_l = mapa_shared(h_empty, 0);
    const uint32_t hs_full_l = mapa_shared(hs_full, 0);
    const uint32_t o_empty_l = mapa_shared(o_empty, 0);
    float* st = sStg + (warp - 4) * 16 * FF_ST_LD;  // [16][FF_ST_LD] fp32 transpose tile of this warp
    const int ci = lane >> 1, seg = lane & 1;      // transposed role: column, 16-token half
    int g = 0, li = 0;
    for (int w = unit0; w < n_items; w += unit_step, ++li) {
      int u, half;
      item(w, u, half);
      const int mt = my_m(u);
      const int c_lo = half < 0 ? 0 : half * Cfg::NHALF, c_hi = half < 0 ? CP : c_lo + Cfg::NHALF;
      // the idle third warpgroup pulls this tile's residual rows (one 256-byte NCHW segment per
      // channel) into L2 while the chunks run, so the output drain's residual loads hit L2
      if (wg == 2 && p.resid != nullptr && mt >= 0 && (mt + 1) * FF_BM <= p.M && p.hw % FF_BM == 0) {
        const int pidx0 = mt * FF_BM / p.hw, pix0 = mt * FF_BM - pidx0 * p.hw;
        for (int ch = c_lo + (threadIdx.x - 384); ch < min(c_hi, p.c_real); ch += 128)
          l2_prefetch(p.resid + ((size_t)pidx0 * p.c_real + ch) * p.hw + pix0, FF_BM * 2);
      }
      // ---- hidden chunks: H -> +b1 -> bf16 -> GELU -> MMA2's A operand (warpgroups 0, 1)
      for (int c = 0; c < NC; ++c, ++g) {
        if (wg >= 2) continue;
        // the chunk's biases (64 per thread, warp-uniform addresses) load while MMA1 runs
        float4 bq[16];
        if (b1_smem) {
          const float4* b1 = reinterpret_cast<const float4*>(sB1 + c * FF_HC + wg * 64);
#pragma unroll
          for (int i = 0; i < 16; ++i) bq[i] = b1[i];
        } else {
          const float4* b1 = reinterpret_cast<const float4*>(p.b1 + c * FF_HC + wg * 64);
#pragma unroll
          for (int i = 0; i < 16; ++i) bq[i] = __ldg(b1 + i);
        }
        tw(h_full, g & 1, 0);
        const bool probe = PROBE && warp == 4 && lane == 0;
        const long long ph0 = probe ? clock64() : 0;
        if (probe) FF_STAMP(g, 4);
        if (probe) { ph[6] += ph0 - *(volatile long long*)&t_mma1; ph[7] += 1; }  // MMA1 issue -> H ready
        tc_fence_after();
        uint32_t r0[32], r1[32];
        PS_TMEM_LD32(tmem + lane_base + Cfg::H_COL + wg * 64, r0);
        PS_TMEM_LD32(tmem + lane_base + Cfg::H_COL + wg * 64 + 32, r1);
        tmem_ld_wait();
        if (probe) ph[0] += clock64() - ph0;
        reg_fence32(r0);
        reg_fence32(r1);
        tc_fence_before();
        mbar_arrive_cluster(h_empty_l);
        if (probe) FF_STAMP(g, 5);
        uint32_t pk[32];
        if (PROBE && p.dbg[31]) {  // timing experiment: the chunk epilogue without the GELU
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            pk[2 * i] = pack_bf16(__uint_as_float(r0[4 * i]) + bq[i].x, __uint_as_float(r0[4 * i + 1]) + bq[i].y);
            pk[2 * i + 1] = pack_bf16(__uint_as_float(r0[4 * i + 2]) + bq[i].z, __uint_as_float(r0[4 * i + 3]) + bq[i].w);
            pk[16 + 2 * i] = pack_bf16(__uint_as_float(r1[4 * i]) + bq[8 + i].x, __uint_as_float(r1[4 * i + 1]) + bq[8 + i].y);
            pk[16 + 2 * i + 1] =
                pack_bf16(__uint_as_float(r1[4 * i + 2]) + bq[8 + i].z, __uint_as_float(r1[4 * i + 3]) + bq[8 + i].w);
          }
        } else
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          pk[2 * i] = gelu_bf16x2(pack_bf16(__uint_as_float(r0[4 * i]) + bq[i].x,
                                            __uint_as_float(r0[4 * i + 1]) + bq[i].y));
          pk[2 * i + 1] = gelu_bf16x2(pack_bf16(__uint_as_float(r0[4 * i + 2]) + bq[i].z,
                                                __uint_as_float(r0[4 * i + 3]) + bq[i].w));
          pk[16 + 2 * i] = gelu_bf16x2(pack_bf16(__uint_as_float(r1[4 * i]) + bq[8 + i].x,
                                                 __uint_as_float(r1[4 * i + 1]) + bq[8 + i].y));
          pk[16 + 2 * i + 1] = gelu_bf16x2(pack_bf16(__uint_as_float(r1[4 * i + 2]) + bq[8 + i].z,
                                                     __uint_as_float(r1[4 * i + 3]) + bq[8 + i].w));
        }
        if (probe) ph[1] += clock64() - ph0;  // load + release + GELU
        if (probe) FF_STAMP(g, 6);
        tw(hs_empty, (g & 1) ^ 1, 1);  // MMA2 of the previous chunk has read the buffer
        if (p.ts) {  // A operand in TMEM: 32 columns of bf16 pairs per warpgroup, no smem traffic
          const long long ph2 = probe ? clock64() : 0;
          PS_TMEM_ST16(tmem + lane_base + Cfg::HB_COL + wg * 32, pk);
          PS_TMEM_ST16(tmem + lane_base + Cfg::HB_COL + wg * 32 + 16, (pk + 16));
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive_cluster(hs_full_l);
          if (probe) { ph[2] += clock64() - ph2; ph[3] += 1; FF_STAMP(g, 7); }
          continue;
        }
        uint8_t* hrow = sH + wg * FF_BM * 128 + row * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<uint4*>(hrow + ((j ^ (row & 7)) << 4)) =
              make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        fence_proxy_async();
        mbar_arrive_cluster(hs_full_l);
      }
      // ---- output: O + b2 + residual -> NCHW (32-column chunks dealt to the 3 warpgroups)
      tw(o_full, li & 1, 2);
      const long long po = (PROBE && warp == 4 && lane == 0) ? clock64() : 0;
      tc_fence_after();
      const bool ok = mt >= 0 && (mt + 1) * FF_BM <= p.M;
      const int tok_v = (mt < 0 ? 0 : mt) * FF_BM + wq * 32 + seg * 16;
      const int pidx_v = tok_v / p.hw, pix_v = tok_v - pidx_v * p.hw;
      bool released = false;
      for (int cc = c_lo + wg * 32; cc < c_hi; cc += 96) {
        // residual (2 pieces x 32 B per lane) in flight before the accumulator load
        uint4 rsd[4];
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2) {
          const int nv = cc + s2 * 16 + ci;
          rsd[2 * s2] = rsd[2 * s2 + 1] = make_uint4(0, 0, 0, 0);
          if (ok && nv < p.c_real && p.resid != nullptr) {
            const size_t off = ((size_t)pidx_v * p.c_real + nv) * p.hw + pix_v;
            rsd[2 * s2] = __ldg(reinterpret_cast<const uint4*>(p.resid + off));
            rsd[2 * s2 + 1] = __ldg(reinterpret_cast<const uint4*>(p.resid + off) + 1);
          }
        }
        uint32_t r[32];
        PS_TMEM_LD32(tmem + lane_base + Cfg::O_COL + cc, r);
        tmem_ld_wait();
        reg_fence32(r);
        if (cc + 96 >= c_hi) {
          tc_fence_before();
          mbar_arrive_cluster(o_empty_l);
          released = true;
        }
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) + 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 b4 = reinterpret_cast<const float4*>(sB2 + cc)[q];
          v[4 * q] += b4.x; v[4 * q + 1] += b4.y; v[4 * q + 2] += b4.z; v[4 * q + 3] += b4.w;
        }
#pragma unroll
        for (int s16 = 0; s16 < 32; s16 += 16) {
          const int nv = cc + s16 + ci;
#pragma unroll
          for (int i = 0; i < 16; ++i) st[i * FF_ST_LD + lane] = v[s16 + i];
          __syncwarp();
          if (ok && nv < p.c_real) {
            const size_t off = ((size_t)pidx_v * p.c_real + nv) * p.hw + pix_v;
            const uint4 rs0 = rsd[s16 / 8], rs1 = rsd[s16 / 8 + 1];
            const float4* src = reinterpret_cast<const float4*>(st + ci * FF_ST_LD + seg * 16);
            float o[16];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 f = src[q];
              o[4 * q] = f.x; o[4 * q + 1] = f.y; o[4 * q + 2] = f.z; o[4 * q + 3] = f.w;
            }
            const __nv_bfloat162* h0 = reinterpret_cast<const __nv_bfloat162*>(&rs0);
            const __nv_bfloat162* h1 = reinterpret_cast<const __nv_bfloat162*>(&rs1);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              o[2 * q] += __low2float(h0[q]);
              o[2 * q + 1] += __high2float(h0[q]);
              o[8 + 2 * q] += __low2float(h1[q]);
              o[8 + 2 * q + 1] += __high2float(h1[q]);
            }
            uint4 w0, w1;
            w0.x = pack_bf16(o[0], o[1]); w0.y = pack_bf16(o[2], o[3]);
            w0.z = pack_bf16(o[4], o[5]); w0.w = pack_bf16(o[6], o[7]);
            w1.x = pack_bf16(o[8], o[9]); w1.y = pack_bf16(o[10], o[11]);
            w1.z = pack_bf16(o[12], o[13]); w1.w = pack_bf16(o[14], o[15]);
            const uint32_t w8[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
            st_global_v8(p.out + off, w8);  // 32-byte aligned: pix_v is a multiple of 16
          }
          __syncwarp();
        }
      }
      if (!released) {  // a warpgroup without output columns (Cp < 96)
        tc_fence_before();
        mbar_arrive_cluster(o_empty_l);
      }
      if (PROBE && warp == 4 && lane == 0) { ph[4] += clock64() - po; ph[5] += 1; }
    }
  }
  if (PROBE && lane == 0 && leader) {
    const unsigned long long tot = clock64() - t_start;
    // [0-3] producer: w_empty, x_empty | [4-8] mma: w_full, h_empty, hs_full, o_empty, total
    // [9-12] epilogue (warp 4): h_full, hs_empty, o_full, total | [13] producer total
    if (warp == 0) { atomicAdd(p.dbg + 0, cnt[0]); atomicAdd(p.dbg + 1, cnt[1]); atomicAdd(p.dbg + 13, tot); }
    if (warp == 1 || warp == 3) {
      for (int k = 0; k < 4; ++k) atomicAdd(p.dbg + 4 + k, cnt[k]);
      if (warp == 1) atomicAdd(p.dbg + 8, tot);
    }
    if (warp == 4) {
      for (int k = 0; k < 3; ++k) atomicAdd(p.dbg + 9 + k, cnt[k]);
      atomicAdd(p.dbg + 12, tot);
      for (int k = 0; k < 8; ++k) atomicAdd(p.dbg + 16 + k, ph[k]);
    }
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_2sm(tmem, 512);
}

template <int CP>
static int launch_ff(const CUtensorMap& x, const CUtensorMap& w1, const CUtensorMap& w2, const FfParams& p,
                     int sms, cudaStream_t st) {
  using Cfg = FfCfg<CP>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(ff_pair_kernel<CP, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    cudaFuncSetAttribute(ff_pair_kernel<CP, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    attr = true;
  }
  const int num_m = p.m_map ? p.m_count : (p.M + FF_BM - 1) / FF_BM;
  const int units = (num_m + 1) / 2;
  if (units == 0) return PS_OK;
  const int grid = 2 * (units < sms / 2 ? units : sms / 2);
  if (p.dbg)
    launch_pdl(ff_pair_kernel<CP, true>, dim3(grid), dim3(FF_THREADS), Cfg::SMEM, st, x, w1, w2, p);
  else
    launch_pdl(ff_pair_kernel<CP, false>, dim3(grid), dim3(FF_THREADS), Cfg::SMEM, st, x, w1, w2, p);
  count_launch();
  return check_launch("ff_pair");
}

int ff_launch(const CUtensorMap& x, const CUtensorMap& w1, const CUtensorMap& w2, const FfParams& p, int cp,
              int sms, cudaStream_t st) {
  switch (cp) {
    case 128: return launch_ff<128>(x, w1, w2, p, sms, st);
    case 192: return launch_ff<192>(x, w1, w2, p, sms, st);
    case 256: return launch_ff<256>(x, w1, w2, p, sms, st);
    case 320: return launch_ff<320>(x, w1, w2, p, sms, st);
    default: return set_error(PS_ERR_INPUT, "fused feed-forward: channels %d unsupported", cp);
  }
}

}  // namespace ps
