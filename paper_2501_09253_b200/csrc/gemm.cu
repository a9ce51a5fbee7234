// tcgen05 / TMEM / TMA GEMM for the patch path's dense contractions (K5, K6, K7 projections).
//
//   D[M x N] = A[M x K] * B[N x K]^T  (bf16 in, fp32 accumulate in TMEM)
//
// A rows are patch tokens in channels-last order (patch-major, row-major inside a
// patch).  Two A loaders:
//   * plain 2-D rows (linear / feed-forward / attention projections,
//     reference kernels.py:99-127, 257-267);
//   * conv3 implicit GEMM over halo frames (P, ps+2, ps+2, Cp): K-block kb is tap
//     (kb / (Cp/64)) and channel chunk (kb % (Cp/64)); one 4-D TMA box per tap
//     lands exactly the 128-token A tile (reference patched.py:92-113 ->
//     kernels.py:148-161; the frames reproduce zero padding at image borders).
// B is the weight matrix, K-major, bf16.
//
// Persistent: one CTA per SM walks tiles t = blockIdx.x + i*gridDim.x in
// n-fastest order (CTAs running together share A tiles in L2).  The TMEM
// accumulator is double-buffered (2 x BN columns), so the epilogue of tile i
// overlaps the MMAs of tile i+1.
// PAIR = true runs the same tile walk on CTA pairs (cluster of 2 on one TPC,
// tcgen05 cta_group::2): a pair owns 256 x BN outputs, each CTA loads its own
// 128 A rows and HALF of the B rows of every MMA, the leader CTA issues M = 256
// MMAs whose accumulator rows land in each CTA's own TMEM, and MMA completions
// are multicast to both CTAs.  Per SM this halves the B bytes TMA writes into
// shared memory and the tensor core reads from it -- the limit of the 1-CTA
// kernel (shared-memory bandwidth: ~200 B/clk of operand traffic for 128 B/clk).
// Warp roles (384 threads): w0 TMA producer, w1 MMA issuer (one lane), w2 TMEM
// allocator, w4..w11 epilogue (warp w reads TMEM lanes 32*(w%4)..+31, and half
// of the tile's columns).
// Epilogues: bias (+GELU) -> channels-last bf16; bias + residual -> NCHW bf16
// (the block output / residual stream, reference patched.py:215-217); split
// store with the trailing columns written transposed (V^T for attention).
#include "common.cuh"
#include "ps_internal.h"

#ifndef GEMM_WARP_ISSUE  // MMA issue by the converged warp (elect.sync in the asm) instead of lane 0
#define GEMM_WARP_ISSUE 1  // conv3 193 -> 180 us (per-MMA tail-split test hoisted; with it inside, 192 -> 211)
#endif
namespace ps {

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
#ifndef PS_GEMM_LAZY_BIAS
#define PS_GEMM_LAZY_BIAS (PS_GEMM_NWG > 2)
#endif
#ifndef PS_GEMM_NWG
#define PS_GEMM_NWG 3
#endif
constexpr int GEMM_NWG = PS_GEMM_NWG;  // epilogue warpgroups
constexpr int GEMM_THREADS = 128 + 128 * GEMM_NWG;
constexpr int GEMM_EPI_THREADS = 128 * GEMM_NWG;

// BN <= 256: double-buffered accumulators (2*BN TMEM columns), one MMA per k-step.
// BN == 320: single accumulator (long-K GEMMs: conv3, FF2), two N=160 MMAs per k-step,
// so A is read once per 128-token tile.
template <int BN, bool PAIR = false>
struct GemmCfg {
  static constexpr int NBUF = BN <= 256 ? 2 : 1;
  static constexpr int MMA_N = BN <= 256 ? BN : BN / 2;
  static constexpr int N_MMA = BN / MMA_N;
  static constexpr int B_ROWS = PAIR ? MMA_N / 2 : MMA_N;  // B rows of one MMA held by this CTA
  static constexpr int A_BYTES = GEMM_BM * 128;
  static constexpr int B_BYTES = N_MMA * B_ROWS * 128;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // BN = 320 (conv3): one epilogue staging buffer per warp instead of two, which pays for a
  // fifth 36 KB operand stage (the MMA warp waited on TMA data 35% of the time with four)
  // (BN = 160, the O-projection: 4 -> 5 stages, 39 -> 36 us single-CTA; the channels-last TMA-store
  // epilogues -- QKV BN = 192 -- keep two boxes: one measured 90 -> 91.5 us)
  static constexpr int TMA_BUFS = (BN == 320 || BN == 160) ? 1 : 2;
  static constexpr int STAGE_EPI_ = GEMM_NWG > 2 ? 0 : GEMM_NWG * 16 * GEMM_BM * 4;
  static constexpr int STAGE_TMA_ = GEMM_NWG * TMA_BUFS * GEMM_BM * 64;
  static constexpr int STAGE_BUDGET = TMA_BUFS == 1 ? 227 * 1024 - STAGE_TMA_ - STAGE_EPI_ - 1280 : 176 * 1024;
  static constexpr int STAGES = STAGE_BUDGET / STAGE_BYTES > 8 ? 8 : STAGE_BUDGET / STAGE_BYTES;
  static constexpr int TMEM_COLS = NBUF * BN <= 128 ? 128 : NBUF * BN <= 256 ? 256 : 512;
  static constexpr int HALF = BN / 2;  // columns per epilogue warp
  static constexpr int STAGE_EPI = GEMM_NWG > 2 ? 0 : GEMM_NWG * 16 * GEMM_BM * 4;  // transposed-store staging
  static constexpr int STAGE_TMA = STAGE_TMA_;  // per warpgroup: TMA_BUFS 128x32 bf16 store boxes
  static constexpr int SMEM = STAGES * STAGE_BYTES + STAGE_EPI + STAGE_TMA + 1024 /*align*/ + 256 /*barriers*/;
  static_assert(MMA_N % 16 == 0 && MMA_N >= 64 && MMA_N <= 256, "invalid UMMA N");
  static_assert(SMEM <= 227 * 1024, "shared memory budget");
  static_assert(B_ROWS % 8 == 0, "B half rows must be whole 128B-swizzle atoms");
  static_assert(BN % 32 == 0 && (BN / 2) % 32 == 0 || BN <= 256, "epilogue chunking");
};

__device__ __forceinline__ void store16_cl(__nv_bfloat16* dst, const float* v) {
  uint4 w0, w1;
  w0.x = pack_bf16(v[0], v[1]);
  w0.y = pack_bf16(v[2], v[3]);
  w0.z = pack_bf16(v[4], v[5]);
  w0.w = pack_bf16(v[6], v[7]);
  w1.x = pack_bf16(v[8], v[9]);
  w1.y = pack_bf16(v[10], v[11]);
  w1.z = pack_bf16(v[12], v[13]);
  w1.w = pack_bf16(v[14], v[15]);
  if ((reinterpret_cast<uintptr_t>(dst) & 31) == 0) {  // one 32-byte store (STG.256)
    const uint32_t w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    st_global_v8(dst, w);
  } else {
    reinterpret_cast<uint4*>(dst)[0] = w0;
    reinterpret_cast<uint4*>(dst)[1] = w1;
  }
}

template <int BN, bool PAIR>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, const GemmParams p) {
  using Cfg = GemmCfg<BN, PAIR>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned, derived from smem_raw by an integer offset so the compiler keeps the
  // shared address space (uintptr_t arithmetic made every access through it a generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* epi_stage = reinterpret_cast<float*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint8_t* tma_stage = smem + Cfg::STAGES * Cfg::STAGE_BYTES + Cfg::STAGE_EPI;
  uint64_t* full = reinterpret_cast<uint64_t*>(tma_stage + Cfg::STAGE_TMA);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* acc_full = empty + Cfg::STAGES;  // [2]
  uint64_t* acc_empty = acc_full + 2;        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (p.store_tma) tma_prefetch(&tmC);
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      const bool split = GEMM_NWG > 2 || Cfg::NBUF == 1 || (p.epi_split && (BN / 2) % 32 == 0);
      mbar_init(&acc_empty[b], (PAIR ? 2 : 1) * (split ? GEMM_EPI_THREADS : GEMM_EPI_THREADS / 2));
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    if (PAIR) tmem_alloc_2sm(tmem_slot, Cfg::TMEM_COLS);
    else tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  }
  tc_fence_before();
  if (PAIR) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // PDL: barrier init, TMEM allocation and descriptor prefetch above overlap the previous
  // kernel's tail; everything below may read what it wrote
  pdl_wait();

  const int num_n = (p.N + BN - 1) / BN;
  const int num_m = p.m_map ? (p.m_count_dev ? *p.m_count_dev : p.m_count) : (p.M + GEMM_BM - 1) / GEMM_BM;
  // PAIR: a work item is (pair of m tiles, n tile); CTA `rank` takes m tile 2*mp + rank
  const uint32_t rank = PAIR ? cluster_rank() : 0;
  const bool leader = rank == 0;
  const int unit0 = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int unit_step = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int num_mu = PAIR ? (num_m + 1) / 2 : num_m;
  const int n_tiles = num_mu * num_n;
  // work items: tiles, except that with p.tail_split (BN = 320, one n tile) the tiles of the
  // last partial wave become two items each, one per N = 160 column half -- a 0.27 wave of
  // full tiles (conv3: 464 pair tiles on 74 pairs) becomes ~0.54 wave of ~0.6-cost items
  const int tail = (GEMM_NWG > 2 && Cfg::N_MMA == 2 && num_n == 1 && p.tail_split &&
                    2 * (n_tiles % unit_step) <= unit_step)
                       ? n_tiles % unit_step : 0;
  const int n_full = n_tiles - tail;
  const int n_items = n_full + 2 * tail;
  auto item = [&](int w, int& half) {  // item -> tile index; half = -1 (whole tile) or 0 / 1
    if (w < n_full) {
      half = -1;
      return w;
    }
    half = (w - n_full) & 1;
    return n_full + ((w - n_full) >> 1);
  };
  const int m_oob = (p.M + GEMM_BM - 1) / GEMM_BM;  // a physical tile past the end: TMA zero-fills it
  // logical -> physical 128-row tile (active-patch compaction); -1 = no tile (odd pair tail)
  auto phys_m = [&](int lm) { return lm >= num_m ? -1 : p.m_map ? __ldg(p.m_map + lm) : lm; };
  auto my_m = [&](int t) { return phys_m(PAIR ? 2 * (t / num_n) + (int)rank : t / num_n); };
  const int num_kb = p.K / GEMM_BK;


  // profiling: cycles each role spends blocked on its barriers (p.dbg != null)
  unsigned long long t_wait = 0, t_wait2 = 0;
  const long long t_start = clock64();
  auto timed_wait = [&](uint64_t* bar, uint32_t par, unsigned long long& acc) {
    if (p.dbg) {
      const long long t0 = clock64();
      mbar_wait(bar, par);
      acc += clock64() - t0;
    } else {
      mbar_wait(bar, par);
    }
  };
  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const int kcb = p.conv_cp / GEMM_BK;
      for (int w = unit0; w < n_items; w += unit_step) {
        int half;
        const int t = item(w, half);
        const int mt = my_m(t);
        const int m_tile = mt < 0 ? m_oob : mt, n0 = (t % num_n) * BN;
        int p0 = 0, y0 = 0;
        if (p.a_mode == A_CONV3) {
          p0 = (m_tile / p.conv_tpp) * p.conv_np;
          y0 = (m_tile % p.conv_tpp) * p.conv_rows;
        }
        // warm L2 with this tile's residual rows (NCHW, 128 contiguous pixels per channel)
        const bool pf = !p.no_prefetch && mt >= 0 && p.epi == EPI_RESID_NCHW && p.resid != nullptr && p.hw >= GEMM_BM && n0 < p.c_real;
        const int tok0 = m_tile * GEMM_BM;
        const int cpk = (p.c_real + num_kb - 1) / num_kb;
        for (int kb = 0; kb < num_kb; ++kb) {
          if (pf && tok0 + GEMM_BM <= p.M) {
            const int pidx = tok0 / p.hw, pix0 = tok0 - pidx * p.hw;
            for (int n = kb * cpk; n < min(p.c_real, (kb + 1) * cpk); ++n)
              l2_prefetch(p.resid + ((size_t)pidx * p.c_real + n) * p.hw + pix0, GEMM_BM * 2);
          }
          timed_wait(&empty[stage], phase ^ 1, t_wait);
          uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          if (PAIR) {
            // both CTAs' bytes complete on the leader's barrier
            const uint32_t fb = mapa_shared(&full[stage], 0);
            if (leader)
              mbar_arrive_expect_tx(&full[stage], 2 * (half < 0 ? Cfg::STAGE_BYTES : Cfg::A_BYTES + Cfg::B_ROWS * 128));
            if (p.a_mode == A_CONV3) {
              const int tap = kb / kcb, cb = kb % kcb;
              tma_load_4d_2sm(sa, &tmA, fb, cb * GEMM_BK, tap % 3, y0 + tap / 3, p0);
            } else if (p.a_mode == A_TILED) {
              tma_load_2d_2sm(sa, &tmA, fb, 0, (m_tile * num_kb + kb) * GEMM_BM);
            } else {
              tma_load_2d_2sm(sa, &tmA, fb, kb * GEMM_BK, m_tile * GEMM_BM);
            }
#pragma unroll
            for (int j = 0; j < Cfg::N_MMA; ++j)
              if (half < 0 || j == half)
                tma_load_2d_2sm(sb + j * Cfg::B_ROWS * 128, &tmB, fb, kb * GEMM_BK,
                                n0 + j * Cfg::MMA_N + (int)rank * Cfg::B_ROWS);
          } else {
            mbar_arrive_expect_tx(&full[stage], half < 0 ? Cfg::STAGE_BYTES : Cfg::A_BYTES + Cfg::MMA_N * 128);
            if (p.a_mode == A_CONV3) {
              const int tap = kb / kcb, cb = kb % kcb;
              tma_load_4d(sa, &tmA, &full[stage], cb * GEMM_BK, tap % 3, y0 + tap / 3, p0);
            } else if (p.a_mode == A_TILED) {
              // tile-major A: the (m_tile, kb) box is one contiguous 16 KB block
              tma_load_2d(sa, &tmA, &full[stage], 0, (m_tile * num_kb + kb) * GEMM_BM);
            } else {
              tma_load_2d(sa, &tmA, &full[stage], kb * GEMM_BK, m_tile * GEMM_BM);
            }
#pragma unroll
            for (int j = 0; j < Cfg::N_MMA; ++j)
              if (half < 0 || j == half)
                tma_load_2d(sb + j * Cfg::MMA_N * 128, &tmB, &full[stage], kb * GEMM_BK, n0 + j * Cfg::MMA_N);
          }
          if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1 && leader) {
    // -------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = idesc_bf16_f32(PAIR ? 2 * GEMM_BM : GEMM_BM, Cfg::MMA_N);
    int stage = 0;
    uint32_t phase = 0;
    int li = 0;
    for (int w = unit0; w < n_items; w += unit_step, ++li) {
      int half;
      (void)item(w, half);
      const int buf = li % Cfg::NBUF;
      const int use = li / Cfg::NBUF;
      timed_wait(&acc_empty[buf], (use & 1) ^ 1, t_wait2);
      tc_fence_after();
      const uint32_t d = tmem + buf * BN;
      for (int kb = 0; kb < num_kb; ++kb) {
        timed_wait(&full[stage], phase, t_wait);
        tc_fence_after();
#if GEMM_WARP_ISSUE
        {  // the converged warp issues (elect.sync in the asm): uniform-register descriptors
          const uint64_t da = sdesc_sw128(smem + stage * Cfg::STAGE_BYTES);
          const uint64_t db = da + (uint64_t)(Cfg::A_BYTES >> 4);
          auto issue = [&](int k, int j) {
            if (PAIR)
              mma_bf16_ss_2sm_w(d + j * Cfg::MMA_N, da + (uint64_t)(k * 2),
                                db + (uint64_t)((j * Cfg::B_ROWS * 128 + k * 32) >> 4), idesc, (kb | k) != 0);
            else
              mma_bf16_ss_w(d + j * Cfg::MMA_N, da + (uint64_t)(k * 2),
                            db + (uint64_t)((j * Cfg::MMA_N * 128 + k * 32) >> 4), idesc, (kb | k) != 0);
          };
          if (half < 0) {  // the common case: no per-MMA condition
#pragma unroll
            for (int k = 0; k < GEMM_BK / 16; ++k)
#pragma unroll
              for (int j = 0; j < Cfg::N_MMA; ++j) issue(k, j);
          } else {
#pragma unroll
            for (int k = 0; k < GEMM_BK / 16; ++k) issue(k, half);
          }
          if (PAIR) {
            mma_commit_2sm_w(&empty[stage], 0x3);
            if (kb == num_kb - 1) mma_commit_2sm_w(&acc_full[buf], 0x3);
          } else {
            mma_commit_w(&empty[stage]);
            if (kb == num_kb - 1) mma_commit_w(&acc_full[buf]);
          }
        }
#else
        if (lane == 0) {
          // descriptor = stage base + (byte offset >> 4): the start-address field is the low bits
          const uint64_t da = sdesc_sw128(smem + stage * Cfg::STAGE_BYTES);
          const uint64_t db = da + (uint64_t)(Cfg::A_BYTES >> 4);
          auto issue = [&](int k, int j) {
            if (PAIR)
              mma_bf16_ss_2sm(d + j * Cfg::MMA_N, da + (uint64_t)(k * 2),
                              db + (uint64_t)((j * Cfg::B_ROWS * 128 + k * 32) >> 4), idesc, (kb | k) != 0);
            else
              mma_bf16_ss(d + j * Cfg::MMA_N, da + (uint64_t)(k * 2),
                          db + (uint64_t)((j * Cfg::MMA_N * 128 + k * 32) >> 4), idesc, (kb | k) != 0);
          };
          if (half < 0) {  // the common case: no per-MMA condition
#pragma unroll
            for (int k = 0; k < GEMM_BK / 16; ++k)
#pragma unroll
              for (int j = 0; j < Cfg::N_MMA; ++j) issue(k, j);
          } else {
#pragma unroll
            for (int k = 0; k < GEMM_BK / 16; ++k) issue(k, half);
          }
          if (PAIR) {
            mma_commit_2sm(&empty[stage], 0x3);
            if (kb == num_kb - 1) mma_commit_2sm(&acc_full[buf], 0x3);
          } else {
            mma_commit(&empty[stage]);
            if (kb == num_kb - 1) mma_commit(&acc_full[buf]);
          }
        }
        __syncwarp();
#endif
        if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogue
    // Two warpgroups.  With double-buffered accumulators (NBUF = 2) warpgroup g
    // owns the tiles whose accumulator is buffer g, so each has two MMA-tile
    // durations for its epilogue; with NBUF = 1 they split the columns.
    //  * channels-last outputs: 32-column chunks staged in a 64B-swizzled
    //    [128 rows x 64 B] smem box, written by one TMA store per chunk;
    //  * NCHW (residual) / V^T outputs: 16-column pieces transposed through smem,
    //    each thread moving 32 contiguous bytes along the token axis.
    const int wg = (warp - 4) >> 2;  // epilogue warpgroup
    const int wq = warp & 3;         // TMEM lane quadrant
    const int row = wq * 32 + lane;  // tile row = TMEM lane
    const int bar_id = 1 + wg;
    const bool wg_leader = (warp & 3) == 0 && lane == 0;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    uint8_t* box_base = tma_stage + wg * Cfg::TMA_BUFS * (GEMM_BM * 64);  // TMA_BUFS 8 KB boxes per warpgroup
    // transposed (NCHW / V^T) stores: a [16][128] fp32 tile per warpgroup, or with
    // warp_store a [16][32] tile per warp (its own 32 rows; only __syncwarp needed)
    const bool wst = GEMM_NWG > 2 || p.warp_store != 0;
    const int st_ld = wst ? 32 : GEMM_BM;
    // GEMM_NWG > 2: the per-warp transpose tile aliases the warp's idle TMA-store box
    // (2 KB; the box two stores back has been read once bulk_wait_read<1> returns)
    float* st = GEMM_NWG > 2 ? nullptr : wst ? epi_stage + (warp - 4) * 16 * 32 : epi_stage + wg * 16 * GEMM_BM;
    const int st_row = wst ? lane : row;
    const int ci = wst ? lane >> 1 : row >> 3, seg = wst ? lane & 1 : row & 7;  // transposed role
    // NBUF == 1 or epi_split: the two warpgroups split every tile's columns (each tile's
    // accumulator drains in half the time); else warpgroup g takes the tiles of buffer g
    const bool split = GEMM_NWG > 2 || Cfg::NBUF == 1 || (p.epi_split && (BN / 2) % 32 == 0);
    // GEMM_NWG > 2: 32-column chunks dealt round-robin to the warpgroups
    const int c_step = GEMM_NWG > 2 ? 32 * GEMM_NWG : 32;
    const int c_lo = GEMM_NWG > 2 ? wg * 32 : split ? wg * (BN / 2) : 0;
    const int c_hi = GEMM_NWG > 2 ? BN : split ? c_lo + BN / 2 : BN;
    int n_store = 0;
    int li = 0;
    // the accumulator buffer is released on the leader CTA's barrier (the MMA issuer's)
    auto release = [&](int b) {
      if (PAIR) mbar_arrive_cluster(mapa_shared(&acc_empty[b], 0));
      else mbar_arrive(&acc_empty[b]);
    };
    for (int w = unit0; w < n_items; w += unit_step, ++li) {
      int half;
      const int t = item(w, half);
      const int buf = li % Cfg::NBUF;
      const int use = li / Cfg::NBUF;
      if (!split && buf != wg) continue;
      const int m_tile = my_m(t), n_tile = t % num_n;
      const int m = m_tile * GEMM_BM + row;
      const bool row_ok = m < p.M;
      const bool tile_full = (m_tile + 1) * GEMM_BM <= p.M;
      const int pidx = p.hw > 0 ? m / p.hw : 0;
      const int pix = p.hw > 0 ? m - pidx * p.hw : 0;
      const int tok_v = m_tile * GEMM_BM + (wst ? wq * 32 : 0) + seg * 16;
      const int pidx_v = p.hw > 0 ? tok_v / p.hw : 0;
      const int pix_v = p.hw > 0 ? tok_v - pidx_v * p.hw : 0;
      const bool vec_nchw = p.epi == EPI_RESID_NCHW && (p.hw % (wst ? 32 : 16)) == 0 && tile_full;
      const bool vec_vt = p.epi == EPI_SPLIT_VT && (p.ldo2 % 8) == 0 && tile_full;
      timed_wait(&acc_full[buf], use & 1, t_wait);
      tc_fence_after();
      if (m_tile < 0 || n_tile * BN + c_lo >= p.N) {  // no rows / columns of this tile here
        tc_fence_before();
        release(buf);
        continue;
      }
      auto load_bias = [&](float (&bv)[32], int nb) {
        if (p.bias != nullptr) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 b4 = __ldg(reinterpret_cast<const float4*>(p.bias + nb) + q);
            bv[4 * q] = b4.x; bv[4 * q + 1] = b4.y; bv[4 * q + 2] = b4.z; bv[4 * q + 3] = b4.w;
          }
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) bv[i] = 0.f;
        }
      };
      // chunk body: bias (+GELU) and store of 32 accumulator columns [c, c + 32) held in r
      auto body = [&](const uint32_t (&r)[32], const float (&bv)[32], int c) {
        const int nb = n_tile * BN + c;
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) + (PS_GEMM_LAZY_BIAS ? 0.f : bv[i]);
        if (PS_GEMM_LAZY_BIAS && p.bias != nullptr) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float4 b4 = __ldg(reinterpret_cast<const float4*>(p.bias + nb) + q);
            v[4 * q] += b4.x; v[4 * q + 1] += b4.y; v[4 * q + 2] += b4.z; v[4 * q + 3] += b4.w;
          }
        }
        const bool cl_tma = p.store_tma &&
                            (p.epi == EPI_STORE_CL || p.epi == EPI_GELU_CL || (p.epi == EPI_SPLIT_VT && nb < p.n_split));
        if (cl_tma) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            pk[e] = pack_bf16(v[2 * e], v[2 * e + 1]);
            if (p.epi == EPI_GELU_CL) pk[e] = gelu_bf16x2(pk[e]);
          }
          if (p.warp_store) {
            // per-warp 32x32 box: no cross-warp barrier, lane 0 issues the TMA store
            uint8_t* box = tma_stage + (warp - 4) * (Cfg::TMA_BUFS * 2048) + (n_store % Cfg::TMA_BUFS) * 2048;
            if (lane == 0) bulk_wait_read<Cfg::TMA_BUFS - 1>();
            __syncwarp();
#pragma unroll
            for (int q = 0; q < 4; ++q)
              *reinterpret_cast<uint4*>(box + lane * 64 + ((q ^ ((lane >> 1) & 3)) << 4)) =
                  make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
              if (p.out_tiled)
                tma_store_2d(&tmC, box, nb & 63, (m_tile * (p.ldo / 64) + nb / 64) * GEMM_BM + wq * 32);
              else
                tma_store_2d(&tmC, box, nb, m_tile * GEMM_BM + wq * 32);
              bulk_commit();
            }
            ++n_store;
            return;
          }
          uint8_t* box = box_base + (n_store % Cfg::TMA_BUFS) * (GEMM_BM * 64);
          if (wg_leader) bulk_wait_read<Cfg::TMA_BUFS - 1>();  // the TMA store that last used this box has read it
          named_bar_sync(bar_id, 128);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<uint4*>(box + row * 64 + ((q ^ ((row >> 1) & 3)) << 4)) =
                make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
          fence_proxy_async();
          named_bar_sync(bar_id, 128);
          if (wg_leader) {
            if (p.out_tiled)
              tma_store_2d(&tmC, box, nb & 63, (m_tile * (p.ldo / 64) + nb / 64) * GEMM_BM);
            else
              tma_store_2d(&tmC, box, nb, m_tile * GEMM_BM);
            bulk_commit();
          }
          ++n_store;
          return;
        }
        if (p.epi == EPI_GELU_CL) {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float x = v[i];
            const float u = 0.7978845608028654f * fmaf(0.044715f * x, x * x, x);
            const float hx = 0.5f * x;
            v[i] = fmaf(hx, tanh_fast(u), hx);
          }
        }
#pragma unroll
        for (int s16 = 0; s16 < 32; s16 += 16) {
          const int n0 = nb + s16;
          if (n0 >= p.N) break;
          const bool tr_vt = vec_vt && n0 >= p.n_split;
          if (vec_nchw || tr_vt) {
            // transposed store: thread (column n0 + ci, tokens tok_v .. +15)
            const int nv = n0 + ci;
            const size_t off_v = tr_vt ? (size_t)(nv - p.n_split) * p.ldo2 + tok_v
                                       : ((size_t)pidx_v * p.c_real + nv) * p.hw + pix_v;
            uint4 rs0 = make_uint4(0, 0, 0, 0), rs1 = rs0;
            if (vec_nchw && p.resid != nullptr && nv < p.c_real) {
              rs0 = __ldg(reinterpret_cast<const uint4*>(p.resid + off_v));
              rs1 = __ldg(reinterpret_cast<const uint4*>(p.resid + off_v) + 1);
            }
            if constexpr (GEMM_NWG > 2) {
              if (lane == 0 && p.store_tma) bulk_wait_read<Cfg::TMA_BUFS - 1>();
              __syncwarp();
              st = reinterpret_cast<float*>(tma_stage + (warp - 4) * (Cfg::TMA_BUFS * 2048) +
                                            (n_store % Cfg::TMA_BUFS) * 2048);
            }
            // per-warp [16][32] tile: 16-byte groups XOR-swizzled by row, so the transposed
            // float4 reads (16 lanes on 16 rows of one column range) hit distinct banks -- plain
            // [16][32] reads were 16-way bank conflicts; writes stay a permutation of each row
#pragma unroll
            for (int i = 0; i < 16; ++i) st[i * st_ld + (wst ? st_row ^ ((i & 7) << 2) : st_row)] = v[s16 + i];
            if (wst) __syncwarp();
            else named_bar_sync(bar_id, 128);
            if (tr_vt || nv < p.c_real) {
              const float4* src = reinterpret_cast<const float4*>(st + ci * st_ld);
              const int swz = wst ? (ci & 7) << 2 : 0;
              float o[16];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float4 f = src[((seg * 16 + 4 * q) ^ swz) >> 2];
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
              store16_cl((tr_vt ? p.out2 : p.out) + off_v, o);
            }
            if (wst) __syncwarp();
            else named_bar_sync(bar_id, 128);
            continue;  // next 16-column piece
          }
          if (!row_ok) continue;
          if (p.epi == EPI_STORE_CL || p.epi == EPI_GELU_CL || p.epi == EPI_SPLIT_VT) {
            if (p.epi == EPI_SPLIT_VT && n0 >= p.n_split) {
#pragma unroll
              for (int i = 0; i < 16; ++i)
                p.out2[(size_t)(n0 + i - p.n_split) * p.ldo2 + m] = __float2bfloat16_rn(v[s16 + i]);
            } else if (p.out_tiled) {
              store16_cl(p.out + (((size_t)m_tile * (p.ldo / 64) + n0 / 64) * GEMM_BM + row) * 64 + (n0 & 63),
                         v + s16);
            } else {
              store16_cl(p.out + (size_t)m * p.ldo + n0, v + s16);
            }
          } else {  // EPI_RESID_NCHW, ragged tile: scalar path
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int n = n0 + i;
              if (n < p.c_real) {
                const size_t off = ((size_t)pidx * p.c_real + n) * p.hw + pix;
                float x = v[s16 + i];
                if (p.resid != nullptr) x += bf(p.resid[off]);
                p.out[off] = __float2bfloat16_rn(x);
              }
            }
          }
        }
      };
      int c_end = min(c_hi, p.N - n_tile * BN);  // columns of this tile for this warpgroup
      int c_beg = c_lo;
      if (half >= 0) {  // a tail item: only this column half of the accumulator was computed
        c_beg = half * Cfg::MMA_N + (c_lo % Cfg::MMA_N);
        c_end = min(c_end, (half + 1) * Cfg::MMA_N);
        if (c_beg >= c_end) {
          tc_fence_before();
          release(buf);
          continue;
        }
      }
#pragma unroll 1
      for (int c = c_beg; c < c_end; c += c_step) {
        uint32_t r[32];
        PS_TMEM_LD32(tmem + lane_base + buf * BN + c, r);
        float bv[32];
        if (!PS_GEMM_LAZY_BIAS) load_bias(bv, n_tile * BN + c);
        tmem_ld_wait();
        reg_fence32(r);
        if (c + c_step >= c_end) {
          // last chunk of this tile for this warpgroup: hand the accumulator back early
          tc_fence_before();
          release(buf);
        }
        if (!p.epi_skip) body(r, bv, c);
      }
    }
  }
  if (warp >= 4 && lane == 0 && p.store_tma) bulk_wait<0>();  // (per-warp or warpgroup-leader stores)
  if (p.dbg && lane == 0) {
    const unsigned long long tot = clock64() - t_start;
    if (warp == 0) { atomicAdd(p.dbg + 0, t_wait); atomicAdd(p.dbg + 1, tot); }
    if (warp == 1) { atomicAdd(p.dbg + 2, t_wait); atomicAdd(p.dbg + 3, t_wait2); atomicAdd(p.dbg + 4, tot); }
    if (warp == 4) { atomicAdd(p.dbg + 5, t_wait); atomicAdd(p.dbg + 6, tot); }
  }
  tc_fence_before();
  if (PAIR) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  if (warp == 2) {
    if (PAIR) tmem_dealloc_2sm(tmem, Cfg::TMEM_COLS);
    else tmem_dealloc(tmem, Cfg::TMEM_COLS);
  }
}

static int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN, bool PAIR>
static int launch_bn(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, const GemmParams& p,
                     cudaStream_t st) {
  using Cfg = GemmCfg<BN, PAIR>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_tc_kernel<BN, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    attr = true;
  }
  const int num_m = p.m_map ? p.m_count : (p.M + GEMM_BM - 1) / GEMM_BM;
  const int units = (PAIR ? (num_m + 1) / 2 : num_m) * ((p.N + BN - 1) / BN);
  if (units == 0) return PS_OK;
  const int per_unit = PAIR ? 2 : 1;
  const int max_units = num_sms() / per_unit;
  const int grid = (units < max_units ? units : max_units) * per_unit;
  if (!PAIR) {
    launch_pdl(gemm_tc_kernel<BN, false>, dim3(grid), dim3(GEMM_THREADS), Cfg::SMEM, st, a, b, c, p);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(GEMM_THREADS);
    cfg.dynamicSmemBytes = Cfg::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cudaLaunchKernelEx(&cfg, gemm_tc_kernel<BN, true>, a, b, c, p);
  }
  count_launch();
  return check_launch(PAIR ? "gemm_tc_pair" : "gemm_tc");
}

int gemm_launch(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, const GemmParams& p, int bn,
                int pair, cudaStream_t st) {
#define PS_GEMM_CASE(N)                                                           \
  case N:                                                                         \
    return pair ? launch_bn<N, true>(a, b, c, p, st) : launch_bn<N, false>(a, b, c, p, st);
  switch (bn) {
    PS_GEMM_CASE(64)
    PS_GEMM_CASE(128)
    PS_GEMM_CASE(160)
    PS_GEMM_CASE(192)
    PS_GEMM_CASE(256)
    PS_GEMM_CASE(320)
    default: return set_error(PS_ERR_INPUT, "unsupported GEMM tile N %d", bn);
  }
#undef PS_GEMM_CASE
}

int gemm_pick_bn(int n, int k, int epi) {
  // long reductions amortise a single accumulator: one 320-wide tile reads A once -- unless
  // the epilogue is the slow NCHW transpose, which then stalls the MMAs of the next tile:
  // two double-buffered 160-wide tiles instead (FF2 + residual 160 -> 135 us)
  if (n == 320 && k >= 1024) return epi == EPI_RESID_NCHW ? 160 : 320;
  static const int choices[] = {256, 192, 160, 128, 64};
  int best = 64, best_cost = 1 << 30;
  for (int bn : choices) {
    const int cost = (n + bn - 1) / bn * bn;
    if (cost < best_cost) { best_cost = cost; best = bn; }
  }
  return best;
}

}  // namespace ps
