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
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer (one lane), w2 TMEM
// allocator, w4..w7 epilogue (TMEM lanes 32*(w%4)..+31 = tile rows).
// Epilogues: bias (+GELU) -> channels-last bf16; bias + residual -> NCHW bf16
// (the block output / residual stream, reference patched.py:215-217); split
// store with the trailing columns written transposed (V^T for attention).
#include "common.cuh"
#include "ps_internal.h"

namespace ps {

constexpr int GEMM_BM = 128;
constexpr int GEMM_BK = 64;
constexpr int GEMM_THREADS = 256;

template <int BN>
struct GemmCfg {
  static constexpr int MMA_N = BN <= 256 ? BN : BN / 2;
  static constexpr int N_MMA = BN / MMA_N;
  static constexpr int A_BYTES = GEMM_BM * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 6 ? 6 : (200 * 1024) / STAGE_BYTES;
  static constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : BN <= 256 ? 256 : 512;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static_assert(MMA_N % 16 == 0 && MMA_N >= 16 && MMA_N <= 256, "invalid UMMA N");
};

template <int BN>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const GemmParams p) {
  using Cfg = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty = full + Cfg::STAGES;
  uint64_t* acc_full = empty + Cfg::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_tile = blockIdx.x, n_tile = blockIdx.y;
  const int n0 = n_tile * BN;
  const int num_kb = p.K / GEMM_BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------------------------------------------------------- producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int p0 = 0, y0 = 0;
      if (p.a_mode == A_CONV3) {
        p0 = (m_tile / p.conv_tpp) * p.conv_np;
        y0 = (m_tile % p.conv_tpp) * p.conv_rows;
      }
      const int kcb = p.conv_cp / GEMM_BK;
      for (int kb = 0; kb < num_kb; ++kb) {
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
        uint8_t* sb = sa + Cfg::A_BYTES;
        mbar_arrive_expect_tx(&full[stage], Cfg::STAGE_BYTES);
        if (p.a_mode == A_CONV3) {
          const int tap = kb / kcb, cb = kb % kcb;
          tma_load_4d(sa, &tmA, &full[stage], cb * GEMM_BK, tap % 3, y0 + tap / 3, p0);
        } else {
          tma_load_2d(sa, &tmA, &full[stage], kb * GEMM_BK, m_tile * GEMM_BM);
        }
#pragma unroll
        for (int j = 0; j < Cfg::N_MMA; ++j)
          tma_load_2d(sb + j * Cfg::MMA_N * 128, &tmB, &full[stage], kb * GEMM_BK, n0 + j * Cfg::MMA_N);
        if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // -------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = idesc_bf16_f32(GEMM_BM, Cfg::MMA_N);
    int stage = 0;
    uint32_t phase = 0;
    for (int kb = 0; kb < num_kb; ++kb) {
      mbar_wait(&full[stage], phase);
      tc_fence_after();
      if (lane == 0) {
        const uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
        const uint8_t* sb = sa + Cfg::A_BYTES;
#pragma unroll
        for (int k = 0; k < GEMM_BK / 16; ++k) {
          const uint64_t ad = sdesc_sw128(sa + k * 32);
#pragma unroll
          for (int j = 0; j < Cfg::N_MMA; ++j) {
            const uint64_t bd = sdesc_sw128(sb + j * Cfg::MMA_N * 128 + k * 32);
            mma_bf16_ss(tmem + j * Cfg::MMA_N, ad, bd, idesc, (kb | k) != 0);
          }
        }
        mma_commit(&empty[stage]);
        if (kb == num_kb - 1) mma_commit(acc_full);
      }
      __syncwarp();
      if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------------- epilogue
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const int m = m_tile * GEMM_BM + row;
    const bool row_ok = m < p.M;
    mbar_wait(acc_full, 0);
    tc_fence_after();
    const uint32_t tbase = tmem + ((uint32_t)(wq * 32) << 16);
    // NCHW addressing for this token row
    const int pidx = p.hw > 0 ? m / p.hw : 0;
    const int pix = p.hw > 0 ? m - pidx * p.hw : 0;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t r[32];
      PS_TMEM_LD32(tbase + c0, r);
      tmem_ld_wait();
      const int nb = n0 + c0;
      if (nb >= p.N) break;
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int n = nb + i;
        float x = __uint_as_float(r[i]);
        if (p.bias != nullptr && n < p.N) x += __ldg(p.bias + n);
        if (p.epi == EPI_GELU_CL) x = gelu_tanh(x);
        v[i] = x;
      }
      if (!row_ok) continue;
      if (p.epi == EPI_STORE_CL || p.epi == EPI_GELU_CL ||
          (p.epi == EPI_SPLIT_VT && nb + 32 <= p.n_split)) {
        __nv_bfloat16* dst = p.out + (size_t)m * p.ldo + nb;
        if (nb + 32 <= p.N) {
          uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 w;
            w.x = pack_bf16(v[8 * q + 0], v[8 * q + 1]);
            w.y = pack_bf16(v[8 * q + 2], v[8 * q + 3]);
            w.z = pack_bf16(v[8 * q + 4], v[8 * q + 5]);
            w.w = pack_bf16(v[8 * q + 6], v[8 * q + 7]);
            d4[q] = w;
          }
        } else {
          for (int i = 0; i < 32 && nb + i < p.N; ++i) dst[i] = __float2bfloat16_rn(v[i]);
        }
      } else if (p.epi == EPI_SPLIT_VT) {
        for (int i = 0; i < 32; ++i) {
          const int n = nb + i;
          if (n >= p.N) break;
          if (n < p.n_split)
            p.out[(size_t)m * p.ldo + n] = __float2bfloat16_rn(v[i]);
          else
            p.out2[(size_t)(n - p.n_split) * p.ldo2 + m] = __float2bfloat16_rn(v[i]);
        }
      } else {  // EPI_RESID_NCHW: block output, (P, C, ps, ps)
        for (int i = 0; i < 32; ++i) {
          const int n = nb + i;
          if (n >= p.c_real) break;
          const size_t off = ((size_t)pidx * p.c_real + n) * p.hw + pix;
          float x = v[i];
          if (p.resid != nullptr) x += bf(p.resid[off]);
          p.out[off] = __float2bfloat16_rn(x);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, Cfg::TMEM_COLS);
}

template <int BN>
static int launch_bn(const CUtensorMap& a, const CUtensorMap& b, const GemmParams& p, cudaStream_t st) {
  using Cfg = GemmCfg<BN>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    attr = true;
  }
  dim3 grid((p.M + GEMM_BM - 1) / GEMM_BM, (p.N + BN - 1) / BN);
  gemm_tc_kernel<BN><<<grid, GEMM_THREADS, Cfg::SMEM, st>>>(a, b, p);
  count_launch();
  return check_launch("gemm_tc");
}

int gemm_launch(const CUtensorMap& a, const CUtensorMap& b, const GemmParams& p, int bn, cudaStream_t st) {
  switch (bn) {
    case 64: return launch_bn<64>(a, b, p, st);
    case 128: return launch_bn<128>(a, b, p, st);
    case 160: return launch_bn<160>(a, b, p, st);
    case 192: return launch_bn<192>(a, b, p, st);
    case 256: return launch_bn<256>(a, b, p, st);
    case 320: return launch_bn<320>(a, b, p, st);
    default: return set_error(PS_ERR_INPUT, "unsupported GEMM tile N %d", bn);
  }
}

}  // namespace ps
