// Internal declarations shared by the CUDA translation units and the C-ABI layer.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/patchserve.h"

namespace ps {

enum AMode { A_PLAIN = 0, A_CONV3 = 1, A_TILED = 2 };
enum Epi { EPI_STORE_CL = 0, EPI_GELU_CL = 1, EPI_RESID_NCHW = 2, EPI_SPLIT_VT = 3 };

struct GemmParams {
  int M, N, K;  // K is a multiple of 64 (channel padding)
  int a_mode;
  // conv3 geometry (A_CONV3): Cp, tiles per patch, patches per tile, frame rows per tile
  int conv_cp, conv_tpp, conv_np, conv_rows;
  int epi;
  const float* bias;  // [N] or null
  __nv_bfloat16* out;
  int ldo;
  __nv_bfloat16* out2;  // EPI_SPLIT_VT: transposed tail [N - n_split, ldo2]
  int ldo2, n_split;
  const __nv_bfloat16* resid;  // EPI_RESID_NCHW: block input (P, c_real, hw) or null
  int c_real, hw;
  int out_tiled;  // CL stores in 128x64 tile-major order ([M/128][ldo/64][128][64])
  unsigned long long* dbg;  // optional per-role wait-cycle counters (profiling)
  int store_tma;            // channels-last stores through the tmC tensor map
  const int* m_map;         // optional: physical 128-row tile of each logical tile (compaction)
  int m_count;              // number of mapped tiles when m_map != null (upper bound with m_count_dev)
  const int* m_count_dev;   // optional DEVICE count of mapped tiles (compaction without a host round trip)
  int epi_skip;             // profiling only (PS_GEMM_EPI_SKIP=1): drain accumulators without storing
  int epi_split;            // both epilogue warpgroups split each tile's columns (else alternate tiles)
  int no_prefetch;          // skip the L2 prefetch of residual rows
  int warp_store;           // channels-last TMA stores per warp (32x32 boxes) instead of per warpgroup
  int tail_split;           // BN = 320 (two N = 160 MMAs): the last partial wave's tiles become one
                            // work item per column half (A re-read, half the MMAs and epilogue)
};

struct FfParams {
  int M;                       // tokens (rows of x)
  const int* m_map;            // optional device list of 128-row tiles (compaction)
  int m_count;
  const int* m_count_dev;      // optional DEVICE count (m_count is then an upper bound)
  int hp;                      // hidden units (multiple of 128)
  int ts;                      // MMA2 reads GELU(H) from TMEM (else from shared memory)
  int tail_split;              // last partial wave split into output-channel halves
  const float* b1;             // [hp]
  const float* b2;             // [Cp]
  int c_real, hw;              // output channels, pixels per patch (NCHW output)
  const __nv_bfloat16* resid;  // NCHW residual or null
  __nv_bfloat16* out;          // NCHW (P, c_real, ps, ps)
  unsigned long long* dbg;     // optional role wait counters [12] (profiling)
};
int ff_launch(const CUtensorMap& x, const CUtensorMap& w1, const CUtensorMap& w2, const FfParams& p, int cp,
              int sms, cudaStream_t st);

int set_error(int code, const char* fmt, ...);
int check_launch(const char* what);
void count_launch();

// Programmatic dependent launch (PDL): the kernel may start while the previous kernel on the
// stream drains; it must execute griddepcontrol.wait (pdl_wait) before touching memory that
// kernel writes.  PS_PDL=0 launches normally.  Captured into CUDA graphs as programmatic edges.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, args...);
}
int gemm_launch(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, const GemmParams& p, int bn,
                int pair, cudaStream_t st);
int gemm_pick_bn(int n, int k, int epi);
// widest element span of `group` consecutive leaves of numpy's pairwise tree over n elements
int64_t pairwise_max_span(int64_t n, int group);
int pairwise_perfect_depth(int64_t n);

struct AttnParams {
  int T_total;   // tokens in the batch (rows of qk / columns of vt)
  int Dp;        // padded head dim (multiple of 64)
  int n_tiles;   // number of (image, 128-query) tiles
  const int* tile_q0;    // [n_tiles] first query token of the tile
  const int* tile_img;   // [n_tiles] image index
  const int* img_tok0;   // [n_img + 1] token offsets of images
  float scale_log2;      // log2(e) / sqrt(D_real)
  __nv_bfloat16* out;    // [T_total, Dp] channels-last
  unsigned long long* dbg;  // optional per-role wait counters (profiling)
  // split-KV (optional): tile t covers key blocks [tile_kb0[t], +tile_nkb[t]) of its image and,
  // when tile_slot[t] >= 0, writes unnormalised fp32 O [slot][128][Dp] and (m, l) [slot][128]
  const int* tile_kb0;
  const int* tile_nkb;
  const int* tile_slot;
  float* part_o;
  float* part_ml;
  // peer K / V (optional, split images across GPUs): key block b (128 local tokens) with
  // kb_src[b] >= 0 is read by TMA from peer kb_src[b]'s buffers, token row kb_row[b],
  // through the tensor maps peer_maps[2 s] (K) and peer_maps[2 s + 1] (V^T) in global memory
  const int* kb_src;
  const int* kb_row;
  const CUtensorMap* peer_maps;
  // profiling (ps_attention_trace): clock64 stamps of the first CTA (pair leader), [event][block]
  long long* trace;
  const int* n_dev;      // optional DEVICE tile count (n_tiles is then an upper bound)
  int epi_tma;           // pair kernel: O tiles staged in smem and TMA-stored (else row stores)
  int* tile_ctr;         // persistent pair kernel: [next tile, clusters done], zero between launches
  const int* tile_slot1; // split-KV pair tiles: partial slot of the second CTA's 128 rows
};
int attention_launch(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& vt, const AttnParams& p,
                     int dp, cudaStream_t st);
int attention_combine_launch(const float* part_o, const float* part_ml, const int* q0s, const int* slot0,
                             const int* nsplit, const int* img_of, const int* img_tok0, int n, int Dp,
                             __nv_bfloat16* out, cudaStream_t st);
int attention2_launch(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& vt, const CUtensorMap& o,
                      const AttnParams& p, int dp, cudaStream_t st);
int attention2_v_rows(int dp);

}  // namespace ps
