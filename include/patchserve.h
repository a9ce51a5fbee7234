/*
 * patchserve.h — C ABI of the B200-native PatchedServe patch-execution path.
 *
 * One shared library (libpatchserve.so, sm_100a) exports these entry points.
 * They take plain device/host pointers, sizes and a CUDA stream (as void*);
 * no framework types cross the boundary.  Each entry cites the reference
 * interface it replaces (paths relative to /root/reference/pkg/src/mixserve/).
 * The Python facade (paper_2501_09253_b200/) binds them with ctypes and keeps
 * the reference's `mixserve` API drop-in; INTEGRATION.md shows the binding.
 *
 * Layouts:
 *   NCHW patch array  (P, C, ps, ps)            — CSPBatch.data / block I/O (csp.py:71)
 *   CL tokens         (P*ps*ps, Cp) bf16         — channels-last, Cp = C rounded up to 64
 *   CL frames         (P, ps+2, ps+2, Cp) bf16   — halo frames (patched.py:57-89), channels-last
 *   NCHW frames       (P, C, ps+2, ps+2)         — reference layout of exchange_halos
 * Integer metadata is int32; neighbour table (P, 8) in N,NE,E,SE,S,SW,W,NW order
 * (csp.py:20-23), -1 where absent.
 *
 * Errors: every entry returns PS_OK or an error code; ps_last_error() gives the
 * message.  PS_ERR_INPUT maps to mixserve.errors.InputError (errors.py:4-5),
 * PS_ERR_INTEGRITY to IntegrityError (errors.py:8-9).  Launch failures are
 * PS_ERR_CUDA.  No entry falls back to the CPU.
 */
#ifndef PATCHSERVE_H
#define PATCHSERVE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PS_OK 0
#define PS_ERR_INPUT 1
#define PS_ERR_INTEGRITY 2
#define PS_ERR_CUDA 3

#define PS_DTYPE_F32 0
#define PS_DTYPE_BF16 1
#define PS_DTYPE_F64 2

/* ABI version: bumped on every signature change (2: ps_blend_reassemble gained src_ptrs and
 * ps_csp_split_bias the nonfinite flag; 3: the cache entry points take the element dtype --
 * bf16 on the hot path, fp32 / fp64 for the numpy-interface drop-in -- and the reuse test is one
 * kernel with a per-patch ticket area at the end of its scratch).
 * Callers check ps_abi_version() == PS_ABI_VERSION after loading the library. */
#define PS_ABI_VERSION 3

/* ------------------------------------------------------------ library */
int ps_abi_version(void);
const char* ps_last_error(void);
/* Number of kernels this library has launched (process lifetime). */
uint64_t ps_launch_count(void);
/* Device properties check: returns PS_OK on an sm_100 device. */
int ps_device_check(int device);

/* ------------------------------------------------- CSP format (csp.py) */
/* Patch count / resolution count of a split: csp.py:117-140 validation. */
int ps_csp_count(int n_req, const int32_t* dims, int32_t patch_size, int32_t* n_patches, int32_t* n_res);
/* Integer half of split(): csp.py:142-179 (stable resolution-major order,
 * request/resolution offsets, per-patch request_index/ordinal/row/col,
 * 8-neighbour table).  Host arrays, sized from ps_csp_count. */
int ps_csp_build(int n_req, const int32_t* dims, int32_t patch_size, int32_t* order, int32_t* request_offset,
                 int32_t* resolution_dims, int32_t* resolution_offset, int32_t* request_index, int32_t* ordinal,
                 int32_t* row, int32_t* col, int32_t* neighbors);
/* Pixel half of split(): csp.py:161-167.  src_ptrs: DEVICE array [n_req] of
 * latent pointers (C, L, L) in storage-slot order; sides: DEVICE [n_req]. */
int ps_csp_split(void* stream, const uint64_t* src_ptrs, const int32_t* request_offset, const int32_t* sides,
                 int n_req, int C, int ps, int dtype, void* dst, int n_patches);
/* reassemble(): csp.py:196-214, the inverse copy into per-request latents. */
int ps_csp_reassemble(void* stream, const void* src, const uint64_t* dst_ptrs, const int32_t* request_offset,
                      const int32_t* sides, int n_req, int C, int ps, int dtype, int n_patches);

/* Fused step ends for a fixed-composition step (pipeline.py): split + prompt bias writes the
 * CSP fp32 latents and h = bf16(latent + prompts[request]) (csp.py:161-167 + model.py:163);
 * blend + reassemble writes (1 - rate) x + rate tanh(h) straight into the per-request images
 * (model.py:129-131 + csp.py:196-214).  fp32 latents, ps % 4 == 0.  dst may be NULL (no CSP
 * copy); blend then reads x from the input images src_ptrs (DEVICE [n_req]) instead of
 * `latent` (which may be NULL).  Image pointers are 32-byte aligned.  nonfinite (DEVICE int, may be
 * NULL; ps in {16, 32, 64}): set to 1 when an input latent is not finite -- kernels.py:20-24
 * rejects those; the caller reads the flag after the step and raises InputError. */
int ps_csp_split_bias(void* stream, const uint64_t* src_ptrs, const int32_t* request_offset, const int32_t* sides,
                      int n_req, int C, int ps, float* dst, int n_patches, const float* prompts, void* h,
                      int* nonfinite);
int ps_blend_reassemble(void* stream, const float* latent, const void* h, const float* rates,
                        const int32_t* request_offset, const int32_t* sides, int n_req, int C, int ps,
                        const uint64_t* dst_ptrs, int n_patches, const uint64_t* src_ptrs);

/* ----------------------------------------- patched operators (patched.py) */
/* exchange_halos(): patched.py:57-89, NCHW frames (P, C, ps+2, ps+2). */
int ps_halo_frames_nchw(void* stream, const void* src, int dtype, const int32_t* neighbors, int P, int C, int ps,
                        void* dst);
/* Per-(patch, group) partial moments of an NCHW bf16 array (first half of
 * stitched_group_norm, patched.py:132-137).  partials: fp32 [P, G, 2] (mean, M2). */
int ps_gn_partials(void* stream, const void* x, int P, int C, int ps, int G, float* partials);
/* ps_gn_partials over a DEVICE list of n patch indices (the patches a GPU owns
 * in the split-image path); other rows of `partials` are untouched. */
int ps_gn_partials_sub(void* stream, const void* x, int P, int C, int ps, int G, const int32_t* patches, int n,
                       float* partials, const int32_t* n_dev);
/* Pool partials per request into mean / rstd (patched.py:135-140, eps).
 * stats: fp32 [R, G, 2] (mean, rstd). */
int ps_gn_finalize(void* stream, const float* partials, const int32_t* request_offset, int R, int G, int cg_hw,
                   float eps, float* stats);
/* NCHW (bf16) -> CL tokens, with optional per-image GroupNorm affine or
 * LayerNorm (kernels.py:209-227).  mode: 0 copy, 1 group_norm, 2 layer_norm. */
int ps_to_cl(void* stream, const void* x, int P, int C, int ps, int Cp, int mode, const float* stats,
             const int32_t* request_index, int G, const float* gamma, const float* beta, float eps, void* out);
/* NCHW (bf16) -> CL halo frames (P, ps+2, ps+2, Cp), optionally GroupNorm-ed on
 * the fly: the fused "stitcher" of stitched_group_norm(emit_halos=True),
 * patched.py:141-144 / PAPER.md:371-373.  mode: 0 copy, 1 group_norm. */
int ps_frames_cl(void* stream, const void* x, int P, int C, int ps, int Cp, int mode, const float* stats,
                 const int32_t* request_index, const int32_t* neighbors, int G, const float* gamma,
                 const float* beta, void* out);
/* ps_frames_cl for a DEVICE list of n patch indices only (split-image path). */
int ps_frames_cl_sub(void* stream, const void* x, int P, int C, int ps, int Cp, int mode, const float* stats,
                     const int32_t* request_index, const int32_t* neighbors, int G, const float* gamma,
                     const float* beta, const int32_t* patches, int n, void* out, const int32_t* n_dev);
/* CL tokens -> NCHW bf16, optionally adding an NCHW bf16 residual (patched.py:215-217). */
int ps_from_cl(void* stream, const void* x_cl, int P, int C, int ps, int Cp, const void* resid, void* out);

/* ------------------------------- split-image exchange movers */
/* Halo strips of an NCHW bf16 patch array across a shard cut (the cross-GPU part
 * of exchange_halos, patched.py:57-89): desc DEVICE [n][2] = (patch, code), code
 * < ps = pixel row, code >= ps = pixel column code-ps; buf [n][C][ps] bf16.
 * unpack = 0: x -> buf, 1: buf -> x. */
int ps_halo_strips(void* stream, void* x, int C, int ps, int n, const int32_t* desc, void* buf, int unpack);
/* n segments of seg_bytes (even): dst + dst_off[i] <- src + src_off[i] (DEVICE
 * int64 byte offsets).  Packs GroupNorm partials (patched.py:132-140) and
 * attention K rows / V^T columns (patched.py:164-176) into NCCL buffers and back. */
int ps_copy_segments(void* stream, const void* src, void* dst, int n, const int64_t* src_off, const int64_t* dst_off,
                     int64_t seg_bytes);
/* As ps_copy_segments with a byte count per segment (seg_bytes[i], even): the split-image K / V^T
 * pack and unpack of every peer's token ranges in one launch.  No reference counterpart. */
int ps_copy_segments_var(void* stream, const void* src, void* dst, int n, const int64_t* src_off,
                         const int64_t* dst_off, const int64_t* seg_bytes);

/* Dense contraction on tcgen05: D[M,N] = A[M,K] B[N,K]^T (+bias), bf16 in, fp32 accumulate.
 * a: CL tokens [M, lda] (a_mode 0), CL frames (a_mode 1: implicit conv3, K = 9*Cp,
 *    B laid out [N, 9*Cp] with K index tap*Cp + c, tap = ky*3 + kx), or tile-major
 *    tokens (a_mode 2: [ceil(M/128)][K/64][128][64], as written with out_tiled = 1).
 * epi: 0 -> out CL [M, ldo]; 1 -> GELU then out CL; 2 -> out NCHW (P, c_real, ps, ps)
 *      with optional NCHW residual `resid`; 3 -> columns < n_split to out [M, ldo],
 *      the rest transposed to out2 [N - n_split, ldo2].
 * Replaces _channel_matmul / _conv_valid / attend_tokens projections
 * (kernels.py:99-111, 148-161, 264-267) behind patched_conv / feed_forward. */
typedef struct ps_gemm_args {
  const void* a; int lda; int M;
  int a_mode; int P; int ps; int Cp;      /* a_mode 1 geometry */
  const void* b; int N; int K;           /* B [N, K] bf16, row-major */
  const float* bias;
  int epi; void* out; int ldo; void* out2; int ldo2; int n_split;
  const void* resid; int c_real;
  int bn;                                 /* tile N: 64,128,160,192,256,320 (0 = auto) */
  int out_tiled;                          /* epi 0/1: write tile-major [ceil(M/128)][ldo/64][128][64] */
  unsigned long long* dbg;                /* optional device counters [8] of per-role wait cycles, or NULL */
  const int32_t* m_map;                   /* optional DEVICE list of 128-row tiles to compute (compaction) */
  int m_count;                            /* entries in m_map */
  int cta_pair;                           /* 0 auto, 1 single-CTA 128-row tiles, 2 CTA-pair 256-row tiles
                                             (tcgen05 cta_group::2) */
  const int32_t* m_count_dev;             /* optional DEVICE count of m_map entries (m_count is then an upper
                                             bound): compaction decided on the device, no host round trip */
} ps_gemm_args;
int ps_gemm(void* stream, const ps_gemm_args* args);

/* Fused feed-forward + residual on CTA pairs (kernels.py:124-127 + patched.py:215-217):
 * out NCHW (P, c_real, ps, ps) = W2 gelu_tanh(W1 x + b1) + b2 (+ resid NCHW), x CL [M, Cp],
 * W1 [Hp, Cp], W2 [Cp, Hp] bf16, biases fp32; the hidden activations never leave the SM.
 * Cp in {128, 192, 256, 320}, Hp % 128 == 0, ps*ps and M multiples of 128; m_map optional
 * (DEVICE list of 128-row tiles).  Bit-identical to the FF1 / FF2 ps_gemm pair. */
/* Profiling: device counters [14] of per-role barrier-wait cycles of later ps_feed_forward launches. */
int ps_feed_forward_debug(unsigned long long* counters);
int ps_feed_forward(void* stream, const void* x, int M, int Cp, const void* w1, const float* b1, const void* w2,
                    const float* b2, int Hp, int c_real, int ps, const void* resid, void* out, const int32_t* m_map,
                    int m_count, const int32_t* m_count_dev);

/* Per-image attention over the CSP token order (patched_self_attention,
 * patched.py:154-176 -> attend_tokens/_attend_single, kernels.py:230-267).
 * qk: [T, 2*Dp] bf16 (Q then K per token), vt: [Dp, ldv] bf16 (V transposed, ldv % 8 == 0),
 * img_tok0: DEVICE [n_img+1] token offsets; tiles: DEVICE [n_tiles] (q0, img).
 * out: [T, Dp] bf16 = softmax(Q K^T / sqrt(D)) V per image. */
int ps_attention(void* stream, const void* qk, const void* vt, int ldv, int T, int Dp, int D, const int32_t* img_tok0,
                 const int32_t* tile_q0, const int32_t* tile_img, int n_tiles, void* out);
/* Same as ps_attention on CTA pairs (cta_group::2, M = 256): each tile is 256
 * queries of one image (pair_q0 steps by 256); default path on B200.  n_dev: optional
 * DEVICE tile count (n_pairs is then an upper bound). */
int ps_attention_pairs(void* stream, const void* qk, const void* vt, int ldv, int T, int Dp, int D,
                       const int32_t* img_tok0, const int32_t* pair_q0, const int32_t* pair_img, int n_pairs,
                       void* out, const int32_t* n_dev);
/* Split-KV attention for few query tiles (a large image split across GPUs leaves a
 * GPU ~64 query tiles for 148 SMs): tile t (DEVICE arrays) covers key blocks
 * [tile_kb0[t], +tile_nkb[t]) of 128 keys of its image; tile_slot[t] >= 0 writes the
 * unnormalised fp32 O [slot][128][Dp] and (m, l) [slot][128][2] instead of `out`.
 * ps_attention_combine merges n query tiles: slots [slot0[i], +nsplit[i]) -> out rows
 * q0s[i] .. +128 (clipped to the image end via img_of / img_tok0).  Same math as
 * patched.py:154-176 (online softmax partials merged in log2 space). */
int ps_attention_splitkv(void* stream, const void* qk, const void* vt, int ldv, int T, int Dp, int D,
                         const int32_t* img_tok0, const int32_t* tile_q0, const int32_t* tile_img,
                         const int32_t* tile_kb0, const int32_t* tile_nkb, const int32_t* tile_slot, int n_tiles,
                         float* part_o, float* part_ml, void* out);
/* Split-KV on CTA pairs (the persistent pair kernel): pair tile t = 256 queries from pair_q0[t]
 * of image pair_img[t] over key blocks [kb0[t], kb0[t] + nkb[t]) of 128 keys.  slot0[t] >= 0:
 * the tile's two 128-row halves leave as fp32 partials (O unnormalised [slot][128][Dp], (m, l)
 * [slot][128]) in slots slot0[t] / slot1[t] for ps_attention_combine; slot0[t] < 0: the tile
 * covers all the image's keys and writes bf16 O to out.  Tiles are dealt in list order. */
int ps_attention_pairs_splitkv(void* stream, const void* qk, const void* vt, int ldv, int T, int Dp, int D,
                               const int32_t* img_tok0, const int32_t* pair_q0, const int32_t* pair_img,
                               const int32_t* kb0, const int32_t* nkb, const int32_t* slot0, const int32_t* slot1,
                               int n_pairs, float* part_o, float* part_ml, void* out);
int ps_attention_combine(void* stream, const float* part_o, const float* part_ml, const int32_t* q0s,
                         const int32_t* slot0, const int32_t* nsplit, const int32_t* img_of,
                         const int32_t* img_tok0, int n, int Dp, void* out);
/* Split images across GPUs without a K/V gather: ps_kv_peer_maps writes [2n] tensor maps
 * (K, V^T of each rank's persistent buffers, as this GPU addresses them over NVLink) into
 * device memory once; ps_attention_peer then TMA-loads every key block whose kb_src (per
 * local 128-token block, -1 = local) names a peer from that peer's buffers at token row
 * kb_row.  tile_kb0/tile_nkb/tile_slot/part_* are the optional split-KV arrays. */
int ps_kv_peer_maps(void* dst_device, int n, const uint64_t* qk_ptrs, const int32_t* T, const uint64_t* vt_ptrs,
                    const int32_t* ldv, int Dp);
int ps_attention_peer(void* stream, const void* qk, const void* vt, int ldv, int T, int Dp, int D,
                      const int32_t* img_tok0, const int32_t* tile_q0, const int32_t* tile_img,
                      const int32_t* tile_kb0, const int32_t* tile_nkb, const int32_t* tile_slot, int n_tiles,
                      float* part_o, float* part_ml, const int32_t* kb_src, const int32_t* kb_row,
                      const void* peer_maps, void* out);
/* Profiling: device counters [8] of per-role barrier-wait cycles for later ps_attention launches (NULL = off). */
int ps_attention_debug(unsigned long long* counters);
/* Profiling: device buffer [11][64] of clock64 stamps (per event, first 64 key blocks) of the
 * first CTA of later ps_attention_pairs launches: S issue start/end, PV issue start/end,
 * softmax S-ready / S-loaded / exp-done / P-free / P-stored, then the S / PV issuers' K / V wait
 * cycles per block (NULL = off). */
int ps_attention_trace(long long* stamps);

/* ------------------------------------------------------ patch cache (cache.py) */
/* Pairwise-summation plan of numpy's add-reduce for n elements (cache.py:54-55
 * via np.mean).  Sizes first (plan == NULL), then fill:
 *   leaves: int32 [2*n_leaves] (start, len); nodes: int32 [2*n_internal] child ids
 *   (ids < n_leaves are leaves), level_off: int32 [n_levels+1]. */
int ps_pairwise_plan(int64_t n, int32_t* n_leaves, int32_t* n_internal, int32_t* n_levels, int32_t* leaves,
                     int32_t* nodes, int32_t* level_off);
/* predict_reuse(): cache.py:107-122 with _mse_predictor (cache.py:87-88):
 * mask[p] = exists[slot] && mse(x[p], snap_in[slot]) < sigma && streak[slot] < max_streak,
 * mse bit-exact to numpy (fp64, same pairwise tree).  x, snap_in: (P, n) / (slots, n) of `dtype`
 * (PS_DTYPE_BF16 / F32 / F64; each element is widened exactly to fp64 before the subtraction);
 * slots: DEVICE int32 [P] (-1 = no entry); scratch: fp64 [P * (n_leaves + n_internal)] followed by
 * P int32 tickets, i.e. P * (n_leaves + n_internal) + (P + 1) / 2 doubles (the tickets are zeroed
 * on the stream by the call); scratch[p, n_leaves + n_internal - 1] holds patch p's sum of squares
 * afterwards (scratch[p, 0] when the tree is a single leaf); counters: int64 [2] += (reused, fresh).
 * One kernel: leaf sums per CTA, the last CTA of a patch evaluates its tree. */
int ps_cache_predict(void* stream, const void* x, int dtype, int P, int64_t n, const int32_t* slots,
                     const void* snap_in, const uint8_t* exists, const int32_t* streak, double sigma, int max_streak,
                     const int32_t* leaves, int n_leaves, const int32_t* nodes, int n_internal,
                     const int32_t* level_off, int n_levels, double* scratch, uint8_t* mask, int64_t* counters);
/* Active-patch compaction (np.flatnonzero(~mask), ascending) + count. */
/* All lists of a compacted block on the device (run_block_active without a host round trip):
 * mask [P] (1 = reused); rows_act / rows_live: 128-row GEMM tiles (tpp per patch) of the
 * active patches / of every patch of an image with an active patch, ascending; attention
 * query tiles (qpp of tq queries per patch: q0 = p*hw + tq*j, image) of the same sets in
 * `order` (the attention patch order), and the live patches ascending.  counts [6]: rows_act,
 * rows_live, attn_act, attn_live, active patches, live patches.  live_scratch: int32 [R]. */
int ps_compact_lists(void* stream, const uint8_t* mask, int P, const int32_t* request_index, int R,
                     const int32_t* order, int tpp, int qpp, int tq, int hw, int32_t* live_scratch, int32_t* rows_act,
                     int32_t* rows_live, int32_t* live_patches, int32_t* attn_q0_act, int32_t* attn_img_act,
                     int32_t* attn_q0_live, int32_t* attn_img_live, int32_t* counts);
int ps_compact(void* stream, const uint8_t* mask, int P, int32_t* active, int32_t* n_active, int32_t* reused,
               int32_t* n_reused);
/* gather(): cache.py:124-137 — cached (inputs, outputs) at masked rows, zeros elsewhere.
 * error_flag: int32, set to 1 when a masked patch has no entry (IntegrityError). */
/* The data-moving cache entry points below take n elements of `dtype` per patch row. */
int ps_cache_gather(void* stream, const uint8_t* mask, const int32_t* slots, const uint8_t* exists, int P,
                    int64_t n, int dtype, const void* snap_in, const void* snap_out, void* ins, void* outs, int32_t* error_flag);
/* batched_fill(): cache.py:139-151 — streak += 1 at masked rows; optional out copy. */
int ps_cache_fill(void* stream, const uint8_t* mask, const int32_t* slots, const uint8_t* exists, int32_t* streak,
                  int P, int64_t n, int dtype, const void* snap_out, void* out, int32_t* error_flag);
/* batched_update(): cache.py:153-169 — fresh snapshots, streak 0 at unmasked rows;
 * counters: int64 [2] += (refreshed, inserted). */
int ps_cache_update(void* stream, const uint8_t* mask, const int32_t* slots, uint8_t* exists, int32_t* streak,
                    int P, int64_t n, int dtype, const void* x, const void* y, void* snap_in, void* snap_out,
                    int64_t* counters);
/* evict_expired(): cache.py:171-181 — clear `exists` for listed slots. */
int ps_cache_evict(void* stream, uint8_t* exists, int32_t* streak, const int32_t* slots, int n_slots);
/* Block-level fusion of the engine's cache sequence (engine.py:137-142):
 * substitute: x_sub = mask ? snap_in[slot] : x   (patched.py:243-244)
 * finish:     masked -> y = snap_out[slot], streak++ (patched.py:246, cache.py:150)
 *             unmasked -> snap_in/out[slot] = x/y, streak = 0, exists = 1 (cache.py:165-169)
 * substitute with `patches` (DEVICE list, n_list entries or the DEVICE count n_dev) writes
 * those patches only (the live patches of a device-decided compaction). */
int ps_cache_substitute(void* stream, const uint8_t* mask, const int32_t* slots, int P, int64_t n, int dtype,
                        const void* x, const void* snap_in, void* x_sub, const int32_t* patches, int n_list, const int32_t* n_dev);
int ps_cache_finish(void* stream, const uint8_t* mask, const int32_t* slots, uint8_t* exists, int32_t* streak,
                    int P, int64_t n, int dtype, const void* x, void* y, void* snap_in, void* snap_out,
                    int64_t* counters);
/* masked selection used by masked_block_forward (patched.py:241-246): out = mask ? a : b. */
int ps_select_patches(void* stream, const uint8_t* mask, int P, int64_t n, int dtype, const void* a, const void* b,
                      void* out);

/* ------------------------------------------------ step wrapper (model.py) */
/* h = bf16(latent + prompt[request_index[p]])  (model.py:163, engine.py:131-132). */
int ps_prompt_bias(void* stream, const float* latent, const float* prompts, const int32_t* request_index, int P,
                   int C, int ps, void* h);
/* blend(): model.py:129-131 with per-request rate (model.py:156-166):
 * out = (1 - r) * latent + r * tanh(h), fp32 master latents. */
int ps_blend(void* stream, const float* latent, const void* h, const float* rates, const int32_t* request_index,
             int P, int C, int ps, float* out);
/* Dtype conversion helpers for the facade (f32 <-> bf16). */
int ps_convert(void* stream, const void* src, int src_dtype, void* dst, int dst_dtype, int64_t n);
/* *out ^= XOR fold of the buffer's 32-byte words (bytes % 32 == 0, data 32-byte aligned; the
 * caller zeroes *out).  No reference counterpart: an integrity check for resident latents and
 * cache snapshots, and the pure streaming-read ceiling bench.py measures the read-only kernels
 * (ps_gn_partials, ps_cache_predict) against. */
int ps_checksum(void* stream, const void* data, int64_t bytes, uint32_t* out);

#ifdef __cplusplus
}
#endif
#endif /* PATCHSERVE_H */
