// C-ABI layer: error state, launch counting, TMA descriptor encoding, host-side
// metadata builders (CSP split plan, numpy pairwise-summation plan) and the GEMM /
// attention entry points.
#include <cudaTypedefs.h>
#include <stdarg.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <functional>
#include <mutex>
#include <numeric>
#include <vector>

#include "ps_internal.h"

namespace ps {

static thread_local char g_err[512] = "";
static std::atomic<uint64_t> g_launches{0};

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}
bool pdl_enabled() {
  static const bool on = !getenv("PS_PDL") || atoi(getenv("PS_PDL")) != 0;
  return on;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(PS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return PS_OK;
}
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// --------------------------------------------------------- tensor maps
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// bf16 tensor map with 128B swizzle; dims/strides innermost first (strides in bytes, rank-1 of them).
int make_tmap(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides_bytes,
              const uint32_t* box, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto fn = encode_fn();
  if (!fn) return set_error(PS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (reinterpret_cast<uintptr_t>(base) % 16) return set_error(PS_ERR_INPUT, "TMA base not 16B aligned");
  for (int i = 0; i < rank - 1; ++i)
    if (strides_bytes[i] % 16) return set_error(PS_ERR_INPUT, "TMA stride %d not a multiple of 16B", i);
  uint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base), dims, strides_bytes, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(PS_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return PS_OK;
}

int make_tmap_2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t ld_elems,
                 uint32_t box_rows) {
  uint64_t dims[2] = {cols, rows};
  uint64_t strides[1] = {ld_elems * 2};
  uint32_t box[2] = {64, box_rows};
  return make_tmap(m, base, 2, dims, strides, box);
}

// leaves (start, length) of numpy's pairwise_sum tree over n elements, in order
static void pairwise_leaves(int64_t lo, int64_t n, std::vector<std::pair<int64_t, int64_t>>& out) {
  if (n <= 128) {
    out.push_back({lo, n});
    return;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  pairwise_leaves(lo, n2, out);
  pairwise_leaves(lo + n2, n - n2, out);
}

// depth of numpy's pairwise tree over n elements when it is a perfect binary tree (every
// internal node's two subtrees are perfect of equal depth), else -1: then the leaf sums
// combine as adjacent pairs level by level, i.e. a plain in-order pairwise reduction.
static int pairwise_depth(int64_t n) {
  if (n <= 128) return 0;
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  const int a = pairwise_depth(n2), b = pairwise_depth(n - n2);
  return (a < 0 || a != b) ? -1 : a + 1;
}

int pairwise_perfect_depth(int64_t n) {
  static std::mutex mu;
  static std::vector<std::pair<int64_t, int>> memo;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : memo)
    if (e.first == n) return e.second;
  const int d = pairwise_depth(n);
  memo.push_back({n, d});
  return d;
}

int64_t pairwise_max_span(int64_t n, int group) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<int64_t, int>, int64_t>> memo;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : memo)
    if (e.first.first == n && e.first.second == group) return e.second;
  std::vector<std::pair<int64_t, int64_t>> lv;
  pairwise_leaves(0, n, lv);
  int64_t best = 0;
  for (size_t i = 0; i < lv.size(); i += group) {
    const size_t j = std::min(lv.size(), i + group) - 1;
    best = std::max(best, lv[j].first + lv[j].second - lv[i].first);
  }
  memo.push_back({{n, group}, best});
  return best;
}

}  // namespace ps

using namespace ps;

static unsigned long long* g_attn_dbg = nullptr;  // profiling hook (ps_attention_debug)
static long long* g_attn_trace = nullptr;           // profiling hook (ps_attention_trace)
static unsigned long long* g_ff_dbg = nullptr;      // profiling hook (ps_feed_forward_debug)

extern "C" {

int ps_abi_version(void) { return PS_ABI_VERSION; }
const char* ps_last_error(void) { return g_err; }
uint64_t ps_launch_count(void) { return g_launches.load(); }

int ps_device_check(int device) {
  cudaDeviceProp prop;
  cudaError_t e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return set_error(PS_ERR_CUDA, "cudaGetDeviceProperties: %s", cudaGetErrorString(e));
  if (prop.major != 10 || prop.minor != 0)
    return set_error(PS_ERR_CUDA, "device %d is sm_%d%d; this library is built for sm_100a", device, prop.major,
                     prop.minor);
  return PS_OK;
}

// ---------------------------------------------------------------- CSP plan
static int csp_validate(int n_req, const int32_t* dims, int32_t ps) {
  if (n_req < 1) return set_error(PS_ERR_INPUT, "empty batch");
  if (ps < 1) return set_error(PS_ERR_INPUT, "patch size must be positive, got %d", ps);
  for (int i = 0; i < n_req; ++i) {
    if (dims[i] <= 0) return set_error(PS_ERR_INPUT, "latent dims must be positive, got %d", dims[i]);
    if (dims[i] % ps) return set_error(PS_ERR_INPUT, "patch size %d does not tile latent dim %d", ps, dims[i]);
  }
  return PS_OK;
}

int ps_csp_count(int n_req, const int32_t* dims, int32_t ps, int32_t* n_patches, int32_t* n_res) {
  int rc = csp_validate(n_req, dims, ps);
  if (rc) return rc;
  int64_t total = 0;
  std::vector<int32_t> d(dims, dims + n_req);
  for (int i = 0; i < n_req; ++i) total += (int64_t)(d[i] / ps) * (d[i] / ps);
  if (total > INT32_MAX) return set_error(PS_ERR_INPUT, "too many patches");
  std::sort(d.begin(), d.end());
  *n_patches = (int32_t)total;
  *n_res = (int32_t)(std::unique(d.begin(), d.end()) - d.begin());
  return PS_OK;
}

// csp.py:142-179: stable sort by latent dim (ties keep arrival order), offsets,
// per-patch row-major ordinals and the 8-neighbour table (N,NE,E,SE,S,SW,W,NW).
int ps_csp_build(int n_req, const int32_t* dims, int32_t ps, int32_t* order, int32_t* request_offset,
                 int32_t* resolution_dims, int32_t* resolution_offset, int32_t* request_index, int32_t* ordinal,
                 int32_t* row, int32_t* col, int32_t* neighbors) {
  int rc = csp_validate(n_req, dims, ps);
  if (rc) return rc;
  static const int dr[8] = {-1, -1, 0, 1, 1, 1, 0, -1};
  static const int dc[8] = {0, 1, 1, 1, 0, -1, -1, -1};
  std::vector<int32_t> ord(n_req);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return dims[a] < dims[b]; });
  int32_t start = 0;
  request_offset[0] = 0;
  int n_res = 0;
  for (int s = 0; s < n_req; ++s) {
    const int src = ord[s];
    order[s] = src;
    const int side = dims[src] / ps;
    for (int r = 0; r < side; ++r)
      for (int c = 0; c < side; ++c) {
        const int p = start + r * side + c;
        request_index[p] = s;
        ordinal[p] = r * side + c;
        row[p] = r;
        col[p] = c;
        for (int d = 0; d < 8; ++d) {
          const int rr = r + dr[d], cc = c + dc[d];
          neighbors[p * 8 + d] = (rr >= 0 && rr < side && cc >= 0 && cc < side) ? start + rr * side + cc : -1;
        }
      }
    start += side * side;
    request_offset[s + 1] = start;
    if (n_res == 0 || resolution_dims[n_res - 1] != dims[src]) {
      resolution_dims[n_res] = dims[src];
      resolution_offset[n_res] = request_offset[s];
      ++n_res;
    }
  }
  resolution_offset[n_res] = start;
  return PS_OK;
}

// ------------------------------------------------------- pairwise plan
// numpy pairwise_sum (loops_utils.h.src, PW_BLOCKSIZE 128): n <= 128 is a leaf
// (sequential below 8, 8 strided accumulators otherwise); larger n splits at
// n2 = n/2 - (n/2 % 8).  Nodes are numbered leaves first (in order), then
// internal nodes grouped by height so a level can be evaluated in parallel.
static int attention_pairs_impl(void* stream, const void* qk, const void* vt, int ldv, int T, int Dp, int D,
                                const int32_t* img_tok0, const int32_t* pair_q0, const int32_t* pair_img,
                                int n_pairs, void* out, const int32_t* n_dev, const int32_t* kb0,
                                const int32_t* nkb, const int32_t* slot0, const int32_t* slot1, float* part_o,
                                float* part_ml) {
  if (Dp % 64 || Dp < 64 || Dp > 320) return set_error(PS_ERR_INPUT, "attention: Dp %d unsupported", Dp);
  if (D < 1 || D > Dp) return set_error(PS_ERR_INPUT, "attention: bad D");
  if (n_pairs < 1) return PS_OK;
  CUtensorMap tq, tk, tv, to;
  int rc = make_tmap_2d(&tq, qk, T, Dp, 2 * (uint64_t)Dp, 128);
  if (!rc) rc = make_tmap_2d(&tk, (const __nv_bfloat16*)qk + Dp, T, Dp, 2 * (uint64_t)Dp, 64);
  if (!rc) rc = make_tmap_2d(&tv, vt, Dp, T, ldv, attention2_v_rows(Dp));
  if (!rc) rc = make_tmap_2d(&to, out, T, Dp, Dp, 128);  // O tiles leave through TMA stores
  if (rc) return rc;
  AttnParams p{};
  p.T_total = T;
  p.Dp = Dp;
  p.n_tiles = n_pairs;
  p.tile_q0 = pair_q0;
  p.tile_img = pair_img;
  p.n_dev = n_dev;
  static const int epi_tma = getenv("PS_ATTN_EPI_TMA") ? atoi(getenv("PS_ATTN_EPI_TMA")) : 1;
  p.epi_tma = epi_tma;
  p.img_tok0 = img_tok0;
  p.scale_log2 = 1.4426950408889634f / sqrtf((float)D);
  p.out = (__nv_bfloat16*)out;
  p.dbg = g_attn_dbg;
  p.trace = g_attn_trace;
  p.tile_kb0 = kb0;
  p.tile_nkb = nkb;
  p.tile_slot = slot0;
  p.tile_slot1 = slot1;
  p.part_o = part_o;
  p.part_ml = part_ml;
  return attention2_launch(tq, tk, tv, to, p, Dp, (cudaStream_t)stream);
}

int ps_attention_pairs(void* stream, const void* qk, const void* vt, int ldv, int T, int Dp, int D,
                       const int32_t* img_tok0, const int32_t* pair_q0, const int32_t* pair_img, int n_pairs,
                       void* out, const int32_t* n_dev) {
  return attention_pairs_impl(stream, qk, vt, ldv, T, Dp, D, img_tok0, pair_q0, pair_img, n_pairs, out, n_dev,
                              nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
}

// Split-KV on CTA pairs: pair tile t (256 queries from pair_q0[t]) covers key blocks
// [kb0[t], kb0[t] + nkb[t]) of its image; with slot0[t] >= 0 the first / second 128 rows
// leave as fp32 partials in slots slot0[t] / slot1[t] (ps_attention_combine merges them),
// with slot0[t] < 0 the tile covers all its keys and writes bf16 O directly.
int ps_attention_pairs_splitkv(void* stream, const void* qk, const void* vt, int ldv, int T, int Dp, int D,
                               const int32_t* img_tok0, const int32_t* pair_q0, const int32_t* pair_img,
                               const int32_t* kb0, const int32_t* nkb, const int32_t* slot0, const int32_t* slot1,
                               int n_pairs, float* part_o, float* part_ml, void* out) {
  if (!kb0 || !nkb || !slot0 || !slot1) return set_error(PS_ERR_INPUT, "attention_pairs_splitkv: null tile arrays");
  if (!part_o || !part_ml) return set_error(PS_ERR_INPUT, "attention_pairs_splitkv: null partial buffers");
  static const bool persist = !getenv("PS_ATTN_PERSIST") || atoi(getenv("PS_ATTN_PERSIST")) != 0;
  if (!persist) return set_error(PS_ERR_INPUT, "attention_pairs_splitkv: needs the persistent pair kernel");
  return attention_pairs_impl(stream, qk, vt, ldv, T, Dp, D, img_tok0, pair_q0, pair_img, n_pairs, out, nullptr,
                              kb0, nkb, slot0, slot1, part_o, part_ml);
}

// Profiling only: device counters [8] that later attention launches accumulate
// per-role barrier-wait cycles into (NULL disables).
int ps_feed_forward_debug(unsigned long long* counters) {
  g_ff_dbg = counters;
  return PS_OK;
}

int ps_attention_trace(long long* stamps) {
  g_attn_trace = stamps;
  return PS_OK;
}

int ps_attention_debug(unsigned long long* counters) {
  g_attn_dbg = counters;
  return PS_OK;
}

int ps_pairwise_plan(int64_t n, int32_t* n_leaves, int32_t* n_internal, int32_t* n_levels, int32_t* leaves,
                     int32_t* nodes, int32_t* level_off) {
  if (n < 1 || n > (int64_t)1 << 30) return set_error(PS_ERR_INPUT, "pairwise plan: bad n %lld", (long long)n);
  struct Node { int64_t lo, len; int left, right, height; };
  std::vector<Node> tree;
  std::vector<std::pair<int64_t, int64_t>> lv;
  // recursive build (depth <= 30)
  std::function<int(int64_t, int64_t)> rec = [&](int64_t lo, int64_t len) -> int {
    if (len <= 128) {
      lv.push_back({lo, len});
      tree.push_back({lo, len, -1 - (int)(lv.size() - 1), -1, 0});
      return (int)tree.size() - 1;
    }
    int64_t n2 = len / 2;
    n2 -= n2 % 8;
    int l = rec(lo, n2);
    int r = rec(lo + n2, len - n2);
    tree.push_back({lo, len, l, r, std::max(tree[l].height, tree[r].height) + 1});
    return (int)tree.size() - 1;
  };
  rec(0, n);
  const int L = (int)lv.size();
  int H = 0;
  for (auto& t : tree) H = std::max(H, t.height);
  const int I = (int)tree.size() - L;
  *n_leaves = L;
  *n_internal = I;
  *n_levels = H;
  if (leaves == nullptr) return PS_OK;
  // final ids: leaf k -> k; internal nodes ordered by (height, post-order)
  std::vector<int> id(tree.size());
  int next = L;
  for (int h = 1; h <= H; ++h) {
    level_off[h - 1] = next - L;
    for (size_t i = 0; i < tree.size(); ++i)
      if (tree[i].height == h && tree[i].right >= 0) id[i] = next++;
  }
  level_off[H] = next - L;
  for (size_t i = 0; i < tree.size(); ++i)
    if (tree[i].right < 0) id[i] = -1 - tree[i].left;
  for (int k = 0; k < L; ++k) {
    leaves[2 * k] = (int32_t)lv[k].first;
    leaves[2 * k + 1] = (int32_t)lv[k].second;
  }
  for (size_t i = 0; i < tree.size(); ++i)
    if (tree[i].right >= 0) {
      const int j = id[i] - L;
      nodes[2 * j] = id[tree[i].left];
      nodes[2 * j + 1] = id[tree[i].right];
    }
  return PS_OK;
}

// ---------------------------------------------------------------- GEMM
int ps_gemm(void* stream, const ps_gemm_args* a) {
  if (!a || !a->a || !a->b || !a->out) return set_error(PS_ERR_INPUT, "gemm: null pointer");
  if (a->K % 64) return set_error(PS_ERR_INPUT, "gemm: K (%d) must be a multiple of 64", a->K);
  if (a->M < 1 || a->N < 1) return set_error(PS_ERR_INPUT, "gemm: empty problem");
  if (a->N % 16) return set_error(PS_ERR_INPUT, "gemm: N (%d) must be a multiple of 16", a->N);
  const int bn = a->bn ? a->bn : gemm_pick_bn(a->N, a->K, a->epi);
  const int mma_n = bn <= 256 ? bn : bn / 2;
  // CTA-pair tiles (cta_group::2) unless asked otherwise or the problem is too small to fill the SMs in pairs
  const int m_tiles = a->m_map ? a->m_count : (a->M + 127) / 128;
  // auto: CTA pairs for the long-K 320-wide tiles (conv3: 219 -> 207 us, tools/gemm_pair_check.py)
  // and, since the warp-wide MMA issue, for every GEMM with at least two waves of pair tiles
  // (O-projection 39 -> 35 us, QKV 90 -> 88 us, tools/gemm_roles.py pair); single-CTA tiles for
  // small (compacted) problems; PS_GEMM_PAIR=1|2 forces single|pairs
  static const int env_pair = getenv("PS_GEMM_PAIR") ? atoi(getenv("PS_GEMM_PAIR")) : 0;
  const int want = a->cta_pair ? a->cta_pair
                   : env_pair  ? env_pair
                               : ((bn == 320 && a->K >= 2048) || m_tiles >= 4 * 148 ? 2 : 1);
  const int pair = want == 2 && m_tiles >= 2 ? 1 : 0;
  CUtensorMap ta, tb;
  GemmParams p{};
  p.M = a->M;
  p.N = a->N;
  p.K = a->K;
  p.a_mode = a->a_mode;
  int rc;
  if (a->a_mode == A_CONV3) {
    const int ps_ = a->ps, hw = ps_ * ps_;
    if (a->K != 9 * a->Cp || a->Cp % 64) return set_error(PS_ERR_INPUT, "conv3 gemm: K must be 9*Cp, Cp %% 64 == 0");
    if ((ps_ & (ps_ - 1)) || ps_ > 128)
      return set_error(PS_ERR_INPUT, "conv3 gemm: patch size %d must be a power of two <= 128", ps_);
    p.conv_cp = a->Cp;
    if (hw >= 128) {
      p.conv_rows = 128 / ps_;
      p.conv_np = 1;
      p.conv_tpp = hw / 128;
    } else {
      p.conv_rows = ps_;
      p.conv_np = 128 / hw;
      p.conv_tpp = 1;
    }
    if (a->M != a->P * hw) return set_error(PS_ERR_INPUT, "conv3 gemm: M must be P*ps*ps");
    const uint64_t f = ps_ + 2;
    uint64_t dims[4] = {(uint64_t)a->Cp, f, f, (uint64_t)a->P};
    uint64_t strides[3] = {(uint64_t)a->Cp * 2, (uint64_t)a->Cp * 2 * f, (uint64_t)a->Cp * 2 * f * f};
    uint32_t box[4] = {64, (uint32_t)ps_, (uint32_t)p.conv_rows, (uint32_t)p.conv_np};
    rc = make_tmap(&ta, a->a, 4, dims, strides, box);
  } else if (a->a_mode == A_TILED) {
    const uint64_t rows = (uint64_t)((a->M + 127) / 128) * (a->K / 64) * 128;
    rc = make_tmap_2d(&ta, a->a, rows, 64, 64, 128);
  } else {
    rc = make_tmap_2d(&ta, a->a, a->M, a->K, a->lda, 128);
  }
  if (rc) return rc;
  rc = make_tmap_2d(&tb, a->b, a->N, a->K, a->K, pair ? mma_n / 2 : mma_n);
  if (rc) return rc;
  p.epi = a->epi;
  p.bias = a->bias;
  p.out = (__nv_bfloat16*)a->out;
  p.ldo = a->ldo;
  p.out2 = (__nv_bfloat16*)a->out2;
  p.ldo2 = a->ldo2;
  p.n_split = a->n_split;
  p.resid = (const __nv_bfloat16*)a->resid;
  p.c_real = a->c_real;
  p.hw = a->ps * a->ps;
  p.out_tiled = a->out_tiled;
  p.dbg = a->dbg;
  p.m_map = a->m_map;
  p.m_count = a->m_map ? a->m_count : 0;
  p.m_count_dev = a->m_map ? a->m_count_dev : nullptr;
  static const int epi_skip = getenv("PS_GEMM_EPI_SKIP") ? atoi(getenv("PS_GEMM_EPI_SKIP")) : 0;
  p.epi_skip = epi_skip;
  // defaults from tools/gemm_roles.py on config-2 shapes: splitting every tile's columns over both
  // epilogue warpgroups drains accumulators sooner (QKV 127 -> 120 us); the L2 prefetch of residual
  // rows by the TMA producer stalled it (FF2 + residual 223 -> 158 us without it)
  static const int epi_split = getenv("PS_GEMM_EPI_SPLIT") ? atoi(getenv("PS_GEMM_EPI_SPLIT")) : 1;
  static const int no_pf = getenv("PS_GEMM_NO_PF") ? atoi(getenv("PS_GEMM_NO_PF")) : 1;
  p.epi_split = epi_split;
  p.no_prefetch = no_pf;
  // channels-last outputs leave through TMA stores (32 rows x 16 columns per warp box)
  // per-warp epilogue stores (no cross-warp barriers): FF1 153 -> 128 us (tools/gemm_roles.py)
  static const int warp_store = getenv("PS_GEMM_WARP_STORE") ? atoi(getenv("PS_GEMM_WARP_STORE")) : 1;
  p.warp_store = warp_store;
  static const int gemm_tail = getenv("PS_GEMM_TAIL_SPLIT") ? atoi(getenv("PS_GEMM_TAIL_SPLIT")) : 1;
  p.tail_split = gemm_tail;
  CUtensorMap tc;
  memset(&tc, 0, sizeof(tc));
  p.store_tma = 0;
  static const int no_tma_store = getenv("PS_GEMM_NO_TMA_STORE") ? atoi(getenv("PS_GEMM_NO_TMA_STORE")) : 0;
  if (!no_tma_store && (a->epi == EPI_STORE_CL || a->epi == EPI_GELU_CL || a->epi == EPI_SPLIT_VT) && a->ldo % 8 == 0) {
    uint64_t dims[2], strides[1];
    if (a->out_tiled) {
      dims[0] = 64;
      dims[1] = (uint64_t)((a->M + 127) / 128) * (a->ldo / 64) * 128;
      strides[0] = 128;
    } else {
      dims[0] = (uint64_t)(a->epi == EPI_SPLIT_VT ? a->n_split : a->N);
      dims[1] = (uint64_t)a->M;
      strides[0] = (uint64_t)a->ldo * 2;
    }
    uint32_t box[2] = {32, (uint32_t)(p.warp_store ? 32 : 128)};
    rc = make_tmap(&tc, a->out, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
    p.store_tma = 1;
  }
  if (a->out_tiled && (a->epi > EPI_GELU_CL || a->ldo % 64 || bn % 64))
    return set_error(PS_ERR_INPUT, "gemm: tiled output needs a channels-last epilogue and ldo %% 64 == 0");
  if (a->epi == EPI_RESID_NCHW && (a->ps < 1 || a->c_real < 1 || a->c_real > a->N))
    return set_error(PS_ERR_INPUT, "gemm: NCHW epilogue needs ps and 1 <= c_real <= N");
  if ((a->epi == EPI_STORE_CL || a->epi == EPI_GELU_CL) && (a->ldo < a->N || a->ldo % 8))
    return set_error(PS_ERR_INPUT, "gemm: ldo must be >= N and a multiple of 8");
  return gemm_launch(ta, tb, tc, p, bn, pair, (cudaStream_t)stream);
}

// ----------------------------------------------------------- attention
int ps_attention(void* stream, const void* qk, const void* vt, int ldv, int T, int Dp, int D, const int32_t* img_tok0,
                 const int32_t* tile_q0, const int32_t* tile_img, int n_tiles, void* out) {
  if (Dp % 64 || Dp < 64 || Dp > 320) return set_error(PS_ERR_INPUT, "attention: Dp %d unsupported", Dp);
  if (D < 1 || D > Dp) return set_error(PS_ERR_INPUT, "attention: bad D");
  if (n_tiles < 1) return PS_OK;
  CUtensorMap tq, tk, tv;
  int rc = make_tmap_2d(&tq, qk, T, Dp, 2 * (uint64_t)Dp, 128);
  if (!rc) rc = make_tmap_2d(&tk, (const __nv_bfloat16*)qk + Dp, T, Dp, 2 * (uint64_t)Dp, 128);
  if (!rc) rc = make_tmap_2d(&tv, vt, Dp, T, ldv, 64);
  if (rc) return rc;
  AttnParams p{};
  p.T_total = T;
  p.Dp = Dp;
  p.n_tiles = n_tiles;
  p.tile_q0 = tile_q0;
  p.tile_img = tile_img;
  p.img_tok0 = img_tok0;
  p.scale_log2 = 1.4426950408889634f / sqrtf((float)D);
  p.out = (__nv_bfloat16*)out;
  p.dbg = g_attn_dbg;
  return attention_launch(tq, tk, tv, p, Dp, (cudaStream_t)stream);
}

}  // extern "C"

extern "C" {
// Split-KV attention (few query tiles per GPU, e.g. one large image split across GPUs):
// tile t = (q0, img, first key block kb0, key blocks nkb, partial slot or -1).
int ps_attention_splitkv(void* stream, const void* qk, const void* vt, int ldv, int T, int Dp, int D,
                         const int32_t* img_tok0, const int32_t* tile_q0, const int32_t* tile_img,
                         const int32_t* tile_kb0, const int32_t* tile_nkb, const int32_t* tile_slot, int n_tiles,
                         float* part_o, float* part_ml, void* out) {
  if (Dp % 64 || Dp < 64 || Dp > 320) return set_error(PS_ERR_INPUT, "attention: Dp %d unsupported", Dp);
  if (D < 1 || D > Dp) return set_error(PS_ERR_INPUT, "attention: bad D");
  if (!tile_kb0 || !tile_nkb || !tile_slot) return set_error(PS_ERR_INPUT, "attention_splitkv: null tile arrays");
  if (n_tiles < 1) return PS_OK;
  CUtensorMap tq, tk, tv;
  int rc = make_tmap_2d(&tq, qk, T, Dp, 2 * (uint64_t)Dp, 128);
  if (!rc) rc = make_tmap_2d(&tk, (const __nv_bfloat16*)qk + Dp, T, Dp, 2 * (uint64_t)Dp, 128);
  if (!rc) rc = make_tmap_2d(&tv, vt, Dp, T, ldv, 64);
  if (rc) return rc;
  AttnParams p{};
  p.T_total = T;
  p.Dp = Dp;
  p.n_tiles = n_tiles;
  p.tile_q0 = tile_q0;
  p.tile_img = tile_img;
  p.img_tok0 = img_tok0;
  p.scale_log2 = 1.4426950408889634f / sqrtf((float)D);
  p.out = (__nv_bfloat16*)out;
  p.dbg = g_attn_dbg;
  p.tile_kb0 = tile_kb0;
  p.tile_nkb = tile_nkb;
  p.tile_slot = tile_slot;
  p.part_o = part_o;
  p.part_ml = part_ml;
  return attention_launch(tq, tk, tv, p, Dp, (cudaStream_t)stream);
}

int ps_attention_combine(void* stream, const float* part_o, const float* part_ml, const int32_t* q0s,
                         const int32_t* slot0, const int32_t* nsplit, const int32_t* img_of,
                         const int32_t* img_tok0, int n, int Dp, void* out) {
  if (Dp % 8) return set_error(PS_ERR_INPUT, "attention_combine: Dp %% 8 != 0");
  return attention_combine_launch(part_o, part_ml, q0s, slot0, nsplit, img_of, img_tok0, n, Dp,
                                  (__nv_bfloat16*)out, (cudaStream_t)stream);
}
}  // extern "C"

extern "C" {
// Tensor maps of n ranks' attention operand buffers (K = columns [Dp, 2 Dp) of qk [T, 2 Dp],
// V^T [Dp, ldv]) written to dst_device as [2 n] CUtensorMap (K, V^T per rank).  Setup-time
// (synchronous copy); the pointers are the ranks' persistent buffers as this GPU addresses
// them (peer-mapped symmetric memory, or local buffers of virtual ranks).
int ps_kv_peer_maps(void* dst_device, int n, const uint64_t* qk_ptrs, const int32_t* T, const uint64_t* vt_ptrs,
                    const int32_t* ldv, int Dp) {
  if (n < 1 || n > 64) return set_error(PS_ERR_INPUT, "kv_peer_maps: n=%d", n);
  if (Dp % 64 || Dp < 64 || Dp > 320) return set_error(PS_ERR_INPUT, "kv_peer_maps: Dp %d unsupported", Dp);
  std::vector<CUtensorMap> maps(2 * (size_t)n);
  for (int i = 0; i < n; ++i) {
    int rc = make_tmap_2d(&maps[2 * i], (const __nv_bfloat16*)qk_ptrs[i] + Dp, T[i], Dp, 2 * (uint64_t)Dp, 128);
    if (!rc) rc = make_tmap_2d(&maps[2 * i + 1], (const void*)vt_ptrs[i], Dp, T[i], ldv[i], 64);
    if (rc) return rc;
  }
  if (cudaMemcpy(dst_device, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice) != cudaSuccess)
    return set_error(PS_ERR_CUDA, "kv_peer_maps: copy failed");
  return PS_OK;
}

// Attention whose keys of split images are read from peer GPUs' K / V^T buffers
// (kb_src / kb_row per local 128-token key block, maps from ps_kv_peer_maps); split-KV
// arrays may be NULL (whole key range per tile, direct output).
int ps_attention_peer(void* stream, const void* qk, const void* vt, int ldv, int T, int Dp, int D,
                      const int32_t* img_tok0, const int32_t* tile_q0, const int32_t* tile_img,
                      const int32_t* tile_kb0, const int32_t* tile_nkb, const int32_t* tile_slot, int n_tiles,
                      float* part_o, float* part_ml, const int32_t* kb_src, const int32_t* kb_row,
                      const void* peer_maps, void* out) {
  if (Dp % 64 || Dp < 64 || Dp > 320) return set_error(PS_ERR_INPUT, "attention: Dp %d unsupported", Dp);
  if (D < 1 || D > Dp) return set_error(PS_ERR_INPUT, "attention: bad D");
  if (!kb_src || !kb_row || !peer_maps) return set_error(PS_ERR_INPUT, "attention_peer: null peer tables");
  if (n_tiles < 1) return PS_OK;
  CUtensorMap tq, tk, tv;
  int rc = make_tmap_2d(&tq, qk, T, Dp, 2 * (uint64_t)Dp, 128);
  if (!rc) rc = make_tmap_2d(&tk, (const __nv_bfloat16*)qk + Dp, T, Dp, 2 * (uint64_t)Dp, 128);
  if (!rc) rc = make_tmap_2d(&tv, vt, Dp, T, ldv, 64);
  if (rc) return rc;
  AttnParams p{};
  p.T_total = T;
  p.Dp = Dp;
  p.n_tiles = n_tiles;
  p.tile_q0 = tile_q0;
  p.tile_img = tile_img;
  p.img_tok0 = img_tok0;
  p.scale_log2 = 1.4426950408889634f / sqrtf((float)D);
  p.out = (__nv_bfloat16*)out;
  p.dbg = g_attn_dbg;
  p.tile_kb0 = tile_kb0;
  p.tile_nkb = tile_nkb;
  p.tile_slot = tile_slot;
  p.part_o = part_o;
  p.part_ml = part_ml;
  p.kb_src = kb_src;
  p.kb_row = kb_row;
  p.peer_maps = (const CUtensorMap*)peer_maps;
  return attention_launch(tq, tk, tv, p, Dp, (cudaStream_t)stream);
}
}  // extern "C"

extern "C" {
// Fused feed-forward + residual (ffused.cu): out NCHW = W2 gelu(W1 x + b1) + b2 + resid.
int ps_feed_forward(void* stream, const void* x, int M, int Cp, const void* w1, const float* b1, const void* w2,
                    const float* b2, int Hp, int c_real, int ps, const void* resid, void* out, const int32_t* m_map,
                    int m_count, const int32_t* m_count_dev) {
  if (!x || !w1 || !w2 || !b1 || !b2 || !out) return set_error(PS_ERR_INPUT, "feed_forward: null pointer");
  if (Cp % 64 || Cp < 128 || Cp > 320) return set_error(PS_ERR_INPUT, "feed_forward: Cp %d unsupported", Cp);
  if (Hp % 128 || Hp < 128) return set_error(PS_ERR_INPUT, "feed_forward: hidden %d must be a multiple of 128", Hp);
  const int hw = ps * ps;
  if (hw % 128 || M % 128) return set_error(PS_ERR_INPUT, "feed_forward: ps*ps and M must be multiples of 128");
  if (c_real < 1 || c_real > Cp) return set_error(PS_ERR_INPUT, "feed_forward: bad c_real");
  CUtensorMap tx, t1, t2;
  int rc = make_tmap_2d(&tx, x, M, Cp, Cp, 128);
  if (!rc) rc = make_tmap_2d(&t1, w1, Hp, Cp, Cp, 64);
  if (!rc) rc = make_tmap_2d(&t2, w2, Cp, Hp, Hp, Cp / 4);
  if (rc) return rc;
  FfParams p{};
  p.M = M;
  p.m_map = m_map;
  p.m_count = m_map ? m_count : 0;
  p.m_count_dev = m_map ? m_count_dev : nullptr;
  p.hp = Hp;
  p.b1 = b1;
  p.b2 = b2;
  p.c_real = c_real;
  p.hw = hw;
  p.resid = (const __nv_bfloat16*)resid;
  p.out = (__nv_bfloat16*)out;
  p.dbg = g_ff_dbg;
  static const int ff_ts = getenv("PS_FF_TS") ? atoi(getenv("PS_FF_TS")) : 1;  // GELU(H) through TMEM (TS MMA) vs shared memory
  p.ts = ff_ts;
  static const int ff_tail = getenv("PS_FF_TAIL_SPLIT") ? atoi(getenv("PS_FF_TAIL_SPLIT")) : 1;
  p.tail_split = ff_tail;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return ff_launch(tx, t1, t2, p, Cp, sms, (cudaStream_t)stream);
}
}  // extern "C"
