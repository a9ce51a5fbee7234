// Patch-level cache reuse test (K8) and cache data movement (K9).
//
// Reference: BlockCache (cache.py:73-181).  predict_reuse marks a patch
// reusable when an entry exists, mse(x, input_snapshot) < sigma (strict) and the
// reuse streak is below max_streak (cache.py:107-122, 87-88).  mse is
// float(np.mean((a-b)**2)) (cache.py:54-55): numpy float64 pairwise summation
// over the C-contiguous (C, ps, ps) patch.  The kernels below reproduce that
// summation tree exactly (plan from ps_pairwise_plan, fp64 with explicit
// round-to-nearest ops, no FMA contraction), so masks are bit-exact given the
// same bf16 inputs.
//
// Device store ("slab"): per block, snapshots live at slot = base[request] +
// ordinal; exists/streak are per-slot arrays.  The engine's per-block sequence
// (engine.py:137-142) is fused into substitute (before the block) and finish
// (after it).
#include <stdlib.h>

#include "common.cuh"
#include "ps_internal.h"

namespace ps {

constexpr int LEAVES_PER_CTA = 128;

__device__ __forceinline__ bool entry_live(int slot, const uint8_t* exists, const int32_t* streak, int max_streak) {
  return slot >= 0 && exists[slot] && streak[slot] < max_streak;
}

// numpy pairwise_sum leaf (n <= 128) over squared differences of bf16 pairs.
__device__ __forceinline__ double leaf_sum(const __nv_bfloat16* a, const __nv_bfloat16* b, int n) {
  auto sq = [&](int i) {
    const double d = __dsub_rn((double)__bfloat162float(a[i]), (double)__bfloat162float(b[i]));
    return __dmul_rn(d, d);
  };
  if (n < 8) {
    double res = -0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, sq(i));
    return res;
  }
  // 8 strided accumulators: element i goes to r[i % 8]; 16-byte smem loads deliver exactly one
  // element per accumulator (leaf starts are multiples of 8 in numpy's tree)
  auto sq8 = [&](int i, double* d8) {
    const uint4 ua = *reinterpret_cast<const uint4*>(a + i);
    const uint4 ub = *reinterpret_cast<const uint4*>(b + i);
    const __nv_bfloat162* ha = reinterpret_cast<const __nv_bfloat162*>(&ua);
    const __nv_bfloat162* hb = reinterpret_cast<const __nv_bfloat162*>(&ub);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double d0 = __dsub_rn((double)__low2float(ha[k]), (double)__low2float(hb[k]));
      const double d1 = __dsub_rn((double)__high2float(ha[k]), (double)__high2float(hb[k]));
      d8[2 * k] = __dmul_rn(d0, d0);
      d8[2 * k + 1] = __dmul_rn(d1, d1);
    }
  };
  double r[8];
  sq8(0, r);
  int i = 8;
  const int stop = n - (n % 8);
  for (; i < stop; i += 8) {
    double d8[8];
    sq8(i, d8);
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], d8[j]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, sq(i));
  return res;
}

// grid (P, ceil(L / 128)): leaf sums of patch p into scratch[p, 0:L].
__global__ void __launch_bounds__(LEAVES_PER_CTA) mse_leaf_kernel(
    const __nv_bfloat16* __restrict__ x, int64_t n, const int32_t* __restrict__ slots,
    const __nv_bfloat16* __restrict__ snap, const uint8_t* __restrict__ exists, const int32_t* __restrict__ streak,
    int max_streak, const int32_t* __restrict__ leaves, int L, int stride_nodes, double* __restrict__ scratch) {
  pdl_wait();
  extern __shared__ __align__(16) __nv_bfloat16 stage[];
  const int p = blockIdx.x;
  const int slot = slots[p];
  if (!entry_live(slot, exists, streak, max_streak)) return;
  const int l0 = blockIdx.y * LEAVES_PER_CTA;
  const int l1 = min(L, l0 + LEAVES_PER_CTA);
  const int64_t e0 = leaves[2 * l0];
  const int64_t e1 = (int64_t)leaves[2 * (l1 - 1)] + leaves[2 * (l1 - 1) + 1];
  const __nv_bfloat16* xa = x + (int64_t)p * n;
  const __nv_bfloat16* xb = snap + (int64_t)slot * n;
  // stage [e0, e1) of both operands (16B vectors when aligned)
  const int64_t v0 = e0 & ~int64_t(7), v1 = (e1 + 7) & ~int64_t(7);
  __nv_bfloat16* sa = stage;
  __nv_bfloat16* sb = stage + (v1 - v0);
  const bool vec = (n % 8 == 0) && v1 <= n;
  __shared__ __align__(8) uint64_t bar;
  if (vec) {
    // two bulk copies (TMA engine, no register staging): the whole span is in flight at once
    const uint32_t bytes = (uint32_t)((v1 - v0) * 2);
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      fence_mbar_init();
      mbar_arrive_expect_tx(&bar, 2 * bytes);
      bulk_load(sa, xa + v0, bytes, &bar);
      bulk_load(sb, xb + v0, bytes, &bar);
    }
    __syncthreads();
    mbar_wait(&bar, 0);
  } else {
    for (int64_t i = e0 + threadIdx.x; i < e1; i += blockDim.x) {
      sa[i - v0] = xa[i];
      sb[i - v0] = xb[i];
    }
  }
  __syncthreads();
  const int l = l0 + threadIdx.x;
  if (l < l1) {
    const int64_t s = leaves[2 * l];
    const int len = leaves[2 * l + 1];
    scratch[(int64_t)p * stride_nodes + l] = leaf_sum(sa + (s - v0), sb + (s - v0), len);
  }
}

// grid P: evaluate internal nodes level by level, then the mask.
__global__ void __launch_bounds__(256) mse_combine_kernel(
    int64_t n, const int32_t* __restrict__ slots, const uint8_t* __restrict__ exists,
    const int32_t* __restrict__ streak, int max_streak, double sigma, int L, const int32_t* __restrict__ nodes,
    int I, const int32_t* __restrict__ level_off, int H, int stride_nodes, double* __restrict__ scratch,
    uint8_t* __restrict__ mask, int64_t* __restrict__ counters, int smem_nodes) {
  pdl_wait();
  const int p = blockIdx.x;
  const int slot = slots[p];
  const bool live = entry_live(slot, exists, streak, max_streak);
  double* v = scratch + (int64_t)p * stride_nodes;
  extern __shared__ double sv[];  // leaf sums + internal nodes when they fit (else in place in scratch)
  __shared__ double root_s;
  const bool in_smem = smem_nodes >= L + I;
  if (live) {
    double* w = v;
    if (in_smem) {
      // the leaf sums (L2-resident, written by mse_leaf_kernel): 8 independent loads in
      // flight per thread instead of one L2 round trip per loop trip
      for (int base = 0; base < L; base += 8 * blockDim.x) {
        double t[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int i = base + k * blockDim.x + threadIdx.x;
          t[k] = i < L ? __ldcg(v + i) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int i = base + k * blockDim.x + threadIdx.x;
          if (i < L) sv[i] = t[k];
        }
      }
      __syncthreads();
      w = sv;
    }
    if (in_smem && smem_nodes >= L + I + I) {
      // node index pairs staged next to the values (int2 per node): the levels then touch
      // shared memory only -- no L2 round trip per level for the tree structure
      int2* sn = reinterpret_cast<int2*>(sv + L + I);
      for (int base = 0; base < I; base += 8 * blockDim.x) {
        int2 t[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int i = base + k * blockDim.x + threadIdx.x;
          t[k] = i < I ? __ldg(reinterpret_cast<const int2*>(nodes) + i) : make_int2(0, 0);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int i = base + k * blockDim.x + threadIdx.x;
          if (i < I) sn[i] = t[k];
        }
      }
      __syncthreads();
      for (int h = 0; h < H; ++h) {
        const int e = __ldg(level_off + h + 1);
        for (int i = __ldg(level_off + h) + threadIdx.x; i < e; i += blockDim.x) {
          const int2 c = sn[i];
          w[L + i] = __dadd_rn(w[c.x], w[c.y]);
        }
        __syncthreads();
      }
    } else {
      for (int h = 0; h < H; ++h) {
        for (int i = level_off[h] + threadIdx.x; i < level_off[h + 1]; i += blockDim.x)
          w[L + i] = __dadd_rn(w[nodes[2 * i]], w[nodes[2 * i + 1]]);
        __syncthreads();
      }
    }
    if (threadIdx.x == 0) {
      root_s = I > 0 ? w[L + I - 1] : w[0];
      if (in_smem && I > 0) v[L + I - 1] = root_s;  // the root stays readable in scratch (ps.mse)
    }
  }
  if (threadIdx.x == 0) {
    bool m = false;
    if (live) {
      const double root = root_s;
      const double mse = __ddiv_rn(__dadd_rn(0.0, root), (double)n);
      m = mse < sigma;
    }
    mask[p] = m ? 1 : 0;
    if (counters) atomicAdd(reinterpret_cast<unsigned long long*>(counters + (m ? 0 : 1)), 1ull);
  }
}

// single CTA: ascending active (mask == 0) and reused (mask == 1) lists.
__global__ void __launch_bounds__(1024) compact_kernel(const uint8_t* __restrict__ mask, int P,
                                                       int32_t* __restrict__ active, int32_t* __restrict__ n_active,
                                                       int32_t* __restrict__ reused, int32_t* __restrict__ n_reused) {
  __shared__ int warp_tot[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int base = 0; base < P; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const int a = (i < P && mask[i] == 0) ? 1 : 0;
    int incl = a;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    if (w == 0) {
      int t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
      int s = t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += u;
      }
      warp_tot[lane] = s - t;  // exclusive
    }
    __syncthreads();
    const int pos = carry + warp_tot[w] + incl - a;
    if (i < P) {
      if (a) active[pos] = i;
      else if (reused) reused[i - pos] = i;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = pos + a;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *n_active = carry;
    if (n_reused) *n_reused = P - carry;
  }
}

enum PatchOp { OP_GATHER, OP_FILL, OP_UPDATE, OP_SUBST, OP_FINISH, OP_SELECT };

struct PatchOpArgs {
  const uint8_t* mask;
  const int32_t* slots;
  uint8_t* exists;
  int32_t* streak;
  int64_t n;
  const __nv_bfloat16* x;  // fresh input / select a
  __nv_bfloat16* y;        // fresh output (finish: in/out) / select b
  __nv_bfloat16* snap_in;
  __nv_bfloat16* snap_out;
  __nv_bfloat16* o1;  // gather ins / fill out / subst x_sub / select out
  __nv_bfloat16* o2;  // gather outs
  int32_t* err;
  int64_t* counters;
  const int32_t* plist;  // optional patch list (grid.x walks it) ...
  const int32_t* n_dev;  // ... with its DEVICE length (grid.x is an upper bound)
};

__device__ __forceinline__ void copy_range(__nv_bfloat16* dst, const __nv_bfloat16* src, int64_t n, bool vec) {
  if (vec) {
    const int64_t nv = n / 8;
    for (int64_t i = blockIdx.y * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.y * blockDim.x)
      reinterpret_cast<uint4*>(dst)[i] = __ldg(reinterpret_cast<const uint4*>(src) + i);
  } else {
    for (int64_t i = blockIdx.y * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.y * blockDim.x)
      dst[i] = src[i];
  }
}
__device__ __forceinline__ void zero_range(__nv_bfloat16* dst, int64_t n, bool vec) {
  if (vec) {
    for (int64_t i = blockIdx.y * (int64_t)blockDim.x + threadIdx.x; i < n / 8; i += (int64_t)gridDim.y * blockDim.x)
      reinterpret_cast<uint4*>(dst)[i] = make_uint4(0, 0, 0, 0);
  } else {
    for (int64_t i = blockIdx.y * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.y * blockDim.x)
      dst[i] = __float2bfloat16_rn(0.f);
  }
}

template <int OP>
__global__ void __launch_bounds__(256) patch_op_kernel(PatchOpArgs a) {
  pdl_wait();
  if (a.n_dev != nullptr && (int)blockIdx.x >= *a.n_dev) return;
  const int p = a.plist ? a.plist[blockIdx.x] : (int)blockIdx.x;
  const bool m = a.mask[p] != 0;
  const int slot = a.slots ? a.slots[p] : -1;
  const int64_t n = a.n;
  const bool vec = (n % 8) == 0;
  const bool lead = blockIdx.y == 0 && threadIdx.x == 0;
  const int64_t po = (int64_t)p * n, so = (int64_t)slot * n;
  if constexpr (OP == OP_SELECT) {
    copy_range(a.o1 + po, m ? a.x + po : a.y + po, n, vec);
    return;
  }
  if constexpr (OP == OP_SUBST) {
    if (m && slot >= 0) copy_range(a.o1 + po, a.snap_in + so, n, vec);
    else copy_range(a.o1 + po, a.x + po, n, vec);
    return;
  }
  const bool have = slot >= 0 && a.exists[slot];
  if constexpr (OP == OP_GATHER) {
    if (m && !have) {
      if (lead) atomicExch(a.err, 1);
      return;
    }
    if (m) {
      copy_range(a.o1 + po, a.snap_in + so, n, vec);
      copy_range(a.o2 + po, a.snap_out + so, n, vec);
    } else {
      zero_range(a.o1 + po, n, vec);
      zero_range(a.o2 + po, n, vec);
    }
    return;
  }
  if constexpr (OP == OP_FILL) {
    if (!m) return;
    if (!have) {
      if (lead) atomicExch(a.err, 1);
      return;
    }
    if (a.o1) copy_range(a.o1 + po, a.snap_out + so, n, vec);
    if (lead) a.streak[slot] += 1;
    return;
  }
  if constexpr (OP == OP_UPDATE || OP == OP_FINISH) {
    if (m) {
      if constexpr (OP == OP_FINISH) {
        copy_range(a.y + po, a.snap_out + so, n, vec);
        if (lead) a.streak[slot] += 1;
      }
      return;
    }
    if (slot < 0) return;
    copy_range(a.snap_in + so, a.x + po, n, vec);
    copy_range(a.snap_out + so, a.y + po, n, vec);
    if (lead) {
      if (a.counters) atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + (have ? 0 : 1)), 1ull);
      a.streak[slot] = 0;
      a.exists[slot] = 1;
    }
  }
}

__global__ void evict_kernel(uint8_t* exists, int32_t* streak, const int32_t* slots, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    exists[slots[i]] = 0;
    streak[slots[i]] = 0;
  }
}

template <int OP>
static int launch_op(cudaStream_t st, int P, int64_t n, const PatchOpArgs& a, const char* name) {
  if (P == 0) return PS_OK;
  const int64_t vecs = (n % 8 == 0) ? n / 8 : n;
  int chunks = (int)((vecs + 255) / 256);
  if (chunks > 16) chunks = 16;
  if (chunks < 1) chunks = 1;
  launch_pdl(patch_op_kernel<OP>, dim3(P, chunks), dim3(256), 0, st, a);
  count_launch();
  return check_launch(name);
}

}  // namespace ps

using namespace ps;

namespace ps {
// Block-wide exclusive scan of one 0/1 flag per thread (1024 threads); returns the
// thread's position, *total gets the chunk's count.
__device__ __forceinline__ int block_excl_scan(int a, int* warp_tot, int* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = a;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  __syncthreads();
  if (lane == 31) warp_tot[w] = incl;
  __syncthreads();
  if (w == 0) {
    const int t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
    int s2 = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, s2, o);
      if (lane >= o) s2 += u;
    }
    warp_tot[lane] = s2 - t;
    if (lane == 31) *total = s2;
  }
  __syncthreads();
  return warp_tot[w] + incl - a;
}

// Device-side lists of a compacted block (run_block_active without a host round trip):
// GEMM row tiles of the active patches (mask == 0) and of every patch of an image with an
// active patch ("live"), attention query tiles of the same two sets over the attention patch
// order `order` (longest images first), and the live patches.  counts: [rows_act, rows_live,
// attn_act, attn_live, active patches, live patches].  Single CTA of 1024 threads; live: int scratch [R].
__global__ void __launch_bounds__(1024) compact_lists_kernel(
    const uint8_t* __restrict__ mask, int P, const int32_t* __restrict__ ri, int R, const int32_t* __restrict__ order,
    int tpp, int qpp, int tq, int hw, int32_t* live, int32_t* __restrict__ rows_act, int32_t* __restrict__ rows_live,
    int32_t* __restrict__ live_patches,
    int32_t* __restrict__ aq_act, int32_t* __restrict__ ai_act, int32_t* __restrict__ aq_live,
    int32_t* __restrict__ ai_live, int32_t* __restrict__ counts) {
  pdl_wait();
  __shared__ int warp_tot[32];
  __shared__ int total;
  for (int r = threadIdx.x; r < R; r += blockDim.x) live[r] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < P; i += blockDim.x)
    if (mask[i] == 0) live[ri[i]] = 1;
  __threadfence_block();
  __syncthreads();
  int c[4] = {0, 0, 0, 0};
  for (int base = 0; base < P; base += blockDim.x) {
    const int i = base + threadIdx.x;
    const bool in = i < P;
    const int po = in ? order[i] : 0;
    const int f[4] = {in && mask[i] == 0, in && live[ri[i]] != 0, in && mask[po] == 0, in && live[ri[po]] != 0};
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int pos = c[l] + block_excl_scan(f[l], warp_tot, &total);
      if (f[l]) {
        if (l < 2) {
          int32_t* dst = l == 0 ? rows_act : rows_live;
          for (int j = 0; j < tpp; ++j) dst[pos * tpp + j] = i * tpp + j;
          if (l == 1) live_patches[pos] = i;
        } else {
          int32_t* dq = l == 2 ? aq_act : aq_live;
          int32_t* di = l == 2 ? ai_act : ai_live;
          for (int j = 0; j < qpp; ++j) {
            dq[pos * qpp + j] = po * hw + tq * j;
            di[pos * qpp + j] = ri[po];
          }
        }
      }
      c[l] += total;
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    counts[0] = c[0] * tpp;
    counts[1] = c[1] * tpp;
    counts[2] = c[2] * qpp;
    counts[3] = c[3] * qpp;
    counts[4] = c[0];
    counts[5] = c[1];
  }
}

}  // namespace ps

extern "C" {

int ps_cache_predict(void* stream, const void* x, int P, int64_t n, const int32_t* slots, const void* snap_in,
                     const uint8_t* exists, const int32_t* streak, double sigma, int max_streak,
                     const int32_t* leaves, int n_leaves, const int32_t* nodes, int n_internal,
                     const int32_t* level_off, int n_levels, double* scratch, uint8_t* mask, int64_t* counters) {
  if (P == 0) return PS_OK;
  if (n < 1 || n_leaves < 1) return set_error(PS_ERR_INPUT, "cache_predict: empty patches");
  cudaStream_t st = (cudaStream_t)stream;
  const int stride = n_leaves + n_internal;
  // shared staging of two operands: the widest span of LEAVES_PER_CTA consecutive leaves of
  // this n's tree (+16 elements of vector alignment slack); smaller staging -> more CTAs per SM
  const int smem = 2 * (int)(pairwise_max_span(n, LEAVES_PER_CTA) + 16) * 2;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(mse_leaf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         2 * (LEAVES_PER_CTA * 128 + 16) * 2);
    attr = true;
  }
  launch_pdl(mse_leaf_kernel, dim3(P, (n_leaves + LEAVES_PER_CTA - 1) / LEAVES_PER_CTA), dim3(LEAVES_PER_CTA),
             (size_t)smem, st, (const __nv_bfloat16*)x, n, slots, (const __nv_bfloat16*)snap_in, exists, streak,
             max_streak, leaves, n_leaves, stride, scratch);
  count_launch();
  int rc = check_launch("mse_leaf");
  if (rc) return rc;
  // the tree in shared memory when it fits (levels then cost smem latency, not L2 round trips)
  const int nodes_all = n_leaves + n_internal;
  // values (8 B per node) + node index pairs (8 B per internal node) in shared memory: 14 -> 9
  // us per launch at config 2 (the in-place L2 levels, PS_MSE_L2_COMBINE=1, wait for an L2
  // round trip per level)
  const int smem_need = nodes_all * 8 + n_internal * 8;
  const int smem_c = (!getenv("PS_MSE_L2_COMBINE") && smem_need <= 200 * 1024) ? smem_need : 0;
  static bool attr_c = false;
  if (!attr_c) {
    cudaFuncSetAttribute(mse_combine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_c = true;
  }
  launch_pdl(mse_combine_kernel, dim3(P), dim3(256), (size_t)smem_c, st, n, slots, exists, streak, max_streak, sigma,
             n_leaves, nodes, n_internal, level_off, n_levels, stride, scratch, mask, counters, smem_c / 8);
  count_launch();
  return check_launch("mse_combine");
}

int ps_compact_lists(void* stream, const uint8_t* mask, int P, const int32_t* request_index, int R,
                     const int32_t* order, int tpp, int qpp, int tq, int hw, int32_t* live_scratch, int32_t* rows_act,
                     int32_t* rows_live, int32_t* live_patches, int32_t* attn_q0_act, int32_t* attn_img_act,
                     int32_t* attn_q0_live, int32_t* attn_img_live, int32_t* counts) {
  if (P < 0 || R < 1 || tpp < 1 || qpp < 1) return set_error(PS_ERR_INPUT, "compact_lists: bad geometry");
  launch_pdl(ps::compact_lists_kernel, dim3(1), dim3(1024), 0, (cudaStream_t)stream, mask, P, request_index, R, order,
             tpp, qpp, tq, hw, live_scratch, rows_act, rows_live, live_patches, attn_q0_act, attn_img_act,
             attn_q0_live, attn_img_live, counts);
  count_launch();
  return check_launch("compact_lists");
}

int ps_compact(void* stream, const uint8_t* mask, int P, int32_t* active, int32_t* n_active, int32_t* reused,
               int32_t* n_reused) {
  compact_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(mask, P, active, n_active, reused, n_reused);
  count_launch();
  return check_launch("compact");
}

int ps_cache_gather(void* stream, const uint8_t* mask, const int32_t* slots, const uint8_t* exists, int P, int64_t n,
                    const void* snap_in, const void* snap_out, void* ins, void* outs, int32_t* error_flag) {
  PatchOpArgs a{};
  a.mask = mask; a.slots = slots; a.exists = const_cast<uint8_t*>(exists); a.n = n;
  a.snap_in = (__nv_bfloat16*)snap_in; a.snap_out = (__nv_bfloat16*)snap_out;
  a.o1 = (__nv_bfloat16*)ins; a.o2 = (__nv_bfloat16*)outs; a.err = error_flag;
  return launch_op<OP_GATHER>((cudaStream_t)stream, P, n, a, "cache_gather");
}

int ps_cache_fill(void* stream, const uint8_t* mask, const int32_t* slots, const uint8_t* exists, int32_t* streak,
                  int P, int64_t n, const void* snap_out, void* out, int32_t* error_flag) {
  PatchOpArgs a{};
  a.mask = mask; a.slots = slots; a.exists = const_cast<uint8_t*>(exists); a.streak = streak; a.n = n;
  a.snap_out = (__nv_bfloat16*)snap_out; a.o1 = (__nv_bfloat16*)out; a.err = error_flag;
  return launch_op<OP_FILL>((cudaStream_t)stream, P, n, a, "cache_fill");
}

int ps_cache_update(void* stream, const uint8_t* mask, const int32_t* slots, uint8_t* exists, int32_t* streak, int P,
                    int64_t n, const void* x, const void* y, void* snap_in, void* snap_out, int64_t* counters) {
  PatchOpArgs a{};
  a.mask = mask; a.slots = slots; a.exists = exists; a.streak = streak; a.n = n;
  a.x = (const __nv_bfloat16*)x; a.y = (__nv_bfloat16*)y;
  a.snap_in = (__nv_bfloat16*)snap_in; a.snap_out = (__nv_bfloat16*)snap_out; a.counters = counters;
  return launch_op<OP_UPDATE>((cudaStream_t)stream, P, n, a, "cache_update");
}

int ps_cache_evict(void* stream, uint8_t* exists, int32_t* streak, const int32_t* slots, int n_slots) {
  if (n_slots == 0) return PS_OK;
  evict_kernel<<<(n_slots + 255) / 256, 256, 0, (cudaStream_t)stream>>>(exists, streak, slots, n_slots);
  count_launch();
  return check_launch("cache_evict");
}

int ps_cache_substitute(void* stream, const uint8_t* mask, const int32_t* slots, int P, int64_t n, const void* x,
                        const void* snap_in, void* x_sub, const int32_t* patches, int n_list, const int32_t* n_dev) {
  PatchOpArgs a{};
  a.mask = mask; a.slots = slots; a.n = n; a.x = (const __nv_bfloat16*)x;
  a.snap_in = (__nv_bfloat16*)snap_in; a.o1 = (__nv_bfloat16*)x_sub;
  a.plist = patches; a.n_dev = patches ? n_dev : nullptr;
  return launch_op<OP_SUBST>((cudaStream_t)stream, patches ? n_list : P, n, a, "cache_substitute");
}

int ps_cache_finish(void* stream, const uint8_t* mask, const int32_t* slots, uint8_t* exists, int32_t* streak, int P,
                    int64_t n, const void* x, void* y, void* snap_in, void* snap_out, int64_t* counters) {
  PatchOpArgs a{};
  a.mask = mask; a.slots = slots; a.exists = exists; a.streak = streak; a.n = n;
  a.x = (const __nv_bfloat16*)x; a.y = (__nv_bfloat16*)y;
  a.snap_in = (__nv_bfloat16*)snap_in; a.snap_out = (__nv_bfloat16*)snap_out; a.counters = counters;
  return launch_op<OP_FINISH>((cudaStream_t)stream, P, n, a, "cache_finish");
}

int ps_select_patches(void* stream, const uint8_t* mask, int P, int64_t n, const void* a_, const void* b_,
                      void* out) {
  PatchOpArgs a{};
  a.mask = mask; a.n = n; a.x = (const __nv_bfloat16*)a_; a.y = (__nv_bfloat16*)b_; a.o1 = (__nv_bfloat16*)out;
  return launch_op<OP_SELECT>((cudaStream_t)stream, P, n, a, "select_patches");
}

}  // extern "C"
