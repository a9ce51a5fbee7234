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

__device__ __forceinline__ bool entry_live(int slot, const uint8_t* exists, const int32_t* streak, int max_streak) {
  return slot >= 0 && exists[slot] && streak[slot] < max_streak;
}

__device__ __forceinline__ double to_d(__nv_bfloat16 v) { return (double)__bfloat162float(v); }
__device__ __forceinline__ double to_d(float v) { return (double)v; }
__device__ __forceinline__ double to_d(double v) { return v; }

// Leaves per CTA of the reuse test (one leaf per thread): both operands' spans of LPC
// consecutive leaves (<= 128 elements each) are staged in shared memory.
template <typename T>
struct MseCfg {
  static constexpr int LPC = sizeof(T) == 2 ? 128 : (sizeof(T) == 4 ? 64 : 32);
  static constexpr int EPV = 16 / (int)sizeof(T);  // elements per 16-byte vector
};

// numpy pairwise_sum leaf (n <= 128, numpy/_core/src/umath/loops_utils.h.src) over the
// squared differences (a - b)^2, fp64 with explicit round-to-nearest ops (no FMA contraction):
// n < 8 sequential from -0.0; else 8 strided accumulators r[i % 8], combined
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the n % 8 tail.
template <typename T>
__device__ __forceinline__ double leaf_sum(const T* a, const T* b, int n) {
  auto sq = [&](int i) {
    const double d = __dsub_rn(to_d(a[i]), to_d(b[i]));
    return __dmul_rn(d, d);
  };
  if (n < 8) {
    double res = -0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, sq(i));
    return res;
  }
  double r[8];
  if constexpr (sizeof(T) == 2) {
    // bf16: one 16-byte smem load per operand delivers exactly one element per accumulator
    // (leaf starts are multiples of 8 in numpy's tree)
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
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = sq(j);
    int i = 8;
    const int stop = n - (n % 8);
    for (; i < stop; i += 8) {
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], sq(i + j));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, sq(i));
    return res;
  }
}

// Internal nodes of patch p's tree, level by level (children from `nodes`, ids < L are
// leaves), over the values w[0 .. L+I) -- in shared memory or in place in scratch -- then the
// mask (mse < sigma, strict) and the reuse / fresh counters.  Called by the CTA that finished
// the patch's last leaves (all CTA threads).
__device__ __forceinline__ void mse_tree_and_mask(int p, double* w, bool w_in_smem, double* v_global, int64_t n, int L,
                                                  const int32_t* __restrict__ nodes, int I,
                                                  const int32_t* __restrict__ level_off, int H, double sigma,
                                                  uint8_t* __restrict__ mask, int64_t* __restrict__ counters) {
  for (int h = 0; h < H; ++h) {
    const int e = __ldg(level_off + h + 1);
    for (int i = __ldg(level_off + h) + threadIdx.x; i < e; i += blockDim.x) {
      const int2 c = __ldg(reinterpret_cast<const int2*>(nodes) + i);
      w[L + i] = __dadd_rn(w[c.x], w[c.y]);
    }
    if (!w_in_smem) __threadfence_block();
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double root = I > 0 ? w[L + I - 1] : w[0];
    if (w_in_smem) v_global[I > 0 ? L + I - 1 : 0] = root;  // the root stays readable in scratch (ps.mse)
    const double mse = __ddiv_rn(__dadd_rn(0.0, root), (double)n);
    const bool m = mse < sigma;
    mask[p] = m ? 1 : 0;
    if (counters) atomicAdd(reinterpret_cast<unsigned long long*>(counters + (m ? 0 : 1)), 1ull);
  }
}

// In-order pairwise reduction of n (a power of two) doubles in shared memory, ping-ponging
// between buf and tmp: level by level w[i] = w[2i] + w[2i+1] -- numpy's tree when it is
// perfect.  Returns the root (all CTA threads).
__device__ __forceinline__ double smem_pairwise(double* buf, double* tmp, int n) {
  double* src = buf;
  double* dst = tmp;
  for (int s = n >> 1; s >= 1; s >>= 1) {
    for (int i = threadIdx.x; i < s; i += blockDim.x) dst[i] = __dadd_rn(src[2 * i], src[2 * i + 1]);
    __syncthreads();
    double* t = src;
    src = dst;
    dst = t;
  }
  return src[0];
}

// grid (ceil(L / LPC), P), LPC threads: the reuse test of patch p in one kernel.  Every CTA
// sums its LPC leaves (both operands' spans staged in shared memory by two bulk copies);
//  * perfect tree (depth >= 0: numpy's tree over n is a perfect binary tree, e.g. n = C ps^2
//    with C = 4 or 320 and ps a power of two): the CTA reduces its leaves pairwise to its
//    subtree root, and the patch's last CTA (per-patch ticket) reduces the CTA roots the
//    same way -- the exact numpy tree, a few levels of shared-memory adds per CTA;
//  * otherwise: the leaf sums go to scratch and the last CTA walks the plan's levels.
// Then the mask (mse < sigma, strict) and the counters.  Patches with no live entry (absent /
// streak exhausted) skip the MSE as the reference's short-circuit does (cache.py:87-88, 116-119).
template <typename T>
__global__ void __launch_bounds__(MseCfg<T>::LPC) mse_fused_kernel(
    const T* __restrict__ x, int64_t n, const int32_t* __restrict__ slots, const T* __restrict__ snap,
    const uint8_t* __restrict__ exists, const int32_t* __restrict__ streak, int max_streak, double sigma,
    const int32_t* __restrict__ leaves, int L, const int32_t* __restrict__ nodes, int I,
    const int32_t* __restrict__ level_off, int H, double* __restrict__ scratch, int* __restrict__ tickets,
    uint8_t* __restrict__ mask, int64_t* __restrict__ counters, int tree_in_smem, int perfect) {
  constexpr int LPC = MseCfg<T>::LPC, EPV = MseCfg<T>::EPV;
  pdl_wait();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[2][LPC];
  const int p = blockIdx.y;
  const int slot = slots[p];
  if (!entry_live(slot, exists, streak, max_streak)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      mask[p] = 0;
      if (counters) atomicAdd(reinterpret_cast<unsigned long long*>(counters + 1), 1ull);
    }
    return;
  }
  const int stride = L + I;
  double* v = scratch + (int64_t)p * stride;
  const int l0 = blockIdx.x * LPC;
  const int l1 = min(L, l0 + LPC);
  const int64_t e0 = leaves[2 * l0];
  const int64_t e1 = (int64_t)leaves[2 * (l1 - 1)] + leaves[2 * (l1 - 1) + 1];
  const T* xa = x + (int64_t)p * n;
  const T* xb = snap + (int64_t)slot * n;
  // stage [e0, e1) of both operands (16-byte vectors when aligned)
  const int64_t v0 = e0 & ~int64_t(EPV - 1), v1 = (e1 + EPV - 1) & ~int64_t(EPV - 1);
  T* sa = reinterpret_cast<T*>(smem_raw);
  T* sb = sa + (v1 - v0);
  const bool vec = (n % EPV == 0) && v1 <= n;
  __shared__ __align__(8) uint64_t bar;
  __shared__ int last;
  if (vec) {
    const uint32_t bytes = (uint32_t)((v1 - v0) * sizeof(T));
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
  double leaf = 0.0;
  if (l < l1) {
    const int64_t st = leaves[2 * l];
    leaf = leaf_sum<T>(sa + (st - v0), sb + (st - v0), leaves[2 * l + 1]);
  }
  if (perfect) {
    red[0][threadIdx.x] = leaf;
    __syncthreads();
    const double root = smem_pairwise(red[0], red[1], l1 - l0);  // l1 - l0: a power of two
    if (threadIdx.x == 0) v[blockIdx.x] = root;                   // CTA subtree root
  } else if (l < l1) {
    v[l] = leaf;
  }
  // ticket: the patch's last CTA finishes the tree
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(tickets + p, 1) == (int)gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (perfect) {
    const int g = gridDim.x;  // a power of two
    double* b0 = reinterpret_cast<double*>(smem_raw);
    double* b1 = b0 + g;
    for (int i = threadIdx.x; i < g; i += blockDim.x) b0[i] = __ldcg(v + i);
    __syncthreads();
    const double root = smem_pairwise(b0, b1, g);
    if (threadIdx.x == 0) {
      v[I > 0 ? L + I - 1 : 0] = root;  // readable in scratch (ps.mse)
      const double mse = __ddiv_rn(__dadd_rn(0.0, root), (double)n);
      const bool m = mse < sigma;
      mask[p] = m ? 1 : 0;
      if (counters) atomicAdd(reinterpret_cast<unsigned long long*>(counters + (m ? 0 : 1)), 1ull);
      tickets[p] = 0;
    }
    return;
  }
  double* w = v;
  if (tree_in_smem) {
    // all leaf sums of the patch (L2-resident) into shared memory, the staging space reused
    w = reinterpret_cast<double*>(smem_raw);
    for (int base = 0; base < L; base += 8 * (int)blockDim.x) {
      double t[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = base + k * blockDim.x + threadIdx.x;
        t[k] = i < L ? __ldcg(v + i) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int i = base + k * blockDim.x + threadIdx.x;
        if (i < L) w[i] = t[k];
      }
    }
    __syncthreads();
  }
  mse_tree_and_mask(p, w, tree_in_smem != 0, v, n, L, nodes, I, level_off, H, sigma, mask, counters);
  if (threadIdx.x == 0) tickets[p] = 0;
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

// Pure data movement: rows are moved as bytes (n elements x esize), so one kernel serves the
// bf16 hot-path slab and the fp32 / fp64 slabs of the numpy-interface drop-in.
struct PatchOpArgs {
  const uint8_t* mask;
  const int32_t* slots;
  uint8_t* exists;
  int32_t* streak;
  int64_t nb;             // bytes per patch row
  const char* x;          // fresh input / select a
  char* y;                // fresh output (finish: in/out) / select b
  char* snap_in;
  char* snap_out;
  char* o1;  // gather ins / fill out / subst x_sub / select out
  char* o2;  // gather outs
  int32_t* err;
  int64_t* counters;
  const int32_t* plist;  // optional patch list (grid.x walks it) ...
  const int32_t* n_dev;  // ... with its DEVICE length (grid.x is an upper bound)
};

__device__ __forceinline__ void copy_range(char* dst, const char* src, int64_t nb) {
  if ((nb & 15) == 0) {
    const int64_t nv = nb / 16;
    for (int64_t i = blockIdx.y * (int64_t)blockDim.x + threadIdx.x; i < nv; i += (int64_t)gridDim.y * blockDim.x)
      reinterpret_cast<uint4*>(dst)[i] = __ldg(reinterpret_cast<const uint4*>(src) + i);
  } else {
    for (int64_t i = blockIdx.y * (int64_t)blockDim.x + threadIdx.x; i < nb; i += (int64_t)gridDim.y * blockDim.x)
      dst[i] = src[i];
  }
}
__device__ __forceinline__ void zero_range(char* dst, int64_t nb) {
  if ((nb & 15) == 0) {
    for (int64_t i = blockIdx.y * (int64_t)blockDim.x + threadIdx.x; i < nb / 16; i += (int64_t)gridDim.y * blockDim.x)
      reinterpret_cast<uint4*>(dst)[i] = make_uint4(0, 0, 0, 0);
  } else {
    for (int64_t i = blockIdx.y * (int64_t)blockDim.x + threadIdx.x; i < nb; i += (int64_t)gridDim.y * blockDim.x)
      dst[i] = 0;
  }
}

template <int OP>
__global__ void __launch_bounds__(256) patch_op_kernel(PatchOpArgs a) {
  pdl_wait();
  if (a.n_dev != nullptr && (int)blockIdx.x >= *a.n_dev) return;
  const int p = a.plist ? a.plist[blockIdx.x] : (int)blockIdx.x;
  const bool m = a.mask[p] != 0;
  const int slot = a.slots ? a.slots[p] : -1;
  const int64_t nb = a.nb;
  const bool lead = blockIdx.y == 0 && threadIdx.x == 0;
  const int64_t po = (int64_t)p * nb, so = (int64_t)slot * nb;
  if constexpr (OP == OP_SELECT) {
    copy_range(a.o1 + po, m ? a.x + po : a.y + po, nb);
    return;
  }
  if constexpr (OP == OP_SUBST) {
    if (m && slot >= 0) copy_range(a.o1 + po, a.snap_in + so, nb);
    else copy_range(a.o1 + po, a.x + po, nb);
    return;
  }
  const bool have = slot >= 0 && a.exists[slot];
  if constexpr (OP == OP_GATHER) {
    if (m && !have) {
      if (lead) atomicExch(a.err, 1);
      return;
    }
    if (m) {
      copy_range(a.o1 + po, a.snap_in + so, nb);
      copy_range(a.o2 + po, a.snap_out + so, nb);
    } else {
      zero_range(a.o1 + po, nb);
      zero_range(a.o2 + po, nb);
    }
    return;
  }
  if constexpr (OP == OP_FILL) {
    if (!m) return;
    if (!have) {
      if (lead) atomicExch(a.err, 1);
      return;
    }
    if (a.o1) copy_range(a.o1 + po, a.snap_out + so, nb);
    if (lead) a.streak[slot] += 1;
    return;
  }
  if constexpr (OP == OP_UPDATE || OP == OP_FINISH) {
    if (m) {
      if constexpr (OP == OP_FINISH) {
        copy_range(a.y + po, a.snap_out + so, nb);
        if (lead) a.streak[slot] += 1;
      }
      return;
    }
    if (slot < 0) return;
    copy_range(a.snap_in + so, a.x + po, nb);
    copy_range(a.snap_out + so, a.y + po, nb);
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

static int dtype_size(int dtype) {
  return dtype == PS_DTYPE_BF16 ? 2 : dtype == PS_DTYPE_F32 ? 4 : dtype == PS_DTYPE_F64 ? 8 : 0;
}

template <int OP>
static int launch_op(cudaStream_t st, int P, int64_t n, int dtype, PatchOpArgs& a, const char* name) {
  if (P == 0) return PS_OK;
  const int es = dtype_size(dtype);
  if (es == 0) return set_error(PS_ERR_INPUT, "%s: unsupported dtype %d", name, dtype);
  a.nb = n * es;
  const int64_t vecs = (a.nb % 16 == 0) ? a.nb / 16 : a.nb;
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

int ps_cache_predict(void* stream, const void* x, int dtype, int P, int64_t n, const int32_t* slots,
                     const void* snap_in, const uint8_t* exists, const int32_t* streak, double sigma, int max_streak,
                     const int32_t* leaves, int n_leaves, const int32_t* nodes, int n_internal,
                     const int32_t* level_off, int n_levels, double* scratch, uint8_t* mask, int64_t* counters) {
  if (P == 0) return PS_OK;
  if (n < 1 || n_leaves < 1) return set_error(PS_ERR_INPUT, "cache_predict: empty patches");
  if (P > 65535) return set_error(PS_ERR_INPUT, "cache_predict: too many patches");
  cudaStream_t st = (cudaStream_t)stream;
  const int stride = n_leaves + n_internal;
  int* tickets = reinterpret_cast<int*>(scratch + (int64_t)P * stride);
  if (cudaMemsetAsync(tickets, 0, (size_t)P * sizeof(int), st) != cudaSuccess)
    return check_launch("cache_predict tickets");
  auto run = [&](auto tag) -> int {
    using T = decltype(tag);
    constexpr int LPC = MseCfg<T>::LPC;
    // staging: the widest span of LPC consecutive leaves of this n's tree (+ vector slack), both
    // operands; the tree values (L + I doubles) reuse it when they fit the budget
    const int stage = 2 * (int)(pairwise_max_span(n, LPC) + 2 * MseCfg<T>::EPV) * (int)sizeof(T);
    // perfect tree: every CTA holds LPC leaves (or all L < LPC) -> power-of-two groups
    const int depth = pairwise_perfect_depth(n);
    const int perfect = depth >= 0 && (n_leaves <= LPC || n_leaves % LPC == 0) ? 1 : 0;
    const int g = (n_leaves + LPC - 1) / LPC;
    int smem, tree_smem = 0;
    if (perfect) {
      smem = stage > 2 * g * 8 ? stage : 2 * g * 8;
    } else {
      const int tree = stride * 8;
      tree_smem = tree <= 100 * 1024 ? 1 : 0;
      smem = tree_smem ? (stage > tree ? stage : tree) : stage;
    }
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(mse_fused_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
    if (smem > 200 * 1024) return set_error(PS_ERR_INPUT, "cache_predict: leaf span too large");
    launch_pdl(mse_fused_kernel<T>, dim3((n_leaves + LPC - 1) / LPC, P), dim3(LPC), (size_t)smem, st,
               (const T*)x, n, slots, (const T*)snap_in, exists, streak, max_streak, sigma, leaves, n_leaves, nodes,
               n_internal, level_off, n_levels, scratch, tickets, mask, counters, tree_smem, perfect);
    count_launch();
    return check_launch("mse_reuse_test");
  };
  if (dtype == PS_DTYPE_BF16) return run(__nv_bfloat16{});
  if (dtype == PS_DTYPE_F32) return run(float{});
  if (dtype == PS_DTYPE_F64) return run(double{});
  return set_error(PS_ERR_INPUT, "cache_predict: unsupported dtype %d", dtype);
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
                    int dtype, const void* snap_in, const void* snap_out, void* ins, void* outs, int32_t* error_flag) {
  PatchOpArgs a{};
  a.mask = mask; a.slots = slots; a.exists = const_cast<uint8_t*>(exists);
  a.snap_in = (char*)snap_in; a.snap_out = (char*)snap_out;
  a.o1 = (char*)ins; a.o2 = (char*)outs; a.err = error_flag;
  return launch_op<OP_GATHER>((cudaStream_t)stream, P, n, dtype, a, "cache_gather");
}

int ps_cache_fill(void* stream, const uint8_t* mask, const int32_t* slots, const uint8_t* exists, int32_t* streak,
                  int P, int64_t n, int dtype, const void* snap_out, void* out, int32_t* error_flag) {
  PatchOpArgs a{};
  a.mask = mask; a.slots = slots; a.exists = const_cast<uint8_t*>(exists); a.streak = streak;
  a.snap_out = (char*)snap_out; a.o1 = (char*)out; a.err = error_flag;
  return launch_op<OP_FILL>((cudaStream_t)stream, P, n, dtype, a, "cache_fill");
}

int ps_cache_update(void* stream, const uint8_t* mask, const int32_t* slots, uint8_t* exists, int32_t* streak, int P,
                    int64_t n, int dtype, const void* x, const void* y, void* snap_in, void* snap_out,
                    int64_t* counters) {
  PatchOpArgs a{};
  a.mask = mask; a.slots = slots; a.exists = exists; a.streak = streak;
  a.x = (const char*)x; a.y = (char*)y;
  a.snap_in = (char*)snap_in; a.snap_out = (char*)snap_out; a.counters = counters;
  return launch_op<OP_UPDATE>((cudaStream_t)stream, P, n, dtype, a, "cache_update");
}

int ps_cache_evict(void* stream, uint8_t* exists, int32_t* streak, const int32_t* slots, int n_slots) {
  if (n_slots == 0) return PS_OK;
  evict_kernel<<<(n_slots + 255) / 256, 256, 0, (cudaStream_t)stream>>>(exists, streak, slots, n_slots);
  count_launch();
  return check_launch("cache_evict");
}

int ps_cache_substitute(void* stream, const uint8_t* mask, const int32_t* slots, int P, int64_t n, int dtype,
                        const void* x, const void* snap_in, void* x_sub, const int32_t* patches, int n_list,
                        const int32_t* n_dev) {
  PatchOpArgs a{};
  a.mask = mask; a.slots = slots; a.x = (const char*)x;
  a.snap_in = (char*)snap_in; a.o1 = (char*)x_sub;
  a.plist = patches; a.n_dev = patches ? n_dev : nullptr;
  return launch_op<OP_SUBST>((cudaStream_t)stream, patches ? n_list : P, n, dtype, a, "cache_substitute");
}

int ps_cache_finish(void* stream, const uint8_t* mask, const int32_t* slots, uint8_t* exists, int32_t* streak, int P,
                    int64_t n, int dtype, const void* x, void* y, void* snap_in, void* snap_out, int64_t* counters) {
  PatchOpArgs a{};
  a.mask = mask; a.slots = slots; a.exists = exists; a.streak = streak;
  a.x = (const char*)x; a.y = (char*)y;
  a.snap_in = (char*)snap_in; a.snap_out = (char*)snap_out; a.counters = counters;
  return launch_op<OP_FINISH>((cudaStream_t)stream, P, n, dtype, a, "cache_finish");
}

int ps_select_patches(void* stream, const uint8_t* mask, int P, int64_t n, int dtype, const void* a_, const void* b_,
                      void* out) {
  PatchOpArgs a{};
  a.mask = mask; a.x = (const char*)a_; a.y = (char*)b_; a.o1 = (char*)out;
  return launch_op<OP_SELECT>((cudaStream_t)stream, P, n, dtype, a, "select_patches");
}

}  // extern "C"
