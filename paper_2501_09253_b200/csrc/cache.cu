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
    // Fast form of the same arithmetic: d = a - b in fp32 is exact iff rounding down and up
    // agree (both finite); then d has <= 24 significant bits, d^2 is exact in fp64, so
    // fma(d, d, r) rounds the same exact sum r + d^2 once -- bit-identical to
    // dadd(r, dmul(dsub(a, b), dsub(a, b))) with one F2F.F64.F32 per element instead of two and one
    // DFMA instead of DSUB + DMUL + DADD.  A group with any inexact difference (exponent gap > 15,
    // overflow, non-finite) takes the fp64 path.
    auto d8f = [&](int i, float* d) {
      const uint4 ua = *reinterpret_cast<const uint4*>(a + i);
      const uint4 ub = *reinterpret_cast<const uint4*>(b + i);
      const __nv_bfloat162* ha = reinterpret_cast<const __nv_bfloat162*>(&ua);
      const __nv_bfloat162* hb = reinterpret_cast<const __nv_bfloat162*>(&ub);
      bool ok = true;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float a0 = __low2float(ha[k]), b0 = __low2float(hb[k]);
        const float a1 = __high2float(ha[k]), b1 = __high2float(hb[k]);
        d[2 * k] = __fsub_rd(a0, b0);
        d[2 * k + 1] = __fsub_rd(a1, b1);
        ok &= (d[2 * k] == __fsub_ru(a0, b0)) & (d[2 * k + 1] == __fsub_ru(a1, b1));
      }
      return ok;
    };
    {
      float d[8];
      if (d8f(0, d)) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dmul_rn((double)d[j], (double)d[j]);
      } else {
        sq8(0, r);
      }
    }
    int i = 8;
    const int stop = n - (n % 8);
    for (; i < stop; i += 8) {
      float d[8];
      if (d8f(i, d)) {
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __fma_rn((double)d[j], (double)d[j], r[j]);
      } else {
        double d8[8];
        sq8(i, d8);
#pragma unroll
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], d8[j]);
      }
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

// Persistent form of the perfect-tree reuse test (default when numpy's tree over n is perfect
// and the operands are vector-aligned): two kernels, no cross-CTA tickets or fences.
//
// mse_ring_kernel: 2 CTAs per SM walk the (patch, chunk of LPC leaves) items with a stride of the
// grid; each keeps S chunks of both operands in flight as 1-D bulk copies, so the loads of the
// next chunks overlap the fp64 leaf sums of the current one.  A bf16 leaf is summed by MSE_TPL = 4
// threads, each owning two of numpy's eight strided accumulators (r[2q], r[2q+1]); the leaf total
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) is formed with two shuffles in that order, then the n % 8
// tail -- numpy's arithmetic, 4x the threads.  The chunk's leaves reduce pairwise (shuffles in
// lane order, one barrier) to the chunk subtree root, written to scratch.
// mse_root_kernel: per patch, the perfect tree over its chunk roots, the mask, the counters.
// (One CTA per chunk with a ticket convoyed -- all resident CTAs of the GPU loaded, then all
// computed with the HBM idle: 40% of DRAM peak, 47 us; a ring with one thread per leaf ran out of
// warps (8 per SM) for the fp64 chains and waited on its MEMBAR.SC ticket fences: 84 us.)
// Bit-identical to mse_fused_kernel.
constexpr int MSE_MAX_STAGES = 4;
template <typename T>
struct MseRing {
  static constexpr int TPL = sizeof(T) == 2 ? 2 : 1;  // threads per leaf
  static constexpr int THREADS = MseCfg<T>::LPC * TPL;
};

// bf16 leaf over TPL = 2 adjacent lanes (h = lane % 2).  All lanes call it (shuffle); `on` masks
// lanes without a leaf.  Returns the leaf sum on h == 0.
__device__ __forceinline__ double leaf_sum_h2(const __nv_bfloat16* a, const __nv_bfloat16* b, int n, int h, bool on) {
  auto sq = [&](int i) {
    const double d = __dsub_rn((double)__bfloat162float(a[i]), (double)__bfloat162float(b[i]));
    return __dmul_rn(d, d);
  };
  if (n < 8) {  // sequential from -0.0, one lane
    double res = -0.0;
    if (on && h == 0)
      for (int i = 0; i < n; ++i) res = __dadd_rn(res, sq(i));
    return res;
  }
  // Lane h owns numpy's accumulators r[4h .. 4h+3]: elements 4h .. 4h+3 of every 8-element
  // group (one 8-byte load per operand).  A branch-free sweep takes the fp32 differences rounded
  // down and up -- equal iff exact (see leaf_sum); the XOR of their bits is OR-accumulated (one
  // LOP3), ignoring the sign bit, which only an exact zero (-0 vs +0) can flip -- and accumulates
  // fma(d, d, r).  If any difference was inexact the lane redoes its sweep in fp64: both sweeps
  // round the same exact values.
  const int stop = n - (n % 8);
  const uint2* pa = reinterpret_cast<const uint2*>(a + 4 * h);
  const uint2* pb = reinterpret_cast<const uint2*>(b + 4 * h);
  const int ng = stop / 8;
  double r[4] = {0.0, 0.0, 0.0, 0.0};
  if (on) {
    uint32_t bad = 0;
    auto diffs = [&](int k, float (&d)[4]) {
      const uint2 ua = pa[2 * k], ub = pb[2 * k];
      const float av[4] = {__uint_as_float(ua.x << 16), __uint_as_float(ua.x & 0xffff0000u),
                           __uint_as_float(ua.y << 16), __uint_as_float(ua.y & 0xffff0000u)};
      const float bv[4] = {__uint_as_float(ub.x << 16), __uint_as_float(ub.x & 0xffff0000u),
                           __uint_as_float(ub.y << 16), __uint_as_float(ub.y & 0xffff0000u)};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        d[e] = __fsub_rd(av[e], bv[e]);
        bad |= __float_as_uint(d[e]) ^ __float_as_uint(__fsub_ru(av[e], bv[e]));
      }
    };
    {
      float d[4];
      diffs(0, d);
#pragma unroll
      for (int e = 0; e < 4; ++e) r[e] = __dmul_rn((double)d[e], (double)d[e]);
    }
#pragma unroll 3
    for (int k = 1; k < ng; ++k) {
      float d[4];
      diffs(k, d);
#pragma unroll
      for (int e = 0; e < 4; ++e) r[e] = __fma_rn((double)d[e], (double)d[e], r[e]);
    }
    if (bad & 0x7fffffffu) {
      for (int k = 0; k < ng; ++k) {
        const uint2 ua = pa[2 * k], ub = pb[2 * k];
        const uint32_t aw[4] = {ua.x << 16, ua.x & 0xffff0000u, ua.y << 16, ua.y & 0xffff0000u};
        const uint32_t bw[4] = {ub.x << 16, ub.x & 0xffff0000u, ub.y << 16, ub.y & 0xffff0000u};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const double f = __dsub_rn((double)__uint_as_float(aw[e]), (double)__uint_as_float(bw[e]));
          r[e] = k ? __dadd_rn(r[e], __dmul_rn(f, f)) : __dmul_rn(f, f);
        }
      }
    }
  }
  const double t = __dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3]));  // h = 0: (r0+r1)+(r2+r3)
  double res = __dadd_rn(t, __shfl_down_sync(0xffffffffu, t, 1));         // + ((r4+r5)+(r6+r7))
  if (on && h == 0)
    for (int i = stop; i < n; ++i) res = __dadd_rn(res, sq(i));
  return res;
}

template <typename T>
__global__ void __launch_bounds__(MseRing<T>::THREADS + 32, 2) mse_ring_kernel(
    const T* __restrict__ x, int64_t n, const int32_t* __restrict__ slots, const T* __restrict__ snap,
    const uint8_t* __restrict__ exists, const int32_t* __restrict__ streak, int max_streak,
    const int32_t* __restrict__ leaves, int L, int I, int CP, int P, int S, int stage_elems,
    int leaf_len, int cp_shift, double* __restrict__ scratch) {
  // leaf_len > 0: every leaf has that many elements (leaf l starts at l * leaf_len), so the item
  // loop reads no plan table; CP = 1 << cp_shift chunks per patch.
  // Warp-specialised: warps [0, NW) sum leaves; warp NW is the producer -- it resolves the
  // entries (slot, exists, streak: three dependent loads) of its next 32 items at once, one item
  // per lane, and issues the bulk copies as stages free up, so no compute warp waits on the
  // dependent loads (on warp 0 they held the whole CTA at the next barrier: 22% of the stalls).
  constexpr int LPC = MseCfg<T>::LPC, EPV = MseCfg<T>::EPV, TPL = MseRing<T>::TPL;
  constexpr int CT = MseRing<T>::THREADS, NW = CT / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t full[MSE_MAX_STAGES], empty[MSE_MAX_STAGES];
  __shared__ int dead[MSE_MAX_STAGES];
  pdl_wait();
  pdl_trigger();  // mse_root_kernel's CTAs become resident now and read their entries early
  const int n_items = P * CP;
  if ((int)blockIdx.x >= n_items) return;
  const int stride = L + I;
  T* stages = reinterpret_cast<T*>(smem_raw);
  double* red = reinterpret_cast<double*>(smem_raw + (size_t)S * 2 * stage_elems * sizeof(T));
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == NW) {  // ---------------------------------------------------------- producer
    int live_w = 0, slot_w = -1;
    int j = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++j) {
      if ((j & 31) == 0) {  // entries of items j .. j+31, one per lane
        const int itl = it + lane * (int)gridDim.x;
        slot_w = -1;
        live_w = 0;
        if (itl < n_items) {
          slot_w = slots[itl >> cp_shift];
          live_w = entry_live(slot_w, exists, streak, max_streak) ? 1 : 0;
        }
      }
      const int live = __shfl_sync(0xffffffffu, live_w, j & 31);
      const int slot = __shfl_sync(0xffffffffu, slot_w, j & 31);
      const int s = j % S;
      if (lane == 0) {
        if (j >= S) mbar_wait(&empty[s], (uint32_t)(((j / S) - 1) & 1));
        dead[s] = live ? 0 : 1;
        if (!live) {
          mbar_arrive(&full[s]);
        } else {
          const int p = it >> cp_shift, c = it & (CP - 1);
          const int l0 = c * LPC, l1 = min(L, l0 + LPC);
          const int64_t e0 = leaf_len > 0 ? (int64_t)l0 * leaf_len : (int64_t)leaves[2 * l0];
          const int64_t e1 = leaf_len > 0 ? (int64_t)l1 * leaf_len
                                          : (int64_t)leaves[2 * (l1 - 1)] + leaves[2 * (l1 - 1) + 1];
          const int64_t v0 = e0 & ~int64_t(EPV - 1), v1 = (e1 + EPV - 1) & ~int64_t(EPV - 1);
          const uint32_t bytes = (uint32_t)((v1 - v0) * sizeof(T));
          T* sa = stages + (size_t)s * 2 * stage_elems;
          mbar_arrive_expect_tx(&full[s], 2 * bytes);
          bulk_load(sa, x + (int64_t)p * n + v0, bytes, &full[s]);
          bulk_load(sa + stage_elems, snap + (int64_t)slot * n + v0, bytes, &full[s]);
        }
      }
      __syncwarp();
    }
    return;
  }
  // ------------------------------------------------------------------------ compute warps
  const int lt = threadIdx.x / TPL, q = threadIdx.x % TPL;
  int j = 0;
  for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++j) {
    const int s = j % S;
    mbar_wait(&full[s], (uint32_t)((j / S) & 1));
    const int p = it >> cp_shift, c = it & (CP - 1);
    if (dead[s]) {  // no entry / streak exhausted: mse_root_kernel writes the mask
      named_bar_sync(1, CT);  // every compute thread has read dead[s] before the stage is released
      if (threadIdx.x == 0) mbar_arrive(&empty[s]);
      continue;
    }
    const int l0 = c * LPC, l1 = min(L, l0 + LPC);
    const int64_t v0 = (leaf_len > 0 ? (int64_t)l0 * leaf_len : (int64_t)leaves[2 * l0]) & ~int64_t(EPV - 1);
    const T* sa = stages + (size_t)s * 2 * stage_elems;
    const int l = l0 + lt;
    const bool on = l < l1;
    const int64_t st = on ? (leaf_len > 0 ? (int64_t)l * leaf_len : (int64_t)leaves[2 * l]) - v0 : 0;
    const int ln = on ? (leaf_len > 0 ? leaf_len : leaves[2 * l + 1]) : 8;
    double leaf;
    if constexpr (TPL == 2) {
      leaf = leaf_sum_h2(sa + st, sa + stage_elems + st, ln, q, on);
    } else {
      leaf = on ? leaf_sum<T>(sa + st, sa + stage_elems + st, ln) : 0.0;
    }
    // the chunk's perfect subtree over its (l1 - l0, a power of two) leaves: butterfly adds in
    // lane order give each warp's subtree (left + right at every level), then warp 0 combines the
    // warp roots the same way.  A chunk shorter than LPC (L < LPC) pads with +0.0 leaves on the
    // right, whose subtrees are +0.0 and add exactly (a leaf sum is never -0.0).
    double t = (q == 0 && on) ? leaf : 0.0;
#pragma unroll
    for (int off = TPL; off < 32; off <<= 1) t = __dadd_rn(t, __shfl_down_sync(0xffffffffu, t, off));
    double* wr = red + (j & 1) * NW;  // double-buffered: the next item writes the other half
    if (lane == 0) wr[warp] = t;
    named_bar_sync(1, CT);  // the stage is consumed: the producer may refill it
    if (threadIdx.x == 0) mbar_arrive(&empty[s]);
    if (warp == 0) {
      double w = lane < NW ? wr[lane] : 0.0;
#pragma unroll
      for (int off = 1; off < NW; off <<= 1) w = __dadd_rn(w, __shfl_down_sync(0xffffffffu, w, off));
      if (lane == 0) scratch[(int64_t)p * stride + c] = w;  // chunk subtree root
    }
  }
}

// grid P, 32 threads: patch p's tree over its CP chunk roots (perfect, CP a power of two), then
// the mask (mse < sigma, strict) and the counters; patches without a live entry get mask 0.
__global__ void __launch_bounds__(32) mse_root_kernel(const int32_t* __restrict__ slots,
                                                      const uint8_t* __restrict__ exists,
                                                      const int32_t* __restrict__ streak, int max_streak,
                                                      double sigma, int64_t n, int L, int I, int CP,
                                                      double* __restrict__ scratch, uint8_t* __restrict__ mask,
                                                      int64_t* __restrict__ counters) {
  extern __shared__ double rr[];
  const int p = blockIdx.x;
  // the entry state was written before mse_ring_kernel started (which triggers this launch
  // after its own pdl_wait), so it is read ahead of the wait for the chunk roots
  const bool live = entry_live(slots[p], exists, streak, max_streak);
  pdl_wait();
  if (!live) {
    if (threadIdx.x == 0) {
      mask[p] = 0;
      if (counters) atomicAdd(reinterpret_cast<unsigned long long*>(counters + 1), 1ull);
    }
    return;
  }
  double* v = scratch + (int64_t)p * (L + I);
  for (int i = threadIdx.x; i < CP; i += blockDim.x) rr[i] = v[i];
  __syncthreads();
  const double r = smem_pairwise(rr, rr + CP, CP);
  if (threadIdx.x == 0) {
    v[I > 0 ? L + I - 1 : 0] = r;  // readable in scratch (ps.mse)
    const double mse = __ddiv_rn(__dadd_rn(0.0, r), (double)n);
    const bool m = mse < sigma;
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


// XOR fold of a buffer's 32-byte words into one u32 (order-independent, so any streaming order
// gives the same value): an integrity check for resident latents / snapshots after a copy, and the
// pure-read ceiling the read-only patch kernels are measured against (bench.py hbm_kernels: a
// streaming read of the same bytes, nothing but the loads -- tools/micro/read_bw.cu swept 14
// read-kernel shapes; this is the fastest of them at 76 / 152 MB: LDG.256, two per thread in
// flight, 8 CTAs of 256 threads per SM).
__global__ void __launch_bounds__(256) checksum_kernel(const uint8_t* __restrict__ p, int64_t nv,
                                                      uint32_t* __restrict__ out) {
  pdl_wait();
  uint32_t acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k0 < nv; k0 += 2 * stride) {
    uint32_t r[2][8];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int64_t k = k0 + i * stride;
      if (k < nv) {
        ld_global_nc_v8(p + k * 32, r[i]);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) r[i][e] = 0;
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc ^= r[i][e];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc != 0) atomicXor(out, acc);
}
}  // namespace ps

extern "C" {

static int ring_num_sms() {
  static int nsm = 0;
  if (nsm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  return nsm;
}

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
      cudaFuncSetAttribute(mse_ring_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
    static const bool ring_off = getenv("PS_MSE_RING_OFF") && atoi(getenv("PS_MSE_RING_OFF")) != 0;
    if (!ring_off && perfect && n % MseCfg<T>::EPV == 0 && ((uintptr_t)x & 15) == 0 && ((uintptr_t)snap_in & 15) == 0) {
      const int stage_elems = (int)(pairwise_max_span(n, LPC) + 2 * MseCfg<T>::EPV);
      const int stage_bytes = 2 * stage_elems * (int)sizeof(T);
      const int RW = 32;  // red: 2 x (warps per CTA <= 16) doubles
      int S = (110 * 1024 - 2 * RW * 8) / stage_bytes;
      if (S > MSE_MAX_STAGES) S = MSE_MAX_STAGES;
      // equal leaves (the widest leaf is n / L): starts by arithmetic; g is a power of two
      const int leaf_len = (n % n_leaves == 0 && pairwise_max_span(n, 1) == n / n_leaves) ? (int)(n / n_leaves) : 0;
      int cp_shift = 0;
      while ((1 << cp_shift) < g) ++cp_shift;
      if (S >= 2 && (size_t)2 * g * 8 <= 48 * 1024 && (1 << cp_shift) == g) {
        const size_t smem_r = (size_t)S * stage_bytes + 2 * RW * 8;
        const int items = P * g;
        const int grid = items < 2 * ring_num_sms() ? items : 2 * ring_num_sms();
        launch_pdl(mse_ring_kernel<T>, dim3(grid), dim3(MseRing<T>::THREADS + 32), smem_r, st, (const T*)x, n, slots,
                   (const T*)snap_in, exists, streak, max_streak, leaves, n_leaves, n_internal, g, P, S, stage_elems,
                   leaf_len, cp_shift, scratch);
        count_launch();
        const int rc = check_launch("mse_reuse_test");
        if (rc != PS_OK) return rc;
        launch_pdl(mse_root_kernel, dim3(P), dim3(32), (size_t)2 * g * 8, st, slots, exists, streak, max_streak,
                   sigma, n, n_leaves, n_internal, g, scratch, mask, counters);
        count_launch();
        return check_launch("mse_reuse_roots");
      }
    }
    if (smem > 200 * 1024) return set_error(PS_ERR_INPUT, "cache_predict: leaf span too large");
    // per-patch tickets of the one-kernel form only (the ring path above has no cross-CTA tickets)
    if (cudaMemsetAsync(tickets, 0, (size_t)P * sizeof(int), st) != cudaSuccess)
      return check_launch("cache_predict tickets");
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

int ps_checksum(void* stream, const void* data, int64_t bytes, uint32_t* out) {
  if (bytes < 0 || bytes % 32 != 0 || ((uintptr_t)data & 31) != 0 || out == nullptr)
    return set_error(PS_ERR_INPUT, "checksum: needs 32-byte aligned data, a multiple of 32 bytes and an output word");
  if (bytes == 0) return PS_OK;
  const int64_t nv = bytes / 32;
  int64_t grid = 8 * (int64_t)ring_num_sms();
  const int64_t need = (nv + 511) / 512;  // two 32-byte loads per thread
  if (need < grid) grid = need;
  launch_pdl(checksum_kernel, dim3((unsigned)grid), dim3(256), 0, (cudaStream_t)stream, (const uint8_t*)data, nv, out);
  count_launch();
  return check_launch("checksum");
}

}  // extern "C"
