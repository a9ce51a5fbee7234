// Data movers of the split-image multi-GPU path: pack / unpack
// of the halo strips (one pixel row or column of a patch, all channels) that a
// conv3 on one GPU reads from a neighbour patch owned by another GPU
// (exchange_halos, patched.py:57-89, across a shard cut), and indexed segment
// copies that pack GroupNorm partials (patched.py:132-140) and attention K / V^T
// token ranges (patched.py:164-176) into contiguous NCCL buffers and back.
//
// Both are HBM copy kernels: 16-byte accesses where alignment allows, grid
// sized to a multiple of the SM count, no shared memory needed (every byte is
// read once and written once).
#include "common.cuh"
#include "ps_internal.h"

namespace ps {

// Thread per (segment, 16-byte chunk).  A segment whose two ends are 16-byte
// aligned moves as uint4; otherwise the chunk moves as up to 8 u16 elements.
__global__ void __launch_bounds__(256) copy_segments_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                                            int n, const int64_t* __restrict__ src_off,
                                                            const int64_t* __restrict__ dst_off, int64_t seg_bytes) {
  const int64_t chunks = (seg_bytes + 15) / 16;
  const int64_t total = (int64_t)n * chunks;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = k / chunks, c = k - s * chunks;
    const uint8_t* a = src + __ldg(src_off + s) + c * 16;
    uint8_t* b = dst + __ldg(dst_off + s) + c * 16;
    const int64_t left = seg_bytes - c * 16;
    if (left >= 16 && (((uintptr_t)a | (uintptr_t)b) & 15) == 0) {
      *reinterpret_cast<uint4*>(b) = __ldg(reinterpret_cast<const uint4*>(a));
    } else {
      const int m = (int)(left < 16 ? left : 16) / 2;
      for (int i = 0; i < m; ++i)
        reinterpret_cast<uint16_t*>(b)[i] = __ldg(reinterpret_cast<const uint16_t*>(a) + i);
    }
  }
}

// Variable-length form: CTA per segment (grid-stride), segment s moves seg_bytes[s] bytes.  The
// K / V^T pack and unpack of every peer's token ranges go out as one launch each instead of one
// per (peer, token-run length).  The segments are V^T rows (ntok x 2 bytes: 24-64 KB at config
// 5), so a whole CTA streams each one (a warp per segment left 40 CTAs: 34 us for 21 MB).
__global__ void __launch_bounds__(256) copy_segments_var_kernel(const uint8_t* __restrict__ src,
                                                                uint8_t* __restrict__ dst, int n,
                                                                const int64_t* __restrict__ src_off,
                                                                const int64_t* __restrict__ dst_off,
                                                                const int64_t* __restrict__ seg_bytes) {
  for (int64_t s = blockIdx.x; s < n; s += gridDim.x) {
    const uint8_t* a = src + __ldg(src_off + s);
    uint8_t* b = dst + __ldg(dst_off + s);
    const int64_t len = __ldg(seg_bytes + s);
    if ((((uintptr_t)a | (uintptr_t)b | (uintptr_t)len) & 15) == 0) {
      const uint4* a4 = reinterpret_cast<const uint4*>(a);
      uint4* b4 = reinterpret_cast<uint4*>(b);
      const int64_t nv = len / 16;
      const int T = blockDim.x;
      int64_t k = threadIdx.x;
      for (; k + T < nv; k += 2 * T) {  // two 16-byte loads in flight per thread
        const uint4 r0 = __ldg(a4 + k), r1 = __ldg(a4 + k + T);
        b4[k] = r0;
        b4[k + T] = r1;
      }
      for (; k < nv; k += T) b4[k] = __ldg(a4 + k);
    } else {
      for (int64_t k = threadIdx.x; k < len / 2; k += blockDim.x)
        reinterpret_cast<uint16_t*>(b)[k] = __ldg(reinterpret_cast<const uint16_t*>(a) + k);
    }
  }
}

// grid (n strips, ceil(C*ps / 256)): strip i = (patch q, code); code < ps is
// pixel row `code`, code >= ps is pixel column `code - ps`.  Buffer strip
// layout [C][ps] bf16.  unpack != 0 writes the buffer back into x.
__global__ void __launch_bounds__(256) halo_strips_kernel(__nv_bfloat16* __restrict__ x, int C, int ps,
                                                          const int32_t* __restrict__ desc,
                                                          __nv_bfloat16* __restrict__ buf, int unpack) {
  const int i = blockIdx.x;
  const int q = __ldg(desc + 2 * i), code = __ldg(desc + 2 * i + 1);
  const int e = blockIdx.y * blockDim.x + threadIdx.x;
  if (e >= C * ps) return;
  const int c = e / ps, j = e - c * ps;
  const int y = code < ps ? code : j, xc = code < ps ? j : code - ps;
  const int64_t xo = (((int64_t)q * C + c) * ps + y) * ps + xc;
  const int64_t bo = (int64_t)i * C * ps + e;
  if (unpack) x[xo] = buf[bo];
  else buf[bo] = x[xo];
}

}  // namespace ps

using namespace ps;

extern "C" {

int ps_copy_segments(void* stream, const void* src, void* dst, int n, const int64_t* src_off, const int64_t* dst_off,
                     int64_t seg_bytes) {
  if (n < 0 || seg_bytes < 0 || seg_bytes % 2)
    return set_error(PS_ERR_INPUT, "copy_segments: n=%d seg_bytes=%lld (must be even)", n, (long long)seg_bytes);
  if (n == 0 || seg_bytes == 0) return PS_OK;
  const int64_t total = (int64_t)n * ((seg_bytes + 15) / 16);
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  copy_segments_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
      (const uint8_t*)src, (uint8_t*)dst, n, src_off, dst_off, seg_bytes);
  count_launch();
  return check_launch("copy_segments");
}

int ps_copy_segments_var(void* stream, const void* src, void* dst, int n, const int64_t* src_off,
                         const int64_t* dst_off, const int64_t* seg_bytes) {
  if (n < 0) return set_error(PS_ERR_INPUT, "copy_segments_var: n=%d", n);
  if (n == 0) return PS_OK;
  const int64_t blocks = n < 148 * 8 ? n : 148 * 8;
  copy_segments_var_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
      (const uint8_t*)src, (uint8_t*)dst, n, src_off, dst_off, seg_bytes);
  count_launch();
  return check_launch("copy_segments_var");
}

int ps_halo_strips(void* stream, void* x, int C, int ps_, int n, const int32_t* desc, void* buf, int unpack) {
  if (n < 0 || C < 1 || ps_ < 1) return set_error(PS_ERR_INPUT, "halo_strips: n=%d C=%d ps=%d", n, C, ps_);
  if (n == 0) return PS_OK;
  halo_strips_kernel<<<dim3(n, (C * ps_ + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      (__nv_bfloat16*)x, C, ps_, desc, (__nv_bfloat16*)buf, unpack);
  count_launch();
  return check_launch("halo_strips");
}

}  // extern "C"
