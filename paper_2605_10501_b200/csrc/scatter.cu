// K6: encoder outputs -> packed backbone token stream at placeholder rows, and its backward.
//
// Not in the reference (4:1 downsampled visual tokens concatenated with
// text).  HBM-bound row movement: one warp per row, 16-byte vectors, several rows in
// flight per warp; the backward is a segmented gather-reduce in fp32 (a 1:1 placeholder map
// degenerates to a copy but the kernel accepts any CSR segment structure).
#include <cuda_bf16.h>

#include "common.cuh"

namespace mb {
namespace {

constexpr int kRowsPerWarp = 4;
// pos != nullptr: the pair range is [pos[k0], pos[k1]) read on device (K5b handoff index of one
// micro-batch), n_rows only bounds the grid
template <bool ACC>
__global__ void __launch_bounds__(256) scatter_rows_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                           const int32_t* __restrict__ src_row,
                                                           const int32_t* __restrict__ dst_row, int n_rows,
                                                           int vec_per_row, const int32_t* __restrict__ pos, int k0,
                                                           int k1) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  int lo = 0, hi = n_rows;
  if (pos != nullptr) {
    lo = pos[k0];
    hi = pos[k1];
  }
  const int r0 = lo + warp * kRowsPerWarp;
#pragma unroll
  for (int k = 0; k < kRowsPerWarp; ++k) {
    const int r = r0 + k;
    if (r >= hi) return;
    const uint4* s = src + (size_t)src_row[r] * vec_per_row;
    uint4* d = dst + (size_t)dst_row[r] * vec_per_row;
    for (int v0 = lane; v0 < vec_per_row; v0 += 4 * 32) {  // four 16-byte loads in flight per lane
      uint4 x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int v = v0 + u * 32;
        if (v < vec_per_row)
          asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(x[u].x), "=r"(x[u].y), "=r"(x[u].z), "=r"(x[u].w)
                       : "l"(s + v));
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (v0 + u * 32 < vec_per_row) {
          if constexpr (ACC) {  // dst += src (bf16 rows, fp32 sum rounded once)
            uint4 y = d[v0 + u * 32];
            __nv_bfloat162* yh = reinterpret_cast<__nv_bfloat162*>(&y);
            const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(&x[u]);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 a = __bfloat1622float2(yh[e]), c = __bfloat1622float2(xh[e]);
              yh[e] = __floats2bfloat162_rn(a.x + c.x, a.y + c.y);
            }
            d[v0 + u * 32] = y;
          } else {
            d[v0 + u * 32] = x[u];
          }
        }
    }
  }
}

__global__ void __launch_bounds__(256) gather_rows_bwd_kernel(const __nv_bfloat16* __restrict__ ddst,
                                                              __nv_bfloat16* __restrict__ dsrc,
                                                              const int32_t* __restrict__ seg,
                                                              const int32_t* __restrict__ seg_dst, int n_src,
                                                              int d) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n_src) return;
  const int k0 = seg[warp], k1 = seg[warp + 1];
  __nv_bfloat16* out = dsrc + (size_t)warp * d;
  // four 16-byte column chunks per step: their loads are independent, so they are in flight together
  for (int c0 = lane * 8; c0 < d; c0 += 4 * 32 * 8) {
    float acc[4][8] = {};
    for (int k = k0; k < k1; ++k) {
      const __nv_bfloat16* row = ddst + (size_t)seg_dst[k] * d;
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (c0 + u * 256 < d) v[u] = *reinterpret_cast<const uint4*>(row + c0 + u * 256);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (c0 + u * 256 >= d) break;
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v[u]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float2 f = __bfloat1622float2(h[j]);
          acc[u][2 * j] += f.x;
          acc[u][2 * j + 1] += f.y;
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (c0 + u * 256 >= d) break;
      uint4 o;
      __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int j = 0; j < 4; ++j) oh[j] = __floats2bfloat162_rn(acc[u][2 * j], acc[u][2 * j + 1]);
      *reinterpret_cast<uint4*>(out + c0 + u * 256) = o;
    }
  }
}

}  // namespace
}  // namespace mb

using namespace mb;

MAESTRO_API int maestro_scatter_rows_fwd(const void* d_src, void* d_dst, const int32_t* d_src_row,
                                         const int32_t* d_dst_row, int32_t n_rows, int32_t d, void* stream) {
  if (n_rows <= 0) return 0;
  if (d % 8) return (int)cudaErrorInvalidValue;
  const int warps = (n_rows + kRowsPerWarp - 1) / kRowsPerWarp;
  const int blocks = (warps * 32 + 255) / 256;
  launch_pdl(scatter_rows_kernel<false>, dim3(blocks), dim3(256), 0, (cudaStream_t)stream, (const uint4*)d_src, (uint4*)d_dst, d_src_row,
                                                                       d_dst_row, n_rows, d / 8, nullptr, 0, 0);
  return launch_status();
}

// Row scatter over the pairs [d_pos[k0], d_pos[k1]) of a handoff index (maestro_handoff_index):
// the range stays on device; max_rows (>= the range length) sizes the grid.  accumulate != 0:
// dst rows += src rows (a downstream section's gradient added into the backbone's).
MAESTRO_API int maestro_scatter_rows_range(const void* d_src, void* d_dst, const int32_t* d_src_row,
                                           const int32_t* d_dst_row, const int32_t* d_pos, int32_t k0, int32_t k1,
                                           int32_t max_rows, int32_t d, int32_t accumulate, void* stream) {
  if (max_rows <= 0 || k1 <= k0) return 0;
  if (d % 8) return (int)cudaErrorInvalidValue;
  const int warps = (max_rows + kRowsPerWarp - 1) / kRowsPerWarp;
  const int blocks = (warps * 32 + 255) / 256;
  if (accumulate)
    launch_pdl(scatter_rows_kernel<true>, dim3(blocks), dim3(256), 0, (cudaStream_t)stream, 
        (const uint4*)d_src, (uint4*)d_dst, d_src_row, d_dst_row, max_rows, d / 8, d_pos, k0, k1);
  else
    launch_pdl(scatter_rows_kernel<false>, dim3(blocks), dim3(256), 0, (cudaStream_t)stream, 
        (const uint4*)d_src, (uint4*)d_dst, d_src_row, d_dst_row, max_rows, d / 8, d_pos, k0, k1);
  return launch_status();
}

MAESTRO_API int maestro_gather_rows_bwd(const void* d_ddst, void* d_dsrc, const int32_t* d_seg,
                                        const int32_t* d_seg_dst, int32_t n_src_rows, int32_t d, void* stream) {
  if (n_src_rows <= 0) return 0;
  if (d % 8) return (int)cudaErrorInvalidValue;
  const int blocks = (n_src_rows * 32 + 255) / 256;
  launch_pdl(gather_rows_bwd_kernel, dim3(blocks), dim3(256), 0, (cudaStream_t)stream, 
      (const __nv_bfloat16*)d_ddst, (__nv_bfloat16*)d_dsrc, d_seg, d_seg_dst, n_src_rows, d);
  return launch_status();
}
