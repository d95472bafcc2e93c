// Memory-bound kernels of the section compute: fused residual-add + RMSNorm (fwd/bwd), RoPE,
// SwiGLU, embedding gather / scatter-add, varlen positions and the fused multi-tensor AdamW.
// All are HBM-bound: 16-byte vectors, fp32 math, one pass where the dependency allows.
#include <cuda_bf16.h>

#include "common.cuh"

namespace mb {
namespace {

__device__ __forceinline__ void ld8(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 v = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 x = __bfloat1622float2(h[j]);
    f[2 * j] = x.x;
    f[2 * j + 1] = x.y;
  }
}
__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 x = __bfloat1622float2(h[j]);
    f[2 * j] = x.x;
    f[2 * j + 1] = x.y;
  }
}
__device__ __forceinline__ void st8(__nv_bfloat16* p, const float (&f)[8]) {
  uint4 v;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
  for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
  *reinterpret_cast<uint4*>(p) = v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// ---------------------------------------------------------------- RMSNorm
// h = x (+ a); y = h * rsqrt(mean(h^2) + eps) * w.  One warp per row, the row held in
// registers (NV 16-byte vectors per lane, d = 256 * NV): one HBM read of x (and a), one write
// of h and y.
template <int NV>
__global__ void __launch_bounds__(256) add_rmsnorm_fwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                              const __nv_bfloat16* __restrict__ a,
                                                              __nv_bfloat16* __restrict__ h,
                                                              __nv_bfloat16* __restrict__ y,
                                                              const __nv_bfloat16* __restrict__ w,
                                                              float* __restrict__ rstd, int T, int d, float eps) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= T) return;
  const size_t base = (size_t)row * d;
  // norm gains first: their (L2-resident) loads overlap the row loads instead of following the
  // reduction as a second dependent round trip
  uint4 wraw[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) wraw[k] = *reinterpret_cast<const uint4*>(w + (k * 32 + lane) * 8);
  float f[NV][8];
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int c = (k * 32 + lane) * 8;
    ld8(x + base + c, f[k]);
    if (a != nullptr) {
      float g[8];
      ld8(a + base + c, g);
#pragma unroll
      for (int j = 0; j < 8; ++j) f[k][j] += g[j];
      // normalise the bf16-rounded residual exactly as stored
      uint4 v;
      __nv_bfloat162* hv = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        hv[j] = __floats2bfloat162_rn(f[k][2 * j], f[k][2 * j + 1]);
        const float2 back = __bfloat1622float2(hv[j]);
        f[k][2 * j] = back.x;
        f[k][2 * j + 1] = back.y;
      }
      *reinterpret_cast<uint4*>(h + base + c) = v;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) ss += f[k][j] * f[k][j];
  }
  ss = warp_sum(ss);
  const float r = rsqrtf(ss / d + eps);
  if (lane == 0) rstd[row] = r;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int c = (k * 32 + lane) * 8;
    float g[8];
    unpack8(wraw[k], g);
#pragma unroll
    for (int j = 0; j < 8; ++j) f[k][j] = f[k][j] * r * g[j];
    st8(y + base + c, f[k]);
  }
}

// dx = dres + r * (w*dy - hn * mean(hn * w * dy)),  hn = h * r;  dw += sum_rows dy * hn.
// Warp per row, rows in registers; each lane owns fixed columns, so its dw partials stay in
// registers across all rows the warp visits and are reduced through smem once per CTA.
template <int NV>
__global__ void __launch_bounds__(256) rmsnorm_bwd_kernel(const __nv_bfloat16* __restrict__ dy,
                                                          const __nv_bfloat16* __restrict__ h,
                                                          const __nv_bfloat16* __restrict__ w,
                                                          const float* __restrict__ rstd,
                                                          const __nv_bfloat16* dres, __nv_bfloat16* dx,
                                                          float* __restrict__ dw, int T, int d) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  extern __shared__ float sdw[];
  for (int c = threadIdx.x; c < d; c += blockDim.x) sdw[c] = 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  float acc[NV][8];
  float wv[NV][8];
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    ld8(w + (k * 32 + lane) * 8, wv[k]);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[k][j] = 0.f;
  }
  if constexpr (NV <= 4) {
  // raw 16-byte vectors of the next row (dy, h, dres) are prefetched while the current row is
  // reduced, so every warp keeps 3 x NV x 16 B per lane in flight across its rows
  const int step = gridDim.x * nw;
  int row = blockIdx.x * nw + warp;
  uint4 ndy[NV], nh[NV], nres[NV];
  auto fetch = [&](int rw) {
    const size_t base = (size_t)rw * d;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int c = (k * 32 + lane) * 8;
      ndy[k] = *reinterpret_cast<const uint4*>(dy + base + c);
      nh[k] = *reinterpret_cast<const uint4*>(h + base + c);
      nres[k] = dres != nullptr ? *reinterpret_cast<const uint4*>(dres + base + c) : make_uint4(0, 0, 0, 0);
    }
  };
  if (row < T) fetch(row);
  for (; row < T; row += step) {
    const size_t base = (size_t)row * d;
    const float r = rstd[row];
    float g[NV][8], hn[NV][8], o[NV][8];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      unpack8(ndy[k], g[k]);
      unpack8(nh[k], hn[k]);
      unpack8(nres[k], o[k]);
    }
    if (row + step < T) fetch(row + step);
    float dot = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        hn[k][j] *= r;
        dot += hn[k][j] * wv[k][j] * g[k][j];
        acc[k][j] += g[k][j] * hn[k][j];
      }
    }
    dot = warp_sum(dot) / d;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int c = (k * 32 + lane) * 8;
#pragma unroll
      for (int j = 0; j < 8; ++j) o[k][j] += r * (wv[k][j] * g[k][j] - hn[k][j] * dot);
      st8(dx + base + c, o[k]);
    }
  }
  } else {  // wide rows: registers cannot hold a prefetched row as well
  for (int row = blockIdx.x * nw + warp; row < T; row += gridDim.x * nw) {
    const size_t base = (size_t)row * d;
    const float r = rstd[row];
    float g[NV][8], hn[NV][8];
    float dot = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int c = (k * 32 + lane) * 8;
      ld8(dy + base + c, g[k]);
      ld8(h + base + c, hn[k]);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        hn[k][j] *= r;
        dot += hn[k][j] * wv[k][j] * g[k][j];
        acc[k][j] += g[k][j] * hn[k][j];
      }
    }
    dot = warp_sum(dot) / d;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int c = (k * 32 + lane) * 8;
      float o[8];
      if (dres != nullptr) {
        ld8(dres + base + c, o);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] += r * (wv[k][j] * g[k][j] - hn[k][j] * dot);
      st8(dx + base + c, o);
    }
  }
  }
#pragma unroll
  for (int k = 0; k < NV; ++k)
#pragma unroll
    for (int j = 0; j < 8; ++j) atomicAdd(&sdw[(k * 32 + lane) * 8 + j], acc[k][j]);
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) atomicAdd(&dw[c], sdw[c]);
}

// ---------------------------------------------------------------- RMSNorm, any d (multiple of 8)
// h = x (+ a); y = h * rsqrt(mean(h^2) + eps) * w.  One warp per row.
__global__ void __launch_bounds__(256) rmsnorm_generic_fwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                              const __nv_bfloat16* __restrict__ a,
                                                              __nv_bfloat16* __restrict__ h,
                                                              __nv_bfloat16* __restrict__ y,
                                                              const __nv_bfloat16* __restrict__ w,
                                                              float* __restrict__ rstd, int T, int d, float eps) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= T) return;
  const size_t base = (size_t)row * d;
  float ss = 0.f;
  for (int c = lane * 8; c < d; c += 256) {
    float f[8];
    ld8(x + base + c, f);
    if (a != nullptr) {
      float g[8];
      ld8(a + base + c, g);
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] += g[j];
      st8(h + base + c, f);
      ld8(h + base + c, f);  // normalise the bf16-rounded residual, as stored
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) ss += f[j] * f[j];
  }
  ss = warp_sum(ss);
  const float r = rsqrtf(ss / d + eps);
  if (lane == 0) rstd[row] = r;
  const __nv_bfloat16* src = a != nullptr ? h : x;
  for (int c = lane * 8; c < d; c += 256) {
    float f[8], g[8];
    ld8(src + base + c, f);
    ld8(w + c, g);
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = f[j] * r * g[j];
    st8(y + base + c, f);
  }
}

// dx = dres + r * (w*dy - hn * mean(hn * w * dy)),  hn = h * r;  dw += sum_rows dy * hn
__global__ void __launch_bounds__(256) rmsnorm_generic_bwd_kernel(const __nv_bfloat16* __restrict__ dy,
                                                          const __nv_bfloat16* __restrict__ h,
                                                          const __nv_bfloat16* __restrict__ w,
                                                          const float* __restrict__ rstd,
                                                          const __nv_bfloat16* dres, __nv_bfloat16* dx,
                                                          float* __restrict__ dw, int T, int d) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  extern __shared__ float sdw[];
  for (int c = threadIdx.x; c < d; c += blockDim.x) sdw[c] = 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  for (int row = blockIdx.x * nw + warp; row < T; row += gridDim.x * nw) {
    const size_t base = (size_t)row * d;
    const float r = rstd[row];
    float dot = 0.f;
    for (int c = lane * 8; c < d; c += 256) {
      float g[8], hh[8], ww[8];
      ld8(dy + base + c, g);
      ld8(h + base + c, hh);
      ld8(w + c, ww);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float hn = hh[j] * r;
        dot += hn * ww[j] * g[j];
        atomicAdd(&sdw[c + j], g[j] * hn);
      }
    }
    dot = warp_sum(dot) / d;
    for (int c = lane * 8; c < d; c += 256) {
      float g[8], hh[8], ww[8], o[8];
      ld8(dy + base + c, g);
      ld8(h + base + c, hh);
      ld8(w + c, ww);
      if (dres != nullptr) {
        ld8(dres + base + c, o);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) o[j] += r * (ww[j] * g[j] - hh[j] * r * dot);
      st8(dx + base + c, o);
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < d; c += blockDim.x) atomicAdd(&dw[c], sdw[c]);
}

// ---------------------------------------------------------------- RoPE (rotate-half pairs)
// qk rows: [T, n_heads, dh] at row pitch `ld`; cs[pos][dh/2] = (cos, sin).  sign=+1 fwd, -1 bwd.
// Thread per (token, head), consecutive threads = consecutive tokens of one head: the token's
// head row moves as 16-byte vectors and the position-tiled (cos, sin) table is read coalesced.
__global__ void rope_kernel(__nv_bfloat16* __restrict__ qk, const int32_t* __restrict__ pos,
                            const float2* __restrict__ cs, int T, int n_heads, int dh, int ld, float sign) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  const int half = dh / 2;
  const long long total = (long long)T * n_heads;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int hd = (int)(i / T), t = (int)(i - (long long)hd * T);
    __nv_bfloat16* p = qk + (size_t)t * ld + hd * dh;
    const int pt = pos[t];
    for (int k0 = 0; k0 < half; k0 += 8) {
      uint4 va = *reinterpret_cast<const uint4*>(p + k0), vb = *reinterpret_cast<const uint4*>(p + k0 + half);
      __nv_bfloat162* a2 = reinterpret_cast<__nv_bfloat162*>(&va);
      __nv_bfloat162* b2 = reinterpret_cast<__nv_bfloat162*>(&vb);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 c0 = rope_cs_at(cs, pt, k0 + 2 * j, half), c1 = rope_cs_at(cs, pt, k0 + 2 * j + 1, half);
        const float2 a = __bfloat1622float2(a2[j]), b = __bfloat1622float2(b2[j]);
        const float s0 = c0.y * sign, s1 = c1.y * sign;
        a2[j] = __floats2bfloat162_rn(a.x * c0.x - b.x * s0, a.y * c1.x - b.y * s1);
        b2[j] = __floats2bfloat162_rn(b.x * c0.x + a.x * s0, b.y * c1.x + a.y * s1);
      }
      *reinterpret_cast<uint4*>(p + k0) = va;
      *reinterpret_cast<uint4*>(p + k0 + half) = vb;
    }
  }
}

// positions inside each packed sequence: pos[t] = t - cu[j] for cu[j] <= t < cu[j+1]
__global__ void positions_kernel(const int32_t* __restrict__ cu, int nseq, int32_t* __restrict__ pos) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  const int j = blockIdx.x;
  if (j >= nseq) return;
  const int a = cu[j], b = cu[j + 1];
  for (int t = a + threadIdx.x; t < b; t += blockDim.x) pos[t] = t - a;
}

// ---------------------------------------------------------------- SwiGLU
// gu: [T, 2F] with gate/up interleaved in 32-column blocks: block j = [g_{32j..32j+31} |
// u_{32j..32j+31}] (the layout the fused gate/up GEMM epilogue consumes); out[T, F] = silu(g)*u.
__device__ __forceinline__ long long gate_col(long long f) { return (f >> 5) * 64 + (f & 31); }

__global__ void swiglu_fwd_kernel(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ out, int T,
                                  int F) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  const long long nv = (long long)T * F / 8;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x) {
    const long long e = i * 8;
    const long long t = e / F, f = e - t * F;
    const __nv_bfloat16* rowp = gu + t * 2 * F + gate_col(f);
    float g[8], u[8], o[8];
    ld8(rowp, g);
    ld8(rowp + 32, u);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = g[j] / (1.f + __expf(-g[j])) * u[j];
    st8(out + e, o);
  }
}

__global__ void swiglu_bwd_kernel(const __nv_bfloat16* __restrict__ dout, const __nv_bfloat16* __restrict__ gu,
                                  __nv_bfloat16* __restrict__ dgu, int T, int F) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  const long long nv = (long long)T * F / 8;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x) {
    const long long e = i * 8;
    const long long t = e / F, f = e - t * F;
    const long long gc = t * 2 * F + gate_col(f);
    float d[8], g[8], u[8], dg[8], du[8];
    ld8(dout + e, d);
    ld8(gu + gc, g);
    ld8(gu + gc + 32, u);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float sg = 1.f / (1.f + __expf(-g[j]));
      du[j] = d[j] * g[j] * sg;
      dg[j] = d[j] * u[j] * sg * (1.f + g[j] * (1.f - sg));
    }
    st8(dgu + gc, dg);
    st8(dgu + gc + 32, du);
  }
}

// ---------------------------------------------------------------- embedding
__global__ void embed_fwd_kernel(const __nv_bfloat16* __restrict__ table, const int32_t* __restrict__ ids,
                                 __nv_bfloat16* __restrict__ out, int T, int d) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= T || ids[row] < 0) return;  // negative id = placeholder row filled by a scatter
  const uint4* src = reinterpret_cast<const uint4*>(table + (size_t)ids[row] * d);
  uint4* dst = reinterpret_cast<uint4*>(out + (size_t)row * d);
  for (int v = lane; v < d / 8; v += 32) dst[v] = src[v];
}

__global__ void embed_bwd_kernel(const __nv_bfloat16* __restrict__ dout, const int32_t* __restrict__ ids,
                                 float* __restrict__ dtable, int T, int d) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= T || ids[row] < 0) return;
  float* dst = dtable + (size_t)ids[row] * d;
  for (int c = lane * 8; c < d; c += 256) {
    float f[8];
    ld8(dout + (size_t)row * d + c, f);
#pragma unroll
    for (int j = 0; j < 8; ++j) atomicAdd(dst + c + j, f[j]);
  }
}

// ---------------------------------------------------------------- AdamW (flat arena)
// p (fp32 master), g (fp32 grad), m, v (fp32), pb (bf16 working copy)
__global__ void adamw_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                             float* __restrict__ v, __nv_bfloat16* __restrict__ pb, long long n, float lr, float b1,
                             float b2, float eps, float wd, float bc1, float bc2, float gscale) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  const long long n4 = n / 4;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x) {
    float4 pp = reinterpret_cast<float4*>(p)[i];
    const float4 gg = reinterpret_cast<const float4*>(g)[i];
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    float* P = &pp.x;
    const float* G = &gg.x;
    float* Mm = &mm.x;
    float* Vv = &vv.x;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float gj = G[j] * gscale;
      Mm[j] = b1 * Mm[j] + (1.f - b1) * gj;
      Vv[j] = b2 * Vv[j] + (1.f - b2) * gj * gj;
      const float upd = (Mm[j] / bc1) / (sqrtf(Vv[j] / bc2) + eps);
      P[j] -= lr * (upd + wd * P[j]);
    }
    reinterpret_cast<float4*>(p)[i] = pp;
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
    __nv_bfloat162* o = reinterpret_cast<__nv_bfloat162*>(pb + 4 * i);
    o[0] = __floats2bfloat162_rn(pp.x, pp.y);
    o[1] = __floats2bfloat162_rn(pp.z, pp.w);
  }
}

inline int grid_for(long long work, int threads) {
  long long b = (work + threads - 1) / threads;
  const long long cap = 148LL * 16;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace
}  // namespace mb

using namespace mb;

static int rmsnorm_generic_fwd(const void* x, const void* a, void* h, void* y, const void* w, float* rstd, int T,
                               int d, float eps, cudaStream_t st) {
  launch_pdl(rmsnorm_generic_fwd_kernel, dim3((T + 7) / 8), dim3(256), 0, st, (const __nv_bfloat16*)x, (const __nv_bfloat16*)a,
                                                          (__nv_bfloat16*)h, (__nv_bfloat16*)y,
                                                          (const __nv_bfloat16*)w, rstd, T, d, eps);
  return launch_status();
}

static int rmsnorm_generic_bwd(const void* dy, const void* h, const void* w, const float* rstd, const void* dres,
                               void* dx, float* dw, int T, int d, cudaStream_t st) {
  const size_t smem = (size_t)d * sizeof(float);
  if (ensure_smem<rmsnorm_generic_bwd_kernel>(smem)) return launch_status();
  // four CTAs per SM (a warp walks its rows with the full load latency per row, so rows in
  // flight per SM set the speed); 592 x d global atomics for dw at the end
  const int grid = (T + 7) / 8 < 148 * 4 ? (T + 7) / 8 : 148 * 4;
  launch_pdl(rmsnorm_generic_bwd_kernel, dim3(grid), dim3(256), smem, st, (const __nv_bfloat16*)dy, (const __nv_bfloat16*)h,
                                                      (const __nv_bfloat16*)w, rstd, (const __nv_bfloat16*)dres,
                                                      (__nv_bfloat16*)dx, dw, T, d);
  return launch_status();
}

template <int NV>
static int rmsnorm_fwd_launch(const void* x, const void* a, void* h, void* y, const void* w, float* rstd, int T, int d,
                              float eps, cudaStream_t st) {
  launch_pdl(add_rmsnorm_fwd_kernel<NV>, dim3((T + 7) / 8), dim3(256), 0, st, (const __nv_bfloat16*)x, (const __nv_bfloat16*)a,
                                                          (__nv_bfloat16*)h, (__nv_bfloat16*)y,
                                                          (const __nv_bfloat16*)w, rstd, T, d, eps);
  return launch_status();
}

template <int NV>
static int rmsnorm_bwd_launch(const void* dy, const void* h, const void* w, const float* rstd, const void* dres,
                              void* dx, float* dw, int T, int d, cudaStream_t st) {
  const size_t smem = (size_t)d * sizeof(float);
  if (ensure_smem<rmsnorm_bwd_kernel<NV>>(smem)) return launch_status();
  const int grid = T / 8 < 148 ? (T + 7) / 8 : 148;  // one CTA per SM: 148 x d atomics for dw, ~7 rows per warp
  launch_pdl(rmsnorm_bwd_kernel<NV>, dim3(grid), dim3(256), smem, st, (const __nv_bfloat16*)dy, (const __nv_bfloat16*)h,
                                                  (const __nv_bfloat16*)w, rstd, (const __nv_bfloat16*)dres,
                                                  (__nv_bfloat16*)dx, dw, T, d);
  return launch_status();
}

// register-resident fast path for d in {256 .. 4096} multiples of 256; generic path otherwise
MAESTRO_API int maestro_add_rmsnorm_fwd(const void* x, const void* a, void* h, void* y, const void* w, float* rstd,
                                        int32_t T, int32_t d, float eps, void* stream) {
  if (T <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  switch (d) {
    case 256: return rmsnorm_fwd_launch<1>(x, a, h, y, w, rstd, T, d, eps, st);
    case 512: return rmsnorm_fwd_launch<2>(x, a, h, y, w, rstd, T, d, eps, st);
    case 768: return rmsnorm_fwd_launch<3>(x, a, h, y, w, rstd, T, d, eps, st);
    case 1024: return rmsnorm_fwd_launch<4>(x, a, h, y, w, rstd, T, d, eps, st);
    case 2048: return rmsnorm_fwd_launch<8>(x, a, h, y, w, rstd, T, d, eps, st);
    case 3584: return rmsnorm_fwd_launch<14>(x, a, h, y, w, rstd, T, d, eps, st);
    case 4096: return rmsnorm_fwd_launch<16>(x, a, h, y, w, rstd, T, d, eps, st);
    default: break;
  }
  if (d % 8) return (int)cudaErrorInvalidValue;
  return rmsnorm_generic_fwd(x, a, h, y, w, rstd, T, d, eps, st);
}

MAESTRO_API int maestro_rmsnorm_bwd(const void* dy, const void* h, const void* w, const float* rstd,
                                    const void* dres, void* dx, float* dw, int32_t T, int32_t d, void* stream) {
  if (T <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  switch (d) {
    case 256: return rmsnorm_bwd_launch<1>(dy, h, w, rstd, dres, dx, dw, T, d, st);
    case 512: return rmsnorm_bwd_launch<2>(dy, h, w, rstd, dres, dx, dw, T, d, st);
    case 768: return rmsnorm_bwd_launch<3>(dy, h, w, rstd, dres, dx, dw, T, d, st);
    case 1024: return rmsnorm_bwd_launch<4>(dy, h, w, rstd, dres, dx, dw, T, d, st);
    case 2048: return rmsnorm_bwd_launch<8>(dy, h, w, rstd, dres, dx, dw, T, d, st);
    default: break;
  }
  if (d % 8) return (int)cudaErrorInvalidValue;
  return rmsnorm_generic_bwd(dy, h, w, rstd, dres, dx, dw, T, d, st);
}

MAESTRO_API int maestro_rope(void* qk, const int32_t* pos, const void* cos_sin, int32_t T, int32_t n_heads,
                             int32_t dh, int32_t ld, int32_t backward, void* stream) {
  if (T <= 0) return 0;
  if ((dh % 16) || (ld % 8)) return (int)cudaErrorInvalidValue;  // 16-byte row vectors
  const long long work = (long long)T * n_heads;
  launch_pdl(rope_kernel, dim3(grid_for(work, 256)), dim3(256), 0, (cudaStream_t)stream, 
      (__nv_bfloat16*)qk, pos, (const float2*)cos_sin, T, n_heads, dh, ld, backward ? -1.f : 1.f);
  return launch_status();
}

MAESTRO_API int maestro_positions(const int32_t* cu, int32_t nseq, int32_t* pos, void* stream) {
  if (nseq <= 0) return 0;
  launch_pdl(positions_kernel, dim3(nseq), dim3(256), 0, (cudaStream_t)stream, cu, nseq, pos);
  return launch_status();
}

MAESTRO_API int maestro_swiglu_fwd(const void* gu, void* out, int32_t T, int32_t F, void* stream) {
  if (T <= 0) return 0;
  if (F % 32) return (int)cudaErrorInvalidValue;
  launch_pdl(swiglu_fwd_kernel, dim3(grid_for((long long)T * F / 8, 256)), dim3(256), 0, (cudaStream_t)stream, 
      (const __nv_bfloat16*)gu, (__nv_bfloat16*)out, T, F);
  return launch_status();
}

MAESTRO_API int maestro_swiglu_bwd(const void* dout, const void* gu, void* dgu, int32_t T, int32_t F, void* stream) {
  if (T <= 0) return 0;
  if (F % 32) return (int)cudaErrorInvalidValue;
  launch_pdl(swiglu_bwd_kernel, dim3(grid_for((long long)T * F / 8, 256)), dim3(256), 0, (cudaStream_t)stream, 
      (const __nv_bfloat16*)dout, (const __nv_bfloat16*)gu, (__nv_bfloat16*)dgu, T, F);
  return launch_status();
}

MAESTRO_API int maestro_embed_fwd(const void* table, const int32_t* ids, void* out, int32_t T, int32_t d,
                                  void* stream) {
  if (T <= 0) return 0;
  launch_pdl(embed_fwd_kernel, dim3((T + 7) / 8), dim3(256), 0, (cudaStream_t)stream, (const __nv_bfloat16*)table, ids,
                                                                  (__nv_bfloat16*)out, T, d);
  return launch_status();
}

MAESTRO_API int maestro_embed_bwd(const void* dout, const int32_t* ids, float* dtable, int32_t T, int32_t d,
                                  void* stream) {
  if (T <= 0) return 0;
  launch_pdl(embed_bwd_kernel, dim3((T + 7) / 8), dim3(256), 0, (cudaStream_t)stream, (const __nv_bfloat16*)dout, ids, dtable, T, d);
  return launch_status();
}

// dst[c][r] = src[r][c] (bf16), 64 x 64 tiles through padded shared memory: 16-byte row loads,
// 16-byte column-gathered stores.  Used to keep K-major copies of weights for the dgrad GEMM.
__device__ __forceinline__ void transpose_tile(const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                               int rows, int cols, int ld_src, int ld_dst, int r0, int c0,
                                               __nv_bfloat16 (*tile)[64 + 8]) {
  for (int i = threadIdx.x; i < 64 * 8; i += blockDim.x) {
    const int r = i >> 3, cv = (i & 7) * 8;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r0 + r < rows && c0 + cv < cols) v = *reinterpret_cast<const uint4*>(src + (size_t)(r0 + r) * ld_src + c0 + cv);
    *reinterpret_cast<uint4*>(&tile[r][cv]) = v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 64 * 8; i += blockDim.x) {
    const int c = i >> 3, rv = (i & 7) * 8;
    if (c0 + c >= cols || r0 + rv >= rows) continue;
    __align__(16) __nv_bfloat16 o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = tile[rv + k][c];
    *reinterpret_cast<uint4*>(dst + (size_t)(c0 + c) * ld_dst + r0 + rv) = *reinterpret_cast<uint4*>(o);
  }
}

__global__ void transpose_bf16_kernel(const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                      int rows, int cols, int ld_src, int ld_dst) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  __shared__ __nv_bfloat16 tile[64][64 + 8];
  transpose_tile(src, dst, rows, cols, ld_src, ld_dst, blockIdx.y * 64, blockIdx.x * 64, tile);
}

// Many matrices in one launch (the K-major weight copies refreshed after every optimizer step:
// ~60 small matrices per section, launch-bound one by one).  desc[i] = {src, dst, rows, cols,
// ld_src, ld_dst, first tile, tiles along cols}; block b handles tile b of the concatenation.
__global__ void transpose_bf16_batched_kernel(const int64_t* __restrict__ desc, int n) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  __shared__ __nv_bfloat16 tile[64][64 + 8];
  __shared__ int s_i;
  const int b = blockIdx.x;
  if (threadIdx.x == 0) {
    int lo = 0, hi = n - 1;  // last matrix whose first tile <= b
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (desc[mid * 8 + 6] <= b) lo = mid; else hi = mid - 1;
    }
    s_i = lo;
  }
  __syncthreads();
  const int64_t* d = desc + s_i * 8;
  const int t = b - (int)d[6], tx = (int)d[7];
  transpose_tile(reinterpret_cast<const __nv_bfloat16*>(d[0]), reinterpret_cast<__nv_bfloat16*>(d[1]), (int)d[2],
                 (int)d[3], (int)d[4], (int)d[5], (t / tx) * 64, (t % tx) * 64, tile);
}

MAESTRO_API int maestro_transpose_bf16(const void* src, void* dst, int32_t rows, int32_t cols, int32_t ld_src,
                                       int32_t ld_dst, void* stream) {
  if (rows <= 0 || cols <= 0) return 0;
  if ((rows % 8) || (cols % 8) || (ld_src % 8) || (ld_dst % 8)) return (int)cudaErrorInvalidValue;
  dim3 grid((cols + 63) / 64, (rows + 63) / 64);
  launch_pdl(transpose_bf16_kernel, dim3(grid), dim3(256), 0, (cudaStream_t)stream, (const __nv_bfloat16*)src, (__nv_bfloat16*)dst, rows,
                                                                 cols, ld_src, ld_dst);
  return launch_status();
}

MAESTRO_API int maestro_transpose_bf16_batched(const int64_t* desc, int32_t n, int32_t total_tiles, void* stream) {
  if (n <= 0 || total_tiles <= 0) return 0;
  launch_pdl(transpose_bf16_batched_kernel, dim3(total_tiles), dim3(256), 0, (cudaStream_t)stream, desc, n);
  return launch_status();
}

MAESTRO_API int maestro_adamw(float* p, const float* g, float* m, float* v, void* pb, int64_t n, float lr, float b1,
                              float b2, float eps, float wd, int32_t step, float gscale, void* stream) {
  if (n <= 0) return 0;
  if (n % 4) return (int)cudaErrorInvalidValue;
  const float bc1 = 1.f - powf(b1, (float)step), bc2 = 1.f - powf(b2, (float)step);
  launch_pdl(adamw_kernel, dim3(grid_for(n / 4, 256)), dim3(256), 0, (cudaStream_t)stream, p, g, m, v, (__nv_bfloat16*)pb, n, lr, b1, b2,
                                                                        eps, wd, bc1, bc2, gscale);
  return launch_status();
}
