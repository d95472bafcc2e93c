// Shared device helpers for the maestro_b200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "maestro_b200.h"

#define MAESTRO_API extern "C" __attribute__((visibility("default")))

namespace mb {

constexpr unsigned kFull = 0xffffffffu;

// splitmix64 finaliser; must match paper_2605_10501_b200/synthetic.py
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Fold one domain error into the device error word (min = earliest in reference raise order).
__device__ __forceinline__ void report(int64_t* err, uint32_t prio, int code, int index) {
  if (err == nullptr) return;
  long long key = ((long long)prio << 32) | ((long long)(code & 0xff) << 24) | (long long)(index & 0xffffff);
  atomicMin(reinterpret_cast<long long*>(err), key);
}

inline int launch_status() { return (int)cudaGetLastError(); }

// ---- programmatic dependent launch (PDL)
// A kernel launched with cudaLaunchAttributeProgrammaticStreamSerialization may start (and run its
// prologue) while the previous kernel on the stream is still finishing; pdl_wait() blocks until
// that kernel has completed and its writes are visible (a no-op for a normal launch).  pdl_trigger()
// lets the next dependent kernel launch once every CTA of this one has executed it.  Every kernel
// launched through launch_pdl() calls pdl_wait() before its first global-memory access.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

inline int& pdl_flag() {  // MAESTRO_PDL=0 or maestro_set_pdl(0): ordinary stream serialisation
  static int v = [] {
    const char* e = getenv("MAESTRO_PDL");
    return e ? atoi(e) : 1;
  }();
  return v;
}
inline bool pdl_enabled() { return pdl_flag() != 0; }

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// Raise a kernel's dynamic shared-memory limit to `bytes` if needed (idempotent, cached
// per kernel).  Returns nonzero on failure (the error stays queued for launch_status()).
template <auto KERNEL>
inline int ensure_smem(size_t bytes) {
  static size_t configured = 0;  // one instance per kernel
  if (bytes <= 48 * 1024 || bytes <= configured) return 0;
  cudaError_t e = cudaFuncSetAttribute(KERNEL, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return (int)e;
  configured = bytes;
  return 0;
}

// RoPE (cos, sin) table, position-tiled: [ceil(P/32)][half][32][2] fp32 -- for a fixed
// frequency k, 32 consecutive positions are contiguous, so a warp whose lanes own consecutive
// rows reads one 256-byte segment per frequency (transformer.rope_table builds it).
__device__ __forceinline__ float2 rope_cs_at(const float2* __restrict__ cs, int pos, int k, int half) {
  return cs[((size_t)(pos >> 5) * half + k) * 32 + (pos & 31)];
}

// 2^x for a pair on the FMA pipe (the MUFU unit retires 16 exponentials per clock per SM, the
// FMA pipe 128 lanes): round-to-nearest split x = n + f with the 1.5*2^23 magic constant, a
// minimax polynomial for 2^f on [-1/2, 1/2] in paired fp32 FMAs, n added to the exponent field.
// x is clamped at -126 so -inf (masked) inputs give ~0.  DEG 3: max relative error 7.5e-5 (P is
// rounded to bf16 anyway); DEG 5: 1.3e-7 (on par with ex2.approx, for fp32 reductions).
template <int DEG>
__device__ __forceinline__ float2 ex2_fma2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 j = __fadd2_rn(x, make_float2(12582912.f, 12582912.f));
  const float2 r = __fadd2_rn(j, make_float2(-12582912.f, -12582912.f));
  const float2 f = __ffma2_rn(r, make_float2(-1.f, -1.f), x);
  float2 p;
  if constexpr (DEG == 3) {
    p = __ffma2_rn(make_float2(0.05516102f, 0.05516102f), f, make_float2(0.24261291f, 0.24261291f));
    p = __ffma2_rn(p, f, make_float2(0.6932625f, 0.6932625f));
    p = __ffma2_rn(p, f, make_float2(0.99992794f, 0.99992794f));
  } else {
    p = __ffma2_rn(make_float2(0.00134518f, 0.00134518f), f, make_float2(0.00968204f, 0.00968204f));
    p = __ffma2_rn(p, f, make_float2(0.05550102f, 0.05550102f));
    p = __ffma2_rn(p, f, make_float2(0.24021935f, 0.24021935f));
    p = __ffma2_rn(p, f, make_float2(0.6931473f, 0.6931473f));
    p = __ffma2_rn(p, f, make_float2(1.0000001f, 1.0000001f));
  }
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(j.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(j.y) << 23)));
}

}  // namespace mb
