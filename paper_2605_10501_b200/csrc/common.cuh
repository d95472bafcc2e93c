// Shared device helpers for the maestro_b200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

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

}  // namespace mb
