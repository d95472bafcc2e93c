// Microbenchmark: tcgen05.mma cycles per instruction for the attention-backward shapes, with zero
// vs random operands (tensor-core power depends on the data), K-major vs MN-major operands.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_10501_b200/csrc scripts/micro/umma_rate2.cu -o scripts/micro/umma_rate2
#include <cstdio>
#include <cstdlib>
constexpr int SMEM_DATA = 196608;
#include "sm100.cuh"
using namespace mb::sm100;

#ifndef N_MMA
#define N_MMA 4096
#endif

// MODE 0: SS N128 K-major (S^T, dP^T); 1: TS N64, B MN-major (dV, dK); 2: SS N64 A,B MN-major (dQ)
// MODE 3: one backward iteration's mix (4 S + 4 dP + 8 dV + 8 dK + 8 dQ = 32 MMAs) with commits;
// MODE 4: the same mix without commits; MODE 5: mix of SS N128 and TS N64 only (no MN-major A)
template <int MODE>
__global__ void __launch_bounds__(128, 1) rate_kernel(long long* out, int rnd) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = align_smem_1024(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + SMEM_DATA);
  uint64_t* dummy = bar + 2;  // [4] commit targets nobody waits on
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5;
  uint32_t st = 0x12345u + threadIdx.x * 7919u + blockIdx.x * 104729u;
  for (int i = threadIdx.x; i < SMEM_DATA / 4; i += blockDim.x) {
    st = st * 1664525u + 1013904223u;
    // random bf16 pairs in [-1, 1): sign | exponent 0x3F0..0x3F7 | random mantissa
    const uint32_t lo = ((st >> 16) & 0x807F) | 0x3F00, hi = ((st & 0x807F) | 0x3F00);
    reinterpret_cast<uint32_t*>(sm)[i] = rnd ? (lo | (hi << 16)) : 0u;
  }
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&dummy[i], 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(slot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (rnd) {  // random A operand in TMEM columns [0, 64) for the TS mode
    uint32_t r[32];
    for (int c = 0; c < 64; c += 32) {
      for (int i = 0; i < 32; ++i) { st = st * 1664525u + 1013904223u; r[i] = ((st >> 16) & 0x807F) | 0x3F00 | ((((st & 0x807F) | 0x3F00)) << 16); }
      tmem_st_32x32b_x32(tmem + ((uint32_t)(warp * 32) << 16) + c, r);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    const uint32_t base = smem_u32(sm);
    long long t0 = clock64();
    if (MODE >= 3 && elect_one()) {
      constexpr bool FENCE = MODE == 6;
      const uint32_t base0 = base;
      const uint32_t id_sp = idesc_bf16_f32(128, 128, false, false), id_kv = idesc_bf16_f32(128, 64, false, true),
                     id_dq = idesc_bf16_f32(128, 64, true, true);
      for (int i = 0; i < N_MMA; i += 32) {
        const uint32_t base = MODE == 7 ? base0 + ((i >> 5) % 3) * 65536 : base0;  // rotate operand stages
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(tmem + 0, smem_desc_sw128(base + kk * 32, 16, 1024), smem_desc_sw128(base + 16384 + kk * 32, 16, 1024), id_sp, kk > 0);
        if (MODE == 3) umma_commit(&dummy[0]);
        if (FENCE) tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16_ts(tmem + 256, tmem + 448 + kk * 8, smem_desc_sw128(base + 32768 + kk * 2048, 8192, 1024), id_kv, 1u);
        if (MODE == 3) umma_commit(&dummy[1]);
        if (FENCE) tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16_ts(tmem + 320, tmem + 128 + (kk >> 2) * 64 + (kk & 3) * 8, smem_desc_sw128(base + 32768 + kk * 2048, 8192, 1024), id_kv, 1u);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (MODE == 5)
            umma_bf16_ts(tmem + 384, tmem + 448 + kk * 8, smem_desc_sw128(base + 32768 + kk * 2048, 8192, 1024), id_kv, 1u);
          else
            umma_bf16(tmem + 384, smem_desc_sw128(base + kk * 2048, 16384, 1024), smem_desc_sw128(base + 32768 + kk * 2048, 8192, 1024), id_dq, kk > 0);
        }
        if (MODE == 3) { umma_commit(&dummy[2]); umma_commit(&dummy[3]); umma_commit(&dummy[0]); }
        if (FENCE) tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          umma_bf16(tmem + 128, smem_desc_sw128(base + 32768 + kk * 32, 16, 1024), smem_desc_sw128(base + 49152 + kk * 32, 16, 1024), id_sp, kk > 0);
        if (MODE == 3) umma_commit(&dummy[1]);
      }
      umma_commit(bar);
    } else if (MODE < 3 && elect_one()) {
      for (int i = 0; i < N_MMA; i += 8) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (MODE == 0)
            umma_bf16(tmem + 256, smem_desc_sw128(base + (kk & 3) * 32, 16, 1024),
                      smem_desc_sw128(base + 16384 + (kk & 3) * 32, 16, 1024), idesc_bf16_f32(128, 128, false, false),
                      1u);
          else if (MODE == 1)
            umma_bf16_ts(tmem + 256, tmem + kk * 8, smem_desc_sw128(base + 32768 + kk * 2048, 8192, 1024),
                         idesc_bf16_f32(128, 64, false, true), 1u);
          else
            umma_bf16(tmem + 256, smem_desc_sw128(base + kk * 2048, 16384, 1024),
                      smem_desc_sw128(base + 32768 + kk * 2048, 8192, 1024), idesc_bf16_f32(128, 64, true, true), 1u);
        }
      }
      umma_commit(bar);
    }
    __syncwarp();
    mbar_wait(bar, 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int MODE>
void run(const char* name, long long* d, int rnd) {
  cudaFuncSetAttribute(rate_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_DATA + 2048);
  const int reps = getenv("REPS") ? atoi(getenv("REPS")) : 3;
  for (int rep = 0; rep < reps; ++rep) rate_kernel<MODE><<<148, 128, SMEM_DATA + 2048>>>(d, rnd);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  printf("%-36s %-6s %s cycles/MMA = %.1f\n", name, rnd ? "random" : "zeros", cudaGetErrorString(e), s / 148 / N_MMA);
}

int main() {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 148);
  if (getenv("ONLYMIX")) {
    run<4>("bwd mix, random, long", d, 1);
    return 0;
  }
  for (int rnd = 0; rnd < 2; ++rnd) {
    run<0>("SS M128 N128 K-major (S, dP)", d, rnd);
    run<1>("TS M128 N64 B MN-major (dV, dK)", d, rnd);
    run<2>("SS M128 N64 A,B MN-major (dQ)", d, rnd);
    run<3>("bwd mix + commits (per MMA; 32/iter)", d, rnd);
    run<4>("bwd mix, no commits", d, rnd);
    run<5>("mix without MN-major-A dQ", d, rnd);
    run<6>("bwd mix + fence::after_thread_sync", d, rnd);
    run<7>("bwd mix, operands rotating over 3 stages", d, rnd);
  }
  return 0;
}
