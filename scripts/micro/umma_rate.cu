// Microbenchmark: issue rate of single-CTA tcgen05.mma shapes (SS vs TS operands) on one SM per
// CTA, all SMs busy.  Cycles per MMA instruction for N_MMA back-to-back MMAs (accumulating).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_10501_b200/csrc scripts/micro/umma_rate.cu -o umma_rate
#include <cstdio>
#include "sm100.cuh"
using namespace mb::sm100;

constexpr int N_MMA = 2048;

template <int MODE>  // 0: SS N128, 1: SS N64, 2: SS N256, 3: TS N64, 4: TS N128, 5: SS N64 (B MN-major), 6: TS N256
__global__ void __launch_bounds__(128, 1) rate_kernel(long long* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = align_smem_1024(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 65536);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); }
  if (warp == 1) tmem_alloc(slot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 0) {
    constexpr int N = (MODE == 1 || MODE == 3 || MODE == 5) ? 64 : (MODE == 2 || MODE == 6) ? 256 : 128;
    constexpr uint32_t idesc = idesc_bf16_f32(128, N, false, MODE == 5);
    const uint32_t base = smem_u32(sm);
    long long t0 = clock64();
    if (elect_one()) {
      for (int i = 0; i < N_MMA; i += 4) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint64_t bd = smem_desc_sw128(base + 32768 + kk * 32, MODE == 5 ? 8192 : 16, 1024);
          if (MODE == 3 || MODE == 4 || MODE == 6)
            umma_bf16_ts(tmem + 256, tmem + kk * 8, bd, idesc, 1u);
          else
            umma_bf16(tmem + (MODE == 2 ? 0 : 256), smem_desc_sw128(base + kk * 32, 16, 1024), bd, idesc, 1u);
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
void run(const char* name, long long* d, int nblk) {
  cudaFuncSetAttribute(rate_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 2048);
  for (int rep = 0; rep < 2; ++rep) rate_kernel<MODE><<<nblk, 128, 65536 + 2048>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(long long) * nblk, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < nblk; ++i) s += h[i];
  printf("%-28s %s cycles/MMA = %.1f\n", name, cudaGetErrorString(e), s / nblk / N_MMA);
}

int main() {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 148);
  run<0>("SS M128 N128 K16", d, 148);
  run<1>("SS M128 N64 K16", d, 148);
  run<2>("SS M128 N256 K16", d, 148);
  run<5>("SS M128 N64 K16 (B MN-major)", d, 148);
  run<3>("TS M128 N64 K16", d, 148);
  run<4>("TS M128 N128 K16", d, 148);
  run<6>("TS M128 N256 K16", d, 148);
  return 0;
}
