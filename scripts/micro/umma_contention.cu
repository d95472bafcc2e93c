// Microbenchmark: tcgen05.mma issue rate (TS M128 N64 K16 and SS M128 N128 K16) while 8 other
// warps load TMEM (tcgen05.ld 32x32b.x32), store TMEM, or read shared memory -- is the tensor
// pipe slowed by concurrent TMEM / SMEM traffic?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_10501_b200/csrc scripts/micro/umma_contention.cu -o scripts/micro/umma_contention
#include <cstdio>
#include "sm100.cuh"
using namespace mb::sm100;

constexpr int N_MMA = 65536;

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,"
      "%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// MMA: 0 = TS N64, 1 = SS N128.  LOAD: 0 none, 1 TMEM ld, 2 TMEM st, 3 LDS.128, 4 STS.128
template <int MMA, int LOAD>
__global__ void __launch_bounds__(320, 1) k(long long* out, int* sink) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = align_smem_1024(smem_raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 98304);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  volatile int* stop = reinterpret_cast<volatile int*>(bar + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 98304 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); *stop = 0; }
  if (warp == 1) tmem_alloc(slot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 0) {
    const uint32_t base = smem_u32(sm);
    long long t0 = clock64();
    if (elect_one()) {
      for (int i = 0; i < N_MMA; i += 4) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if (MMA == 0)
            umma_bf16_ts(tmem + 256, tmem + kk * 8, smem_desc_sw128(base + 32768 + kk * 2048, 8192, 1024),
                         idesc_bf16_f32(128, 64, false, true), 1u);
          else
            umma_bf16(tmem + 256, smem_desc_sw128(base + kk * 32, 16, 1024), smem_desc_sw128(base + 16384 + kk * 32, 16, 1024),
                      idesc_bf16_f32(128, 128, false, false), 1u);
        }
      }
      umma_commit(bar);
    }
    __syncwarp();
    mbar_wait(bar, 0);
    long long t1 = clock64();
    if (lane == 0) { out[blockIdx.x] = t1 - t0; *stop = 1; }
  } else if (warp >= 2) {
    const uint32_t lb = (uint32_t)((warp & 3) * 32) << 16;
    int acc = 0;
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = i;
    while (!*stop) {
      if (LOAD == 1) {
        tmem_ld32(tmem + lb + 128 + ((warp >> 2) & 1) * 32, r);
        acc += r[lane & 31];
      } else if (LOAD == 2) {
        tmem_st_32x32b_x32(tmem + lb + 128 + ((warp >> 2) & 1) * 32, r);
        tmem_st_wait();
      } else if (LOAD == 3) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint4 v = *reinterpret_cast<const uint4*>(sm + 65536 + ((warp * 8 + u) * 512 + lane * 16) % 32768);
          acc += v.x;
        }
      } else if (LOAD == 4) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          *reinterpret_cast<uint4*>(sm + 65536 + ((warp * 8 + u) * 512 + lane * 16) % 32768) = make_uint4(acc, u, 0, 0);
      } else if (LOAD == 5) {  // ALU + MUFU heavy (softmax-like power draw)
        float x = __uint_as_float(r[lane]) * 1e-3f;
#pragma unroll
        for (int u = 0; u < 64; ++u) {
          float y;
          asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
          x = fmaf(y, 0.999f, -0.5f);
        }
        acc += __float_as_uint(x);
      } else {
        break;
      }
    }
    if (acc == 12345) sink[0] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int MMA, int LOAD>
void run(const char* name, long long* d, int* sink) {
  const int smem = 98304 + 2048;
  cudaFuncSetAttribute(k<MMA, LOAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) k<MMA, LOAD><<<148, 320, smem>>>(d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  printf("%-40s %s cycles/MMA = %.1f\n", name, cudaGetErrorString(e), s / 148 / N_MMA);
}

int main() {
  long long* d;
  int* sink;
  cudaMalloc(&d, sizeof(long long) * 148);
  cudaMalloc(&sink, 64);
  run<0, 0>("TS N64 alone", d, sink);
  run<0, 1>("TS N64 + 8 warps TMEM ld", d, sink);
  run<0, 2>("TS N64 + 8 warps TMEM st", d, sink);
  run<0, 3>("TS N64 + 8 warps LDS.128", d, sink);
  run<0, 4>("TS N64 + 8 warps STS.128", d, sink);
  run<1, 0>("SS N128 alone", d, sink);
  run<1, 1>("SS N128 + 8 warps TMEM ld", d, sink);
  run<1, 2>("SS N128 + 8 warps TMEM st", d, sink);
  run<1, 3>("SS N128 + 8 warps LDS.128", d, sink);
  run<1, 4>("SS N128 + 8 warps STS.128", d, sink);
  run<0, 5>("TS N64 + 8 warps FMA+MUFU", d, sink);
  run<1, 5>("SS N128 + 8 warps FMA+MUFU", d, sink);
  return 0;
}
