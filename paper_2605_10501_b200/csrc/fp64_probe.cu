// fp64 CUDA-core probes -- the denominators of the scheduler kernels' roofline (K1-K4 run fp64
// recurrences; SURVEY §8d asks for a measured fp64 add throughput, not a datasheet value).
//   mode 0: throughput -- every thread runs 8 independent add chains for `iters` steps
//   mode 1: latency    -- one thread runs one dependent add chain for `iters` steps
// The result is written to out[] so nothing is optimised away.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace mb {
namespace {

__global__ void fp64_add_throughput(double* out, int iters, double step) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = __dadd_rn(x[c], step);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  if (s == -1.0) out[blockIdx.x] = s;  // never true; keeps the chains live
}

__global__ void fp64_add_latency(double* out, int iters, double step) {
  double x = threadIdx.x;
  for (int i = 0; i < iters; ++i) x = __dadd_rn(x, step);
  out[0] = x;
}

}  // namespace
}  // namespace mb

using namespace mb;

// mode 0: launches (blocks x 256 threads x 8 chains x iters) adds; mode 1: iters dependent adds.
MAESTRO_API int maestro_fp64_probe(double* out, int32_t mode, int32_t iters, int32_t blocks, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (mode == 0)
    fp64_add_throughput<<<blocks, 256, 0, st>>>(out, iters, 1e-12);
  else
    fp64_add_latency<<<1, 1, 0, st>>>(out, iters, 1e-12);
  return launch_status();
}
