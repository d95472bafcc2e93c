// Reshard data mover: N-d strided box copy (the device half of plan_reshard / apply_plan and of
// Endpoint.pull's fragment gather; reference mq.py:163-174, 460-469).
//
// A transfer moves a box (shape[ndim]) from a strided source view to a strided destination view.
// HBM-bound: 2 x box bytes per copy.  When the innermost dimension is contiguous on both sides and
// every row start is 16-byte aligned, each thread moves 16-byte vectors; otherwise elements.
// Work is flattened over (row, vector) so one launch covers any box shape with coalesced rows.
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "tma_host.cuh"

namespace mb {
namespace {

constexpr int MAX_DIMS = 6;

struct BoxArgs {
  const unsigned char* src;
  unsigned char* dst;
  int64_t shape[MAX_DIMS];
  int64_t ss[MAX_DIMS];  // source strides in BYTES
  int64_t ds[MAX_DIMS];  // destination strides in BYTES
  int ndim;              // >= 1; dims [0, ndim-1) are "rows", dim ndim-1 the row
  int64_t rows;
  int64_t units_per_row;  // vectors (or elements) per row
  int unit;               // bytes per unit (16 for the vector path, else the element size)
};

__device__ __forceinline__ void row_offsets(const BoxArgs& a, int64_t row, int64_t& so, int64_t& dof) {
  so = 0;
  dof = 0;
  for (int k = a.ndim - 2; k >= 0; --k) {
    const int64_t i = row % a.shape[k];
    row /= a.shape[k];
    so += i * a.ss[k];
    dof += i * a.ds[k];
  }
}

template <int UNIT>
__global__ void box_copy_kernel(const BoxArgs a) {
  const int64_t total = a.rows * a.units_per_row;
  const int64_t inner_ss = a.ss[a.ndim - 1], inner_ds = a.ds[a.ndim - 1];
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = idx / a.units_per_row, u = idx - row * a.units_per_row;
    int64_t so, dof;
    row_offsets(a, row, so, dof);
    if (UNIT == 16) {
      *reinterpret_cast<uint4*>(a.dst + dof + u * 16) = *reinterpret_cast<const uint4*>(a.src + so + u * 16);
    } else if (UNIT == 8) {
      *reinterpret_cast<uint64_t*>(a.dst + dof + u * inner_ds) = *reinterpret_cast<const uint64_t*>(a.src + so + u * inner_ss);
    } else if (UNIT == 4) {
      *reinterpret_cast<uint32_t*>(a.dst + dof + u * inner_ds) = *reinterpret_cast<const uint32_t*>(a.src + so + u * inner_ss);
    } else if (UNIT == 2) {
      *reinterpret_cast<uint16_t*>(a.dst + dof + u * inner_ds) = *reinterpret_cast<const uint16_t*>(a.src + so + u * inner_ss);
    } else {
      a.dst[dof + u * inner_ds] = a.src[so + u * inner_ss];
    }
  }
}

}  // namespace
}  // namespace mb

using namespace mb;

// dst[box] = src[box]; strides in ELEMENTS, elem_bytes in {1, 2, 4, 8}, ndim in [1, 6].
MAESTRO_API int maestro_box_copy(const void* src, const int64_t* src_strides, void* dst, const int64_t* dst_strides,
                                 const int64_t* shape, int32_t ndim, int32_t elem_bytes, void* stream) {
  if (ndim < 1 || ndim > MAX_DIMS) return (int)cudaErrorInvalidValue;
  if (elem_bytes != 1 && elem_bytes != 2 && elem_bytes != 4 && elem_bytes != 8) return (int)cudaErrorInvalidValue;
  BoxArgs a;
  a.src = reinterpret_cast<const unsigned char*>(src);
  a.dst = reinterpret_cast<unsigned char*>(dst);
  a.ndim = ndim;
  a.rows = 1;
  for (int k = 0; k < ndim; ++k) {
    if (shape[k] < 0) return (int)cudaErrorInvalidValue;
    if (shape[k] == 0) return 0;
    a.shape[k] = shape[k];
    a.ss[k] = src_strides[k] * elem_bytes;
    a.ds[k] = dst_strides[k] * elem_bytes;
    if (k < ndim - 1) a.rows *= shape[k];
  }
  const int64_t inner = shape[ndim - 1];
  const int64_t row_bytes = inner * elem_bytes;
  bool vec = src_strides[ndim - 1] == 1 && dst_strides[ndim - 1] == 1 && row_bytes % 16 == 0 &&
             (reinterpret_cast<uintptr_t>(src) % 16) == 0 && (reinterpret_cast<uintptr_t>(dst) % 16) == 0;
  for (int k = 0; vec && k < ndim - 1; ++k) vec = (a.ss[k] % 16) == 0 && (a.ds[k] % 16) == 0;
  a.unit = vec ? 16 : elem_bytes;
  a.units_per_row = vec ? row_bytes / 16 : inner;
  const int64_t total = a.rows * a.units_per_row;
  const int64_t want = (total + 255) / 256;
  const int grid = (int)(want < (int64_t)num_sms() * 8 ? want : (int64_t)num_sms() * 8);
  cudaStream_t st = (cudaStream_t)stream;
  switch (a.unit) {
    case 16: box_copy_kernel<16><<<grid, 256, 0, st>>>(a); break;
    case 8: box_copy_kernel<8><<<grid, 256, 0, st>>>(a); break;
    case 4: box_copy_kernel<4><<<grid, 256, 0, st>>>(a); break;
    case 2: box_copy_kernel<2><<<grid, 256, 0, st>>>(a); break;
    default: box_copy_kernel<1><<<grid, 256, 0, st>>>(a); break;
  }
  return launch_status();
}

// Upper bound on the SMs persistent grids (GEMM, attention, box copy) may use; 0 = all.
MAESTRO_API int maestro_set_sm_budget(int32_t n_sms) {
  if (n_sms < 0) return (int)cudaErrorInvalidValue;
  sm_budget() = n_sms;
  return 0;
}

// Programmatic dependent launch of the step kernels on (1) or off (0); returns the previous
// setting.  Executors that run several sections' streams concurrently turn it off: a dependent
// kernel's early CTAs hold SMs the other streams could use (cfg 3/4: -1 % with it on).
MAESTRO_API int maestro_set_pdl(int32_t on) {
  const int prev = pdl_flag();
  pdl_flag() = on ? 1 : 0;
  return prev;
}
