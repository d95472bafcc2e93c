// K5b: handoff (scatter) indices between a producer section's row buffer and the critical
// section's packed varlen token stream -- north_star item (2): modality-encoder outputs land in
// the backbone's packed stream at placeholder positions (the 2x2-merged visual
// tokens are concatenated with the text tokens), computed on device from the schedule's orders.
//
//   producer order  up[nu]       samples in the producer section's (fan-out merged) order; the
//                                producer writes sample up[j]'s rows[i] output rows contiguously,
//                                in that order, into one row buffer
//   consumer order  crit[n]      the critical rank's order, packed by varlen_pack: sample crit[k]
//                                starts at token tok_off[k]; micro-batch m = positions [m*mbs, ...)
//   rows[B], dst_off[B]          per sample id: rows it exchanges (0 = not activated) and the
//                                offset of those rows inside its own sequence (the placeholder)
//
// Output pairs for every consumer position k (sample i) and r < rows[i], at index pos[k] + r:
//   src = row of the producer buffer          = (sum of rows[] of the samples before i in up[]) + r
//   dst = row inside consumer micro-batch k/mbs = tok_off[k] - tok_off[(k/mbs)*mbs] + dst_off[i] + r
// pos[n+1] is the exclusive scan of rows[] over the consumer order, so micro-batch m's pairs are
// [pos[m*mbs], pos[min(n, (m+1)*mbs)]).  A sample activated in the consumer order but missing from
// the producer order is a schedule inconsistency (error word, code of InconsistentSchedule).
#include "common.cuh"

namespace mb {
namespace {

// Exclusive block-wide scan of one int per thread (1024 threads); returns the block total.
__device__ __forceinline__ int block_exclusive_scan(int v, int* ws, int& excl) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) ws[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    const int x0 = lane < nw ? ws[lane] : 0;
    int x = x0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane < nw) ws[lane] = x - x0;
    if (lane == 31) ws[32] = x;
  }
  __syncthreads();
  excl = ws[warp] + incl - v;
  const int total = ws[32];
  __syncthreads();
  return total;
}

// One block: producer row offsets per sample id (scratch up_off[B], -1 = absent), then the
// consumer-order scan pos[].
__global__ void __launch_bounds__(1024) handoff_scan_kernel(const int32_t* __restrict__ up, int nu,
                                                            const int32_t* __restrict__ crit, int n,
                                                            const int32_t* __restrict__ rows, int B,
                                                            int32_t* __restrict__ up_off, int32_t* __restrict__ pos,
                                                            int64_t* __restrict__ err) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  __shared__ int ws[33];
  for (int i = threadIdx.x; i < B; i += blockDim.x) up_off[i] = -1;
  __syncthreads();
  int carry = 0;
  for (int j0 = 0; j0 < nu; j0 += blockDim.x) {
    const int j = j0 + threadIdx.x;
    const int v = j < nu ? rows[up[j]] : 0;
    int excl;
    const int tot = block_exclusive_scan(v, ws, excl);
    if (j < nu) up_off[up[j]] = carry + excl;
    carry += tot;
  }
  __syncthreads();
  carry = 0;
  for (int k0 = 0; k0 < n; k0 += blockDim.x) {
    const int k = k0 + threadIdx.x;
    const int i = k < n ? crit[k] : 0;
    const int v = k < n ? rows[i] : 0;
    int excl;
    const int tot = block_exclusive_scan(v, ws, excl);
    if (k < n) {
      pos[k] = carry + excl;
      if (v > 0 && up_off[i] < 0) report(err, 6, 7, k);  // activated but not produced
    }
    carry += tot;
  }
  if (threadIdx.x == 0) pos[n] = carry;
}

// One block per consumer position: its rows' (src, dst) pairs (16-byte vector stores when aligned
// would not pay: a sample's pairs are a few KB).
__global__ void handoff_fill_kernel(const int32_t* __restrict__ crit, int n, const int32_t* __restrict__ tok_off,
                                    int mbs, const int32_t* __restrict__ rows, const int32_t* __restrict__ dst_off,
                                    const int32_t* __restrict__ up_off, const int32_t* __restrict__ pos,
                                    int32_t* __restrict__ src_rows, int32_t* __restrict__ dst_rows) {
  pdl_wait();  // programmatic dependent launch (launch_pdl): previous kernel done
  pdl_trigger();
  for (int k = blockIdx.x; k < n; k += gridDim.x) {
    const int i = crit[k];
    const int nr = rows[i];
    if (nr <= 0 || up_off[i] < 0) continue;
    const int base_dst = tok_off[k] - tok_off[(k / mbs) * mbs] + dst_off[i];
    const int base_src = up_off[i];
    const int o = pos[k];
    for (int r = threadIdx.x; r < nr; r += blockDim.x) {
      src_rows[o + r] = base_src + r;
      dst_rows[o + r] = base_dst + r;
    }
  }
}

}  // namespace
}  // namespace mb

using namespace mb;

MAESTRO_API int maestro_handoff_index(const int32_t* d_up_order, int32_t nu, const int32_t* d_crit_order, int32_t n,
                                      const int32_t* d_tok_off, int32_t mbs, const int32_t* d_rows,
                                      const int32_t* d_dst_off, int32_t B, int32_t* d_scratch, int32_t* d_pos,
                                      int32_t* d_src_rows, int32_t* d_dst_rows, int64_t* d_err, void* stream) {
  if (n < 0 || nu < 0 || B <= 0 || mbs <= 0) return (int)cudaErrorInvalidValue;
  cudaStream_t st = (cudaStream_t)stream;
  launch_pdl(handoff_scan_kernel, dim3(1), dim3(1024), 0, st, d_up_order, nu, d_crit_order, n, d_rows, B, d_scratch, d_pos, d_err);
  if (n > 0)
    launch_pdl(handoff_fill_kernel, dim3(n < 1024 ? n : 1024), dim3(128), 0, st, d_crit_order, n, d_tok_off, mbs, d_rows, d_dst_off,
                                                             d_scratch, d_pos, d_src_rows, d_dst_rows);
  return launch_status();
}
