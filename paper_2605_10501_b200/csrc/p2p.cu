// One-sided NVLink handoff primitives (the device transport behind mq.PeerTransport, C1).
//
// A receiver exports a slot arena and one 32-bit flag per slot through CUDA IPC; the sender maps
// them once.  A send is three stream-ordered operations on the sender's stream:
//   wait   credit >= seq - slots + 1      (the receiver released the slot's previous message)
//   copy   payload -> peer slot            (copy engine over NVLink, no SM involvement)
//   write  peer flag[slot] = seq + 1       (driver stream memory op, after the copy + a barrier)
// and a receive is: wait flag[slot] >= seq + 1, consume, write the sender's credit = seq + 1.
// Neither side runs a kernel that spins on another GPU, so persistent compute grids keep every
// SM (an NCCL point-to-point kernel waiting for its peer holds SMs for the whole wait).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "common.cuh"

namespace mb {
namespace {

typedef CUresult (*WaitValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*WriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

template <typename F>
F driver_fn(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(fn);
}

WaitValue32Fn wait_fn() {
  static WaitValue32Fn f = driver_fn<WaitValue32Fn>("cuStreamWaitValue32");
  return f;
}
WriteValue32Fn write_fn() {
  static WriteValue32Fn f = driver_fn<WriteValue32Fn>("cuStreamWriteValue32");
  return f;
}

}  // namespace
}  // namespace mb

using namespace mb;

// 64-byte CUDA IPC handle of the allocation containing dev_ptr (export side).
MAESTRO_API int maestro_ipc_get_handle(const void* dev_ptr, void* handle_out) {
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr));
  if (e != cudaSuccess) return (int)e;
  memcpy(handle_out, &h, sizeof(h));
  return 0;
}

// Map a peer process's allocation; *dev_ptr_out is usable by copies and stream memory ops.
MAESTRO_API int maestro_ipc_open_handle(const void* handle, void** dev_ptr_out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  return (int)cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
}

MAESTRO_API int maestro_ipc_close(void* dev_ptr) { return (int)cudaIpcCloseMemHandle(dev_ptr); }

// Stream waits until the 32-bit word at dev_addr is >= value (wrap-around compare); no kernel.
MAESTRO_API int maestro_stream_wait_geq(void* stream, const void* dev_addr, uint32_t value) {
  WaitValue32Fn f = wait_fn();
  if (f == nullptr) return (int)cudaErrorNotSupported;
  const CUresult r = f((CUstream)stream, (CUdeviceptr)dev_addr, value, CU_STREAM_WAIT_VALUE_GEQ);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorLaunchFailure;
}

// Stream writes value to the 32-bit word at dev_addr (local or peer memory) after all earlier
// work of the stream, behind a memory barrier (so a preceding copy is visible first).
MAESTRO_API int maestro_stream_write(void* stream, void* dev_addr, uint32_t value) {
  WriteValue32Fn f = write_fn();
  if (f == nullptr) return (int)cudaErrorNotSupported;
  const CUresult r = f((CUstream)stream, (CUdeviceptr)dev_addr, value, CU_STREAM_WRITE_VALUE_DEFAULT);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorLaunchFailure;
}

// Async copy between any two device addresses (peer allocations included) on the copy engine.
MAESTRO_API int maestro_copy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes <= 0) return 0;
  return (int)cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, (cudaStream_t)stream);
}

// Zero-initialised device allocation owned by the caller (IPC-exportable: its own base pointer).
MAESTRO_API int maestro_device_alloc(int64_t bytes, void** dev_ptr_out) {
  cudaError_t e = cudaMalloc(dev_ptr_out, (size_t)bytes);
  if (e != cudaSuccess) return (int)e;
  return (int)cudaMemset(*dev_ptr_out, 0, (size_t)bytes);
}

MAESTRO_API int maestro_device_free(void* dev_ptr) { return (int)cudaFree(dev_ptr); }
