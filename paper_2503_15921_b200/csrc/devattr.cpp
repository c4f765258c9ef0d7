// Per-device kernel attribute bookkeeping (gemm.cuh ensure_smem_optin).
#include <cuda_runtime.h>

#include <cstdlib>

#include <map>
#include <mutex>
#include <utility>

#include "gemm.cuh"

namespace spin {

cudaError_t ensure_smem_optin(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  const cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{kernel, dev}];
  if (bytes <= have) return cudaSuccess;
  const cudaError_t r = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  if (r == cudaSuccess) have = bytes;
  return r;
}

// A synchronous cudaMemcpy from pageable host memory returns once the source is staged; the
// DMA into device memory is ordered only on the legacy default stream, which the engine's
// non-blocking streams do not wait for. Uploads read by kernels on those streams go through
// here: a non-blocking stream per device, synchronised before returning.
// cudaMemset of device memory is likewise asynchronous on the legacy stream (zero_sync).
static cudaError_t on_upload_stream(void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return cudaSuccess;
  static std::mutex mu;
  static std::map<int, cudaStream_t> streams;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  cudaStream_t& s = streams[dev];
  if (!s && (e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)) != cudaSuccess) return e;
  e = src ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s) : cudaMemsetAsync(dst, 0, bytes, s);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(s);
}

cudaError_t upload_sync(void* dst, const void* src, size_t bytes) { return on_upload_stream(dst, src, bytes); }
cudaError_t zero_sync(void* dst, size_t bytes) { return on_upload_stream(dst, nullptr, bytes); }

int pdl_allowed() {
  static const int v = std::getenv("SPIN_NO_PDL") != nullptr ? 0 : 1;
  return v;
}

}  // namespace spin
