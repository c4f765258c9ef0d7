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

int pdl_allowed() {
  static const int v = std::getenv("SPIN_NO_PDL") != nullptr ? 0 : 1;
  return v;
}

}  // namespace spin
