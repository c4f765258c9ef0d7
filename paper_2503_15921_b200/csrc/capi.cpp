// extern "C" entry points of libspin.so (declared in include/spin_c.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "gemm.cuh"
#include "pack.hpp"
#include "spin_c.h"
#include "status.hpp"

namespace spin {
namespace {
thread_local std::string g_last_error;
int num_sms_cached() {
  static int n = [] {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
  }();
  return n;
}
}  // namespace
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace spin

using namespace spin;

extern "C" {

int spin_abi_version(void) { return SPIN_ABI_VERSION; }
const char* spin_last_error(void) { return g_last_error.c_str(); }

spin_status spin_pack(const int32_t* kv_lens, int32_t n, int32_t width, int32_t* length, int32_t* rows,
                      spin_segment* segments, int32_t seg_cap, int32_t* n_segments, int64_t* padding_tokens,
                      int32_t* q_replica_rows) {
  return guarded([&] {
    if (n < 0 || (n > 0 && kv_lens == nullptr)) fail(SPIN_INPUT_ERROR, "spin_pack: bad input arrays");
    const PackResult p = pack_lengths(kv_lens, n, width);
    if (static_cast<int32_t>(p.segments.size()) > seg_cap)
      fail(SPIN_SIZE_ERROR, "spin_pack: segment buffer too small");
    if (length) *length = p.length;
    if (rows) *rows = p.rows;
    if (n_segments) *n_segments = static_cast<int32_t>(p.segments.size());
    if (padding_tokens) *padding_tokens = p.padding;
    if (segments && !p.segments.empty())
      std::memcpy(segments, p.segments.data(), p.segments.size() * sizeof(spin_segment));
    if (q_replica_rows && n > 0) std::memcpy(q_replica_rows, p.q_replica_rows.data(), n * sizeof(int32_t));
  });
}

spin_status spin_naive_padding(const int32_t* kv_lens, int32_t n, int64_t* padding) {
  return guarded([&] { *padding = naive_padding_of(kv_lens, n); });
}

spin_status spin_verify_batch_cost(const int32_t* kv_lens, int32_t n, int32_t window, int32_t packing,
                                   int32_t pack_width, int64_t* tokens, int64_t* padding) {
  return guarded([&] {
    const VerifyCost c = verify_cost(kv_lens, n, window, packing != 0, pack_width);
    *tokens = c.tokens;
    *padding = c.padding;
  });
}

spin_status spin_gemm_info(int32_t n_out, int32_t k, int32_t t, int32_t mode, int32_t* max_pieces, int32_t* grid,
                           int32_t* bn) {
  return guarded([&] {
    if (n_out < 1 || k < 1 || t < 1) fail(SPIN_INPUT_ERROR, "spin_gemm_info: empty shape");
    const GemmPlan p = gemm_plan(n_out, k, t, mode, num_sms_cached());
    if (max_pieces) *max_pieces = p.max_pieces;
    if (grid) *grid = p.grid;
    if (bn) *bn = p.bn;
  });
}

spin_status spin_gemm(void* stream, const void* w, const void* x, int32_t n_out, int32_t k, int32_t t, int32_t mode,
                      float* part, float* amax_val, int32_t* amax_idx, float* logits) {
  return guarded([&] {
    if (n_out < 1 || k < 1 || t < 1) fail(SPIN_INPUT_ERROR, "spin_gemm: empty shape");
    if (k % 8 != 0) fail(SPIN_INPUT_ERROR, "spin_gemm: K must be a multiple of 8 (16-B rows)");
    const GemmPlan p = gemm_plan(n_out, k, t, mode, num_sms_cached());
    GemmEpilogue e;
    e.mode = mode;
    e.part = part;
    e.amax_val = amax_val;
    e.amax_idx = amax_idx;
    e.logits = logits;
    if (mode == kGemmPartial && part == nullptr) fail(SPIN_INPUT_ERROR, "spin_gemm: partial buffer missing");
    if (mode == kGemmArgmax && (amax_val == nullptr || amax_idx == nullptr))
      fail(SPIN_INPUT_ERROR, "spin_gemm: argmax buffers missing");
    check_cuda(gemm_launch(p, w, x, e, static_cast<cudaStream_t>(stream), false), "gemm launch");
    check_cuda(cudaGetLastError(), "gemm launch");
  });
}

}  // extern "C"
