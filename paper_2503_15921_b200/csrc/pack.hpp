// Request decomposition: the host restatement of the reference packer
// (packing.cpp:16-103) plus the verify cost accounting (slot_engine.cpp:24-45).
// The same algorithm runs on the device in meta_kernel (kernels.cu) so that the
// device-resident round loop needs no host round trip; the parity tests check
// the two bit-for-bit.
#pragma once

#include <cstdint>
#include <vector>

#include "spin_c.h"

namespace spin {

struct PackResult {
  int32_t length = 0;  // L
  int32_t rows = 0;    // rows actually used = min(width, n)
  int64_t padding = 0;
  std::vector<spin_segment> segments;
  std::vector<int32_t> q_replica_rows;
};

// Throws SpinError(SPIN_CONFIG_ERROR) on width < 1 or any length < 1.
void pack_validate(const int32_t* kv_lens, int32_t n, int32_t width);
PackResult pack_lengths(const int32_t* kv_lens, int32_t n, int32_t width);
int64_t naive_padding_of(const int32_t* kv_lens, int32_t n);  // SPIN_INPUT_ERROR on n == 0

struct VerifyCost {
  int64_t tokens = 0;
  int64_t padding = 0;
};
VerifyCost verify_cost(const int32_t* kv_lens, int32_t n, int32_t window, bool packing, int32_t pack_width);

}  // namespace spin
