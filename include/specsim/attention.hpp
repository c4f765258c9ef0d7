// Packed attention operator of the drop-in API (the reference's
// core/include/specsim/attention.hpp:11-49), computed on the B200 by the
// split-KV kernel family of the verifier (fp64 on the device).
#pragma once

#include <cstdint>
#include <vector>

#include "specsim/packing.hpp"

namespace specsim {

struct Matrix {
  int rows = 0;
  int cols = 0;
  std::vector<double> data;
  Matrix() = default;
  Matrix(int r, int c) : rows(r), cols(c), data(static_cast<std::size_t>(r) * c, 0.0) {}
  double at(int r, int c) const { return data[static_cast<std::size_t>(r) * cols + c]; }
  double& at(int r, int c) { return data[static_cast<std::size_t>(r) * cols + c]; }
};

struct ToyAttentionInput {
  Matrix q;
  Matrix k;
  Matrix v;
};

Matrix reference_attention(const Matrix& q, const Matrix& k, const Matrix& v);
std::vector<Matrix> decomposed_attention(const std::vector<ToyAttentionInput>& inputs, const PackedLayout& layout,
                                         const IndicatorMask& mask);
ToyAttentionInput make_toy_input(std::uint64_t seed, int queries, int kv_len, int dim);

}  // namespace specsim
