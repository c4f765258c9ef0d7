// Exception taxonomy of the drop-in API (mirrors the reference's
// core/include/specsim/errors.hpp:7-33); the C ABI's spin_status values map 1:1
// onto these, plus CudaError for device failures.
#pragma once

#include <stdexcept>
#include <string>

namespace specsim {

#define SPECSIM_ERROR_TYPE(Name)                                \
  struct Name : std::runtime_error {                            \
    explicit Name(const std::string& what) : std::runtime_error(what) {} \
  }

SPECSIM_ERROR_TYPE(ConfigError);       // invalid configuration / spec
SPECSIM_ERROR_TYPE(CapacityError);     // a batch or context exceeds capacity
SPECSIM_ERROR_TYPE(InputError);        // malformed call arguments
SPECSIM_ERROR_TYPE(SizeError);         // buffer / size limits
SPECSIM_ERROR_TYPE(ConsistencyError);  // layouts or state that do not agree
SPECSIM_ERROR_TYPE(MetricError);
SPECSIM_ERROR_TYPE(IoError);
SPECSIM_ERROR_TYPE(CudaError);  // B200 backend only

#undef SPECSIM_ERROR_TYPE

// Throws the exception type matching a spin_status code (spin_c.h); no-op for 0.
void throw_status(int status, const std::string& message);

}  // namespace specsim
