// Error plumbing for the C ABI: a thread-local message plus a status code that
// maps 1:1 onto the reference's exception taxonomy (errors.hpp:7-33).
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "spin_c.h"

namespace spin {

struct SpinError : std::runtime_error {
  spin_status status;
  SpinError(spin_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

void set_last_error(const std::string& msg);

[[noreturn]] inline void fail(spin_status s, const std::string& msg) { throw SpinError(s, msg); }

inline void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(SPIN_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

// Runs `f`, converting exceptions into a status + thread-local message.
template <typename F>
spin_status guarded(F&& f) {
  try {
    f();
    set_last_error("");
    return SPIN_OK;
  } catch (const SpinError& e) {
    set_last_error(e.what());
    return e.status;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return SPIN_SIZE_ERROR;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return SPIN_CONSISTENCY_ERROR;
  }
}

}  // namespace spin
