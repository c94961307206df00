// Error taxonomy of the reference (proj/include/minimt/errors.hpp:8-34) carried
// across the C ABI as integer status codes (include/minimt_gpu.h).
#pragma once

#include <stdexcept>
#include <string>

#include <cuda_runtime.h>

namespace mtg {

enum Status : int {
  kOk = 0,
  kShapeError = 1,   // minimt::ShapeError
  kValueError = 2,   // minimt::ValueError
  kIndexError = 3,   // minimt::IndexError
  kStateError = 4,   // minimt::StateError
  kFormatError = 5,  // minimt::FormatError
  kUsageError = 6,   // minimt::UsageError
  kIoError = 7,      // minimt::IoError
  kCudaError = 8,    // device / driver failure (no reference counterpart)
};

struct Error : std::runtime_error {
  Status status;
  Error(Status s, const std::string& msg) : std::runtime_error(msg), status(s) {}
};

[[noreturn]] inline void fail(Status s, const std::string& msg) { throw Error(s, msg); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess)
    fail(kCudaError, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file +
                         ":" + std::to_string(line) + ")");
}

}  // namespace mtg

#define MTG_CUDA(x) ::mtg::cuda_check((x), #x, __FILE__, __LINE__)
