// Host error types mirroring proj/include/cpstream/errors.hpp:9-26, plus a
// CUDA failure type.  The C-ABI maps them to status codes (octen_b200.h).
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

namespace octen {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ConfigError : Error {
    using Error::Error;
};
struct NumericError : Error {
    using Error::Error;
};
struct IoError : Error {
    using Error::Error;
};
struct CudaError : Error {
    using Error::Error;
};

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

}  // namespace octen

#define OCTEN_CUDA(x) ::octen::cuda_check((x), #x)
