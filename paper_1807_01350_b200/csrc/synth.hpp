// On-device generate_synthetic (proj/src/commands.cpp:110-134), slice batch
// by slice batch along the last mode (synth.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "devbuf.hpp"
#include "small_linalg.cuh"

namespace octen {

class SynthStream {
public:
    SynthStream(const std::vector<std::int64_t>& dims, int rank, std::uint64_t seed, double mu, double sigma,
                int device);
    ~SynthStream();
    SynthStream(const SynthStream&) = delete;
    SynthStream& operator=(const SynthStream&) = delete;
    // The next t slices (I x J x t, first index fastest) into device memory,
    // fp64 (dtype 0) or rounded to fp32 (dtype 1).
    void next(std::int64_t t, void* out, int dtype);
    // The normalized truth (model.normalize(), cp_als.cpp:216-228).
    void truth(double* const* factors, double* lambda) const;

    std::vector<std::int64_t> dims;
    int rank;
    std::uint64_t seed;
    double mu, sigma;
    int device;
    std::int64_t k_next = 0;
    cudaStream_t st = nullptr;

private:
    std::vector<std::vector<double>> hF;
    DevBuf<double> dF[3];  // order 3
    DevBuf<Mt64> state;
    DevBuf<double> X, U;
    DevBuf<int> flag;
    bool noisy = false, have_spare = false;
    double spare = 0.0;
};

}  // namespace octen
