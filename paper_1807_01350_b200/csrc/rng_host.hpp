// Host-side deterministic RNG, restating the reference's
// proj/include/cpstream/rng.hpp: SplitMix64 `derive` over frozen key kinds
// (rng.hpp:14-45) and the mt19937_64 Substream with 53-bit uniforms
// (rng.hpp:51-85).  std::mt19937_64 has a standardized output sequence, so the
// projection matrices, temporal rows and ALS mixtures drawn here are
// bit-identical to the reference's.
#pragma once

#include <cmath>
#include <cstdint>
#include <initializer_list>
#include <random>

namespace octen::rng {

constexpr std::uint64_t mix(std::uint64_t z) {
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

inline std::uint64_t derive(std::uint64_t master, std::initializer_list<std::uint64_t> path) {
    std::uint64_t z = mix(master);
    for (std::uint64_t k : path) z = mix(z ^ mix(k));
    return z;
}

enum : std::uint64_t {
    kNontemporalShared = 1,
    kNontemporalPrivate = 2,
    kTemporalShared = 3,
    kTemporalPrivate = 4,
    kAlsRestart = 5,
    kAlsFactor = 6,
    kAlsRescue = 7,
    kStreamAls = 8,
    kSynthFactor = 9,
    kSynthNoise = 10,
    kAlsGevd = 11,
};

class Substream {
public:
    explicit Substream(std::uint64_t seed) : eng_(seed) {}
    double uniform01() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
    // Column-major fill of a rows x cols block with leading dimension ld.
    void fill_uniform(double* dst, std::int64_t rows, std::int64_t cols, std::int64_t ld) {
        for (std::int64_t c = 0; c < cols; ++c)
            for (std::int64_t r = 0; r < rows; ++r) dst[r + ld * c] = uniform01();
    }

private:
    std::mt19937_64 eng_;
};

}  // namespace octen::rng
