// ccl/generate.hpp — synthetic workloads (source-compatible with
// /root/reference/proj/include/ccl/generate.hpp): a seed fully defines the
// image, byte-for-byte identical to the reference generators, so benchmark
// and parity inputs are the reference's own inputs.
#pragma once

#include <cstdint>
#include <string>

#include "ccl/image.hpp"

namespace ccl {

// xoshiro256** seeded through splitmix64 (generate.hpp:10-43).
class Xoshiro256ss {
public:
    explicit Xoshiro256ss(std::uint64_t seed);
    std::uint64_t next();

private:
    std::uint64_t s_[4];
};

// One draw per pixel, raster order, fg iff (next() >> 11) < density * 2^53
// (generate.cpp:9-18).  std::invalid_argument unless 0 <= density <= 1.
BinaryImage random_image(std::uint32_t w, std::uint32_t h, double density, std::uint64_t seed);

enum class PatternKind { stripes, spiral, blobs, checkerboard };

PatternKind parse_pattern_kind(const std::string& s);

struct PatternParams {
    std::uint32_t period = 2;
    double density = 0.5;
    std::uint64_t seed = 0;
};

// generate.cpp:30-106: stripes (period >= 2), spiral (one component), blobs
// (seeded discs, radius max(2, min(w,h)/16)), checkerboard.
BinaryImage pattern_image(PatternKind kind, std::uint32_t w, std::uint32_t h, const PatternParams& params = {});

}  // namespace ccl
