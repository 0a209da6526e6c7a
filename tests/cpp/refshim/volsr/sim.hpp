// Include shim for "volsr/sim.hpp": degrade comes from the B200 mirror
// (vsr_degrade); the phantom and noise generators are input synthesis,
// outside the hot path, restated in refshim_extras.cpp.  TEST INFRASTRUCTURE.
#pragma once
#include <cstdint>

#include "volsr_b200/volsr.hpp"

namespace volsr {
enum class PhantomKind { NestedEllipsoids, RandomSmooth, Constant };
Volume3D make_phantom(const Dims3& dims, PhantomKind kind, std::uint64_t seed = 0, double constant_value = 0.5);
inline constexpr const char* kNoiseAlgorithm = "mt19937_64-boxmuller";
Volume3D gaussian_noise(const Dims3& dims, std::uint64_t seed);
}  // namespace volsr
