// Include shim for "volsr/spectral.hpp" -> the B200 mirror, plus the dense
// Eq.-8 check (a dense Eigen oracle, restated in refshim_extras.cpp).
// TEST INFRASTRUCTURE.
#pragma once
#include "volsr_b200/volsr.hpp"

namespace volsr {
double verify_eq8(const DecimationSpec& spec);
}  // namespace volsr
