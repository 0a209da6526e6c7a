// Include shim for "volsr/solvers.hpp" -> the B200 mirror, plus the dense
// normal-equation oracles of the reference API (dense_tikhonov,
// dense_tv_x_update; restated in refshim_extras.cpp).  TEST INFRASTRUCTURE.
#pragma once
#include "volsr/spectral.hpp"

namespace volsr {
Volume3D dense_tikhonov(const Volume3D& y, const Volume3D& psf, const DecimationSpec& spec,
                        const TikhonovConfig& cfg);
Volume3D dense_tv_x_update(const Volume3D& y, const Volume3D& psf, const DecimationSpec& spec, double mu,
                           const Volume3D& theta, double tau);
}  // namespace volsr
