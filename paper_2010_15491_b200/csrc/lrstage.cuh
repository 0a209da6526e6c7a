// Persistent (cooperative) LR stage of the spatial-expansion Tikhonov solve:
// r2c rows -> axis 2 -> axis-3 filter sandwich -> inverse axis 2 -> c2r rows
// minus q, one launch with grid barriers (lrstage.cu).
#pragma once

#include "vsr_common.cuh"

namespace vsr {

bool lr_stage_ok(const Dims& lr);
// u = c2r(IFFT_23(cfac / (a2 b2 c2 + shift) * FFT_23(r2c(y)))) - q on the LR grid;
// Yh: half-spectrum scratch (half_pitch(ml) x nl x sl complex).
void launch_lr_stage(const Dims& lr, const double* y, double2* Yh, double* u, const double* q, const double* a2,
                     const double* b2, const double* c2, double cfac, double shift, cudaStream_t st);

}  // namespace vsr
