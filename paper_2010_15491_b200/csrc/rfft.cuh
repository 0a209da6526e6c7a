// Real <-> Hermitian half-spectrum transforms along axis 1 (see rfft.cu).
#pragma once

#include "vsr_common.cuh"

namespace vsr {

// Row lengths L served (even powers of two, 16..2048).
bool rfft_rows_ok(size_t L);
// Pitch (complex elements) of a half-spectrum row: >= L/2 + 1, multiple of 8.
int half_pitch(size_t L);
// X[row][k] = sum_n x[row][n] e^{-2 pi i k n / L}, k = 0..L/2 (unnormalised),
// pad columns zeroed.  x: rows x L real, X: rows x half_pitch(L) complex.
void rfft_rows_forward(size_t L, const double* x, double2* X, long long rows, cudaStream_t st);
// x[row][n] = scale * sum_k Xh[row][k] e^{+2 pi i k n / L} - sub[row][n]
// (Xh = Hermitian extension of X; sub optional).
void rfft_rows_inverse(size_t L, const double2* X, double* x, long long rows, double scale, const double* sub,
                       cudaStream_t st);

}  // namespace vsr
