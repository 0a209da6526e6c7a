// Spatial expansion of the closed-form Tikhonov solve for a separable,
// compactly supported blur and a prior on the decimation lattice.
//
// With Lambda(f) = a(f1) b(f2) c(f3) and fft3(xbar) = Z(g) replicated over
// the aliases (xbar = D^H z), the fold of TikhonovOperator::solve
// (solvers.cpp:53-62) factors per axis:
//   sum_b Lambda_b = A1 B1 C1,  sum_b |Lambda_b|^2 = A2 B2 C2   (per-axis alias sums)
//   w(g) = (yv G2 + 2 reg Z G1) / (G2 + 2 reg d),   yv = F_l(y) / sqrt(d)
//   x_hat(f) = Z(g) + conj(Lambda(f)) U(g),  U = (yv - w) / (2 reg)
//            = (d yv - Z G1) / (G2 + 2 reg d)      (no 1/(2 reg) cancellation)
// and since F_HR^-1 of an LR-periodic spectrum is sqrt(d) D^H F_l^-1:
//   x = D^H z + sqrt(d) H^T D^H u,   u = F_l^-1(U)   (real)
// H^T D^H u is a separable correlation of the lattice-sparse volume with the
// PSF's 1-D factors (support 2h+1 per axis), evaluated directly: one HBM pass
// writing x.  Exact up to rounding; the FFT budget stays one forward (F_l y)
// and one inverse (F_l^-1 V) transform per solve.
#pragma once

#include <vector>

#include "vsr_common.cuh"

namespace vsr {

struct SpatialPlan {
    bool ok = false;
    int h[3] = {0, 0, 0};                 // half supports of the 1-D PSF factors
    int dmin[3] = {0, 0, 0};              // first LR offset of the polyphase window, -floor(h / r)
    int ndelta[3] = {0, 0, 0};            // LR offsets a phase can touch
    int dm = 0;                           // padded taps per phase (kernel template width)
    const double* kp = nullptr;           // device phase-padded taps (spatial_phase_taps)
    std::vector<double> kp_host;          // the same taps on the host (march kernel: kernel parameters)
    // per-axis alias sums of the spectral tables (device): A1, A2 (ml), B1, B2 (nl), C1, C2 (sl)
    const double2* s1[3] = {nullptr, nullptr, nullptr};
    const double* s2[3] = {nullptr, nullptr, nullptr};
};

// Host: 1-D spatial PSF factors and per-axis alias sums from the separable
// tables (a | b | c concatenated, m + n + s entries).  taps: (2h+1) per axis
// concatenated; s1/s2: ml + nl + sl entries.  false: not real / not compact.
bool spatial_plan_host(const Dims& hr, const int rates[3], const std::vector<double2>& tabs,
                       std::vector<double>& taps, int h[3], std::vector<double2>& s1, std::vector<double>& s2);

// Padded taps-per-phase width the expand kernel uses for this plan (fills
// nothing), 0 if the support is too wide for the shared-memory tile.
int spatial_tile(const SpatialPlan& p, const int rates[3]);

// Host: phase-padded taps kp[phi * dm + i] = k[r (dmin + i) - phi + h] (0 off
// the support), axes concatenated.
void spatial_phase_taps(const int rates[3], const int h[3], const int dmin[3], const std::vector<double>& taps,
                        int dm, std::vector<double>& out);

// U(g) = (d yv - Z G1) / (G2 + 2 reg d) for the LR grid (dims ml x nl x sl).
void launch_spatial_v(const Dims& lr, int d, const SpatialPlan& p, const double2* Yl, const double2* Zl,
                      double reg, double2* V, cudaStream_t st);

// Fused LR stage, in place on Y holding the forward axis-1/2 passes of y
// (unscaled): forward axis-3 FFT (x fwd_scale), U, inverse axis-3 FFT
// (x out_scale).  The axis-2/1 inverse passes then give u.
bool spatial_sandwich_ok(const Dims& lr);
void launch_spatial_sandwich(const Dims& lr, int d, const SpatialPlan& p, double2* Y, const double2* Zl,
                             double reg, double fwd_scale, double out_scale, cudaStream_t st);

// x = D^H z + c0 * H^T D^H v   (hr grid, rates); non-finite index -> bad (atomicMin)
void launch_spatial_expand(const Dims& hr, const int rates[3], const SpatialPlan& p, const double* v,
                           const double* z, double c0, double* x, unsigned long long* bad, cudaStream_t st);
// fp32 mode: the z-march expansion in fp32 arithmetic writing fp32 x (u and
// the lattice prior stay fp64); only for the geometries the z march serves.
bool spatial_march_ok(const Dims& hr, const int rates[3], const SpatialPlan& p);
void launch_spatial_expand_f32(const Dims& hr, const int rates[3], const SpatialPlan& p, const double* u,
                               const double* z, float* x, unsigned long long* bad, cudaStream_t st);

}  // namespace vsr
