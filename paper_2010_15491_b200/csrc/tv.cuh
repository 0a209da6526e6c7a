// ADMM-TV spatial kernels: fused forward-difference / isotropic shrink / dual
// update / divergence stencil, plus the small elementwise operators of the
// forward model (reference proj/src/operators.cpp, proj/src/solvers.cpp).
#pragma once

#include "vsr_common.cuh"

namespace vsr {

// Per-block partial layout of the stencil: [resid, tv, dx2, xprev2].
constexpr int kStencilVals = 4;

struct StencilGeom {
    dim3 grid;
    int kc;  // planes per CTA chunk
    size_t blocks() const { return (size_t)grid.x * grid.y * grid.z; }
};
StencilGeom stencil_geom(const Dims& d);

// One fused pass over the HR grid (solvers.cpp:367-393 restated):
//   lx_a = x(j + e_a) - x(j); nu = lx + dual; u = shrink(nu, thr);
//   dual' = nu - u; rho = u - dual'; theta(j) = sum_a rho_a(j - e_a) - rho_a(j)
// init = true: iteration-0 state u = Lx, dual = 0 (solvers.cpp:356-358);
//   dual_out is zeroed and theta = L^T L x.
// xprev (optional): accumulates ||x - xprev||^2, ||xprev||^2 (rel_change, :24-32).
// partials: kStencilVals doubles per block (resid, tv, dx2, xprev2).
void launch_tv_stencil(const Dims& d, bool init, const double* x, const double* dual_in,
                       double* dual_out, double* theta, double thr, const double* xprev,
                       double* partials, cudaStream_t st);

// Slab of a y-distributed volume (slab.cu): local dims (m, n/P, s), z
// periodic; the halo rows -1 / n/P come from the neighbouring ranks' x
// (ylo_x: row n/P - 1 of the rank below, yhi_x: row 0 of the rank above)
// and dual_in (ylo_d), read in place (NVLink peer memory); the dual arrays
// hold 3 components of the local volume.  axis 1 must be even.
void launch_tv_stencil_yslab(const Dims& loc, bool init, const double* x, const double* dual_in, double* dual_out,
                             double* theta, double thr, const double* xprev, double* partials, const double* ylo_x,
                             const double* yhi_x, const double* ylo_d, cudaStream_t st);

// fp32 mode: the same fused stencil with x, dual, dual' and theta stored in
// fp32 (arithmetic and reductions in fp64); axis 1 must be even.
void launch_tv_stencil_f32(const Dims& d, bool init, const float* x, const float* dual_in, float* dual_out,
                           float* theta, double thr, const float* xprev, double* partials, cudaStream_t st);

// Per-iteration scalar reduction for admm_tv (fixed order, single CTA):
// report[iter] objective / primal residual / rel change, residue check.
struct TvIterScalars {
    double* objective;        // [max_iters]
    double* primal_residual;  // [max_iters]
    double* rel_change;       // [max_iters]
    double* status;           // [4]: first residue violation iter (-1 none), its ratio, last ratio, pad
    int* iter_dev = nullptr;  // optional device iteration counter (read and advanced by the finalize),
                              // so a captured iteration replays without new kernel arguments
};
void launch_tv_finalize(int iter, const double* fit_partials, size_t fit_blocks,
                        const double* st_partials, size_t st_blocks, const double* res_partials,
                        size_t res_blocks, double tv_weight, double max_rel_imag,
                        TvIterScalars sc, double* init_objective_out, cudaStream_t st);

// Elementwise operators (operators.cpp:133-223, solvers.cpp:286-301).
void launch_decimate(const Dims& hr, const int rates[3], const double* x, double* y, cudaStream_t st);
void launch_decimate_adjoint(const Dims& hr, const int rates[3], const double* y, double* x,
                             double scale, cudaStream_t st);
void launch_nn_upsample(const Dims& hr, const int rates[3], const double* y, double* x,
                        cudaStream_t st);
void launch_diff(const Dims& d, int axis, bool adjoint, const double* x, double* out,
                 cudaStream_t st);
void launch_shrink(size_t count, const double* nu1, const double* nu2, const double* nu3,
                   double thr, double* o1, double* o2, double* o3, cudaStream_t st);
void launch_gamma(const Dims& d, const double* nr, const double* nc, const double* ns, double tau,
                  double* gamma, cudaStream_t st);
// sum over voxels of ||(Lx)_j||_2 -> per-block partials (objective_tv TV term, :304-317)
size_t tv_norm_blocks(const Dims& d);
void launch_tv_norm(const Dims& d, const double* x, double* partials, cudaStream_t st);

}  // namespace vsr
