// Spectral decimation fold/unfold kernels (paper Eq. 8/9; reference
// proj/src/spectral.cpp and the solver loops in proj/src/solvers.cpp).
#pragma once

#include "vsr_common.cuh"

namespace vsr {

// HR/LR geometry of a DecimationSpec (reference src/operators.cpp:8-21).
// Alias b = (br, bc, bs) of LR frequency g = (g1, g2, g3) sits at HR
// frequency (g1 + br*ml, g2 + bc*nl, g3 + bs*sl): contiguous blocks
// (reference include/volsr/spectral.hpp:7-11).  b_lin = br + dr*bc + dr*dc*bs.
struct FoldGeom {
    long long m, n, s;
    long long ml, nl, sl;
    int dr, dc, ds, d;
};

FoldGeom make_geom(const Dims& hr, const int rates[3]);

// Separable blur spectrum Lambda(f) = a[f1] * b[f2] * c[f3] (a Gaussian PSF
// is separable, so its DFT is the product of three 1-D DFTs).  When set, the
// fused fold kernels rebuild Lambda from these O(m+n+s) tables instead of
// streaming the 16N-byte HR spectrum.  a == nullptr: not separable.
struct SepTables {
    const double2* a = nullptr;
    const double2* b = nullptr;
    const double2* c = nullptr;
};

// Detects separability of an HR spectrum on the device (relative deviation
// <= tol) and, if so, fills a/b/c (device arrays of m, n, s) so that
// lam ~= a[f1] b[f2] c[f3].  Synchronizes the stream.
bool detect_separable(const Dims& hr, const double2* lam, double2* a, double2* b, double2* c, double tol,
                      cudaStream_t st);

// Per-axis |e^{2 pi i f/len} - 1|^2 tables on the device for make_gamma
// (reference src/operators.cpp:225-243, src/solvers.cpp:191-205).
struct GammaTables {
    const double* nr;
    const double* nc;
    const double* ns;
    double tau;
    // optional LR table Gw(g) = sum_b Gamma_b |Lambda_b|^2 (constant across
    // ADMM iterations, spectral.cpp:133-142): the TV fold then needs only one
    // cross-alias sum per LR frequency
    const double* gw = nullptr;
    // 1: W holds only planes f3 <= s/2 of a Hermitian spectrum (axis 3 r2c);
    // alias rows with f3 > s/2 are read as conj(row(-f2, s - f3)) and not stored
    int half3 = 0;
    // slab-sharded sandwich (slab.cu, half3 only): a rank holds a subset of
    // the half-spectrum planes.  wplane[f3] (f3 <= s/2) is the local plane of
    // W / the output, lplane[f3] (f3 < s) the local plane of a dense Lambda,
    // and tiles[i] = (g2 block, g3) the tiles this launch runs (ntiles of
    // them).  nullptr: identity / every tile.
    const int* wplane = nullptr;
    const int* lplane = nullptr;
    const int2* tiles = nullptr;
    int ntiles = 0;
    // 1: the axis-1 TV sandwich only reports the data fit of its INPUT
    // spectrum, ||Yl - (1/sqrt d) sum_b Lambda_b W_b||^2 per tile, and writes
    // nothing (the initial objective of a slab-sharded admm_tv)
    int fit_only = 0;
};

// Gw(g) = sum_b Gamma_b |Lambda_b|^2 over the d aliases of every LR frequency
// (b_lin ascending, gram_diag_weighted spectral.cpp:133-142).
void launch_tv_gram(const FoldGeom& G, const double2* lam, const SepTables& sep, const GammaTables& tabs,
                    double* gw, cudaStream_t st);

// ---- fused Tikhonov fold (TikhonovOperator::solve, solvers.cpp:53-62)
// x_hat[f] for every HR f from the LR spectrum Yl of y, Lambda and X̄ = fft3(xbar).
void launch_tik_fold(const FoldGeom& G, const double2* Yl, const double2* lam, const double2* xbh,
                     double2* xh, double reg, cudaStream_t st);

// ---- fused TV x-update fold (tv_x_core, solvers.cpp:219-233, with k_hat
// = conj(Lambda) F D^H y + mu*theta_hat assembled on the fly, :375).
// Gamma from tables (gam == nullptr) or an explicit HR array.
// fit_partials (optional): per-block sum |Yl - (1/sqrt d) sum_b Lambda_b x_hat_b|^2
// = ||y - D H x||^2 by LR Parseval (objective data term, :395-401).
size_t tv_fold_blocks(const FoldGeom& G);
void launch_tv_fold(const FoldGeom& G, const double2* Yl, const double2* lam, const double2* th,
                    double2* xh, const double* gam, const GammaTables& tabs, double mu,
                    double* fit_partials, cudaStream_t st);

// ---- data fit only: per-block partials of ||Yl - (1/sqrt d) sum_b Lambda_b Xh_b||^2
size_t fit_blocks(const FoldGeom& G);
void launch_fit_partials(const FoldGeom& G, const double2* Yl, const double2* lam,
                         const double2* xh, double* fit_partials, cudaStream_t st);

// ---- FoldedSpectrum primitives (spectral.cpp:67-142) for the general API.
// weights may be null (unweighted).  lam may be null (pure alias_fold/expand).
void launch_fold_apply(const FoldGeom& G, const double2* lam, const double* weights,
                       const double2* hr_in, double2* lr_out, cudaStream_t st);
void launch_fold_adjoint(const FoldGeom& G, const double2* lam, const double* weights,
                         const double2* lr_in, double2* hr_out, cudaStream_t st);
void launch_gram(const FoldGeom& G, const double2* lam, const double* weights, double* lr_out,
                 cudaStream_t st);
void launch_swap_blocks(const FoldGeom& G, double2* lam, cudaStream_t st);

// Per-block partial sums -> scalars (fixed order; single CTA).
void launch_finalize_sum(const double* partials, int stride, int nvals, size_t nblocks,
                         double* out, cudaStream_t st);

}  // namespace vsr
