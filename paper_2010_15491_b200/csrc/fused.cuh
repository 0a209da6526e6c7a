// Fused spectral-fold + axis-3 FFT kernels.
//
// The d aliases of an LR frequency g = (g1, g2, g3) sit at HR frequencies
// (g1 + br ml, g2 + bc nl, g3 + bs sl).  A CTA owns T consecutive g1 x one g2
// and the A = dr*dc axis-3 lines through their (br, bc) aliases, full length
// s: the bs aliases of every g3 then lie in one thread's registers and the
// (br, bc) aliases in lanes of one warp.  So the fold needs no extra HBM pass:
//   Tikhonov: x̂ = fold(Lambda, X̄, Ŷ) -> inverse axis-3 FFT        (one pass)
//   TV      : W -> forward axis-3 FFT -> fold -> inverse axis-3 FFT (one pass)
#pragma once

#include "fold.cuh"

#include <vector>

namespace vsr {

// Whether the fused kernels cover this geometry (otherwise callers use the
// separate fold + axis-pass kernels).
bool fused_axis3_ok(const FoldGeom& G);

// out = IFFT_axis3(x̂) (unscaled) with x̂ from TikhonovOperator::solve's fold
// (solvers.cpp:53-62).  out must not alias lam / xbh.  Zl (optional, LR
// layout): when the prior x̄ lives on the decimation lattice, fft3(x̄) at alias
// b of g equals Zl[g] for every b, so the 16N-byte X̄ is not read.
void launch_tik_fold_ifft3(const FoldGeom& G, const double2* Yl, const double2* lam,
                           const double2* xbh, double2* out, double reg, cudaStream_t st,
                           const SepTables& sep = SepTables{}, const double2* Zl = nullptr);

// In place on W (spectrum after forward axes 1,2): forward axis-3 FFT scaled
// by fwd_scale, TV x-update fold (solvers.cpp:219-233 with k̂ = data_hat +
// mu theta_hat), inverse axis-3 FFT (unscaled).  fit_partials: one double per
// block (||y - D H x||^2 by LR Parseval), sized by tv_sandwich_blocks().
size_t tv_sandwich_blocks(const FoldGeom& G);
void launch_tv_sandwich(const FoldGeom& G, const double2* Yl, const double2* lam, double2* W,
                        const GammaTables& tabs, double mu, double fwd_scale, double* fit_partials,
                        cudaStream_t st, const SepTables& sep = SepTables{});

// Same folds fused with the contiguous axis-1 pass instead (tile = the
// dc*ds alias rows of T consecutive g2, full rows along axis 1):
//   Tikhonov: out = IFFT_axis1(x̂); TV: W -> FFT_axis1 -> fold -> IFFT_axis1 -> W.
bool fused_axis1_ok(const FoldGeom& G);
void launch_tik_fold_ifft1(const FoldGeom& G, const double2* Yl, const double2* lam, const double2* xbh,
                           double2* out, double reg, cudaStream_t st, const SepTables& sep = SepTables{},
                           const double2* Zl = nullptr);
size_t tv_sandwich1_blocks(const FoldGeom& G);
// consecutive g2 per tile of the axis-1 sandwich (tile = (g2 / T, g3)); 0 if unsupported
int tv_sandwich1_tile_g2(const FoldGeom& G);
// Wout (optional): write x̂ there instead of in place (required with
// tabs.half3, where lines read other tiles' rows as conjugate mirrors).
void launch_tv_sandwich1(const FoldGeom& G, const double2* Yl, const double2* lam, double2* W,
                         const GammaTables& tabs, double mu, double fwd_scale, double* fit_partials,
                         cudaStream_t st, const SepTables& sep = SepTables{}, double2* Wout = nullptr);

// The pipelined variant of the half-spectrum TV sandwich (sandwich.cu):
// persistent CTAs, bulk-copy row loads into a 3-buffer ring, separable Lambda
// and the Gw table required, out != W, an explicit tile list (tabs.tiles).
// Returns false (nothing launched) when it does not cover the call.
bool tv_sandwich_pipe(const FoldGeom& G, const double2* Yl, const SepTables& sep, const double2* W, double2* out,
                      const GammaTables& tabs, double cA, double shift, double inv_scale, double fwd_scale,
                      double* fit_partials, cudaStream_t st);
// whether the pipelined sandwich covers the geometry (half spectrum, T = 1)
bool tv_sandwich_pipe_ok(const FoldGeom& G);
// fp32 mode: the same kernel on float2 rows, the transforms in fp32
// arithmetic and the fold in fp64.  W / out are float2 half spectra.
bool tv_sandwich_pipe_f32(const FoldGeom& G, const double2* Yl, const SepTables& sep, const float2* W, float2* out,
                          const GammaTables& tabs, double cA, double shift, double inv_scale, double fwd_scale,
                          double* fit_partials, cudaStream_t st);
// The tiles (g2, g3) of the half-spectrum axis-1 sandwich that do work (one
// of each conjugate pair of alias sets; tile = one LR (g2, g3)), g3-major.
std::vector<int2> tv_sandwich1_active_tiles(const FoldGeom& G);

}  // namespace vsr
