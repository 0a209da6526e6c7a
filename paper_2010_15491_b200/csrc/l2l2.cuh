// admm_l2l2 device kernels (l2l2.cu); orchestration in capi.cu.
#pragma once

#include <algorithm>

#include "vsr_common.cuh"

namespace vsr {

struct L2Dims {
    long long m, n, s, N;
    long long ml, nl;
    int dr, dc, ds;
};

struct L2Scalars {
    double* objective;        // [max_iters]
    double* primal_residual;  // [max_iters]
    double* rel_change;       // [max_iters]
    double* status;           // [0] = 1 on an imaginary-residue violation, [1] = its ratio
    double* init_obj;
};

size_t l2_partial_blocks();  // partial-sum blocks of launch_l2_update (5 doubles each)
void launch_l2_sub(const double* v, const double* dual, double* t, long long N, cudaStream_t st);
void launch_l2_mul(double2* W, const double2* lam, long long N, cudaStream_t st);
void launch_l2_xhat(double2* W, double2* W2, const double2* lam, const double2* xbh, double mu, double reg,
                    long long N, cudaStream_t st);
void launch_l2_update(const L2Dims& D, bool update, const double* hx, const double* x, const double* xbar,
                      const double* y, double* v, double* dual, const double* xprev, double mu, double* partials,
                      cudaStream_t st);
// iter < 0: initial objective into sc.init_obj
void launch_l2_finalize(int iter, const double* up, const double* px, const double* ph, long long resn, double reg,
                        double max_rel_imag, const L2Scalars& sc, cudaStream_t st);

}  // namespace vsr
