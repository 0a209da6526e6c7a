// Device kernels of admm_l2l2 (reference src/solvers.cpp:95-189): the
// iterative l2-l2 comparator with the split v = Hx.
// Orchestration is in capi.cu (vsr_admm_l2l2); every reduction is per-block
// partials in a fixed grid followed by a single-CTA fixed-order sum, so runs
// are byte-identical.
#include "l2l2.cuh"

namespace vsr {
namespace {

constexpr int L2_THREADS = 256;
constexpr int L2_BLOCKS = 148 * 8;  // fixed grid: partial-sum order does not depend on N

__global__ void __launch_bounds__(L2_THREADS) l2_sub_kernel(const double* __restrict__ v,
                                                            const double* __restrict__ dual, double* __restrict__ t,
                                                            long long N) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < N; p += (long long)gridDim.x * blockDim.x)
        t[p] = v[p] - dual[p];
}

__global__ void __launch_bounds__(L2_THREADS) l2_mul_kernel(double2* __restrict__ W, const double2* __restrict__ lam,
                                                            long long N) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < N; p += (long long)gridDim.x * blockDim.x)
        W[p] = cmul(lam[p], W[p]);
}

// x_hat = (mu conj(L) t_hat + 2 reg xbar_hat) / (mu |L|^2 + 2 reg)   (solvers.cpp:108-111,144-146)
// W2 = L x_hat                                                       (:149-150)
__global__ void __launch_bounds__(L2_THREADS) l2_xhat_kernel(double2* __restrict__ W, double2* __restrict__ W2,
                                                             const double2* __restrict__ lam,
                                                             const double2* __restrict__ xbh, double mu,
                                                             double reg2, long long N) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < N;
         p += (long long)gridDim.x * blockDim.x) {
        const double2 L = lam[p];
        const double denom = mu * cnorm(L) + reg2;
        const double2 a = cmulc(L, W[p]);  // conj(L) t_hat
        const double2 num = cadd(cscale(a, mu), cscale(xbh[p], reg2));
        const double2 xh = make_double2(num.x / denom, num.y / denom);
        W[p] = xh;
        W2[p] = cmul(L, xh);
    }
}

// v / dual update (:153-167) and the objective / residual / rel-change sums
// (:169-180, :24-32).  UPDATE = false: initial objective only (fit, reg).
template <bool UPDATE>
__global__ void __launch_bounds__(L2_THREADS) l2_update_kernel(L2Dims D, const double* __restrict__ hx,
                                                               const double* __restrict__ x,
                                                               const double* __restrict__ xbar,
                                                               const double* __restrict__ y, double* __restrict__ v,
                                                               double* __restrict__ dual,
                                                               const double* __restrict__ xprev, double mu,
                                                               double* __restrict__ partials) {
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};  // fit, reg, residual, |dx|^2, |xprev|^2
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < D.N;
         p += (long long)gridDim.x * blockDim.x) {
        const long long i = p % D.m, r = p / D.m, j = r % D.n, k = r / D.n;
        const bool lat = (i % D.dr) == 0 && (j % D.dc) == 0 && (k % D.ds) == 0;
        const double h = hx[p];
        double yv = 0.0;
        if (lat) {
            yv = y[(k / D.ds * D.nl + j / D.dc) * D.ml + i / D.dr];
            const double e = yv - h;  // decimate(hx) at the lattice
            acc[0] += e * e;
        }
        const double xv = x[p];
        const double dx = xv - xbar[p];
        acc[1] += dx * dx;
        if constexpr (UPDATE) {
            const double work = h + dual[p];
            const double vn = lat ? (yv + mu * work) / (1.0 + mu) : work;
            v[p] = vn;
            const double rr = h - vn;
            dual[p] += rr;
            acc[2] += rr * rr;
            if (xprev) {
                const double xp = xprev[p];
                acc[3] += (xv - xp) * (xv - xp);
                acc[4] += xp * xp;
            }
        }
    }
    __shared__ double red[32 * 5];
    block_reduce_sum<5>(acc, red);
    if (threadIdx.x == 0)
        for (int q = 0; q < 5; ++q) partials[5 * blockIdx.x + q] = acc[q];
}

__device__ void fixed_sum_l2(const double* part, int stride, int nv, long long nb, double* out, double* red) {
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (long long b = threadIdx.x; b < nb; b += blockDim.x)
        for (int q = 0; q < nv; ++q) acc[q] += part[b * stride + q];
    block_reduce_sum<5>(acc, red);
    if (threadIdx.x == 0)
        for (int q = 0; q < nv; ++q) out[q] = acc[q];
    __syncthreads();
}

__global__ void l2_finalize_kernel(int iter, const double* up, long long upn, const double* px, const double* ph,
                                   long long resn, double reg, double max_rel_imag, L2Scalars sc) {
    __shared__ double red[32 * 5];
    __shared__ double vals[9];
    fixed_sum_l2(up, 5, 5, upn, vals, red);
    if (px) fixed_sum_l2(px, 2, 2, resn, vals + 5, red);
    if (ph) fixed_sum_l2(ph, 2, 2, resn, vals + 7, red);
    if (threadIdx.x == 0) {
        const double obj = 0.5 * vals[0] + reg * vals[1];  // solvers.cpp:178
        if (iter < 0) {
            *sc.init_obj = obj;
        } else {
            sc.objective[iter] = obj;
            sc.primal_residual[iter] = sqrt(vals[2]);
            sc.rel_change[iter] = sqrt(vals[3]) / fmax(sqrt(vals[4]), 1e-300);
        }
        // ifft3_real residue checks of x and hx (fft.cpp:84-93): first violation wins
        for (int w = 0; w < 2; ++w) {
            if (!(w == 0 ? px : ph)) continue;
            const double im2 = vals[5 + 2 * w], tot2 = vals[6 + 2 * w];
            const double ratio = tot2 > 0.0 ? sqrt(im2 / tot2) : 0.0;
            if (tot2 > 0.0 && ratio > max_rel_imag && sc.status[0] == 0.0) {
                sc.status[0] = 1.0;
                sc.status[1] = ratio;
            }
        }
    }
}

unsigned blocks_for(long long N) { return (unsigned)std::min<long long>((N + L2_THREADS - 1) / L2_THREADS, L2_BLOCKS); }

}  // namespace

size_t l2_partial_blocks() { return L2_BLOCKS; }

void launch_l2_sub(const double* v, const double* dual, double* t, long long N, cudaStream_t st) {
    l2_sub_kernel<<<blocks_for(N), L2_THREADS, 0, st>>>(v, dual, t, N);
    VSR_LAUNCH_CHECK();
}

void launch_l2_mul(double2* W, const double2* lam, long long N, cudaStream_t st) {
    l2_mul_kernel<<<blocks_for(N), L2_THREADS, 0, st>>>(W, lam, N);
    VSR_LAUNCH_CHECK();
}

void launch_l2_xhat(double2* W, double2* W2, const double2* lam, const double2* xbh, double mu, double reg,
                    long long N, cudaStream_t st) {
    l2_xhat_kernel<<<blocks_for(N), L2_THREADS, 0, st>>>(W, W2, lam, xbh, mu, 2.0 * reg, N);
    VSR_LAUNCH_CHECK();
}

void launch_l2_update(const L2Dims& D, bool update, const double* hx, const double* x, const double* xbar,
                      const double* y, double* v, double* dual, const double* xprev, double mu, double* partials,
                      cudaStream_t st) {
    // fixed grid (L2_BLOCKS), independent of N, so the partial order is reproducible
    if (update)
        l2_update_kernel<true><<<L2_BLOCKS, L2_THREADS, 0, st>>>(D, hx, x, xbar, y, v, dual, xprev, mu, partials);
    else
        l2_update_kernel<false><<<L2_BLOCKS, L2_THREADS, 0, st>>>(D, hx, x, xbar, y, v, dual, xprev, mu, partials);
    VSR_LAUNCH_CHECK();
}

void launch_l2_finalize(int iter, const double* up, const double* px, const double* ph, long long resn, double reg,
                        double max_rel_imag, const L2Scalars& sc, cudaStream_t st) {
    l2_finalize_kernel<<<1, 1024, 0, st>>>(iter, up, L2_BLOCKS, px, ph, resn, reg, max_rel_imag, sc);
    VSR_LAUNCH_CHECK();
}

}  // namespace vsr
