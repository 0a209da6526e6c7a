// Spectral fold kernels.  One thread per LR frequency g; the d aliases of g
// are visited in b_lin order (b_r fastest), which is the reference's
// summation order (spectral.cpp:67-75: out[g] += block * v, b ascending).
// For d <= 8 the per-alias operands stay in registers (one HBM read per
// alias); for larger d a second sweep re-reads them (L2-resident: the CTA's
// alias footprint is a few tens of KB).
#include <cstring>

#include <algorithm>

#include "fold.cuh"

namespace vsr {

FoldGeom make_geom(const Dims& hr, const int rates[3]) {
    FoldGeom G;
    G.m = (long long)hr.m;
    G.n = (long long)hr.n;
    G.s = (long long)hr.s;
    G.dr = rates[0];
    G.dc = rates[1];
    G.ds = rates[2];
    G.ml = G.m / G.dr;
    G.nl = G.n / G.dc;
    G.sl = G.s / G.ds;
    G.d = G.dr * G.dc * G.ds;
    return G;
}

namespace {

constexpr int kFoldThreads = 128;

struct LrPos {
    long long g1, g2, g3;
};

__device__ __forceinline__ LrPos lr_pos(const FoldGeom& G, long long g) {
    LrPos p;
    p.g1 = g % G.ml;
    const long long r = g / G.ml;
    p.g2 = r % G.nl;
    p.g3 = r / G.nl;
    return p;
}

__device__ __forceinline__ long long alias_index(const FoldGeom& G, const LrPos& p, int b,
                                                 long long* f1, long long* f2, long long* f3) {
    const int br = b % G.dr;
    const int bc = (b / G.dr) % G.dc;
    const int bs = b / (G.dr * G.dc);
    *f1 = p.g1 + br * G.ml;
    *f2 = p.g2 + bc * G.nl;
    *f3 = p.g3 + bs * G.sl;
    return *f1 + G.m * (*f2 + G.n * *f3);
}

// ---------------------------------------------------------------- Tikhonov
// k_b   = conj(L_b) * (Yl[g]/sqrt d) + (2 reg) * X̄_b        (solvers.cpp:53-54)
// w     = (sum_b L_b k_b) / (sum_b |L_b|^2 + 2 reg d)     (:56-57, ctor :42-44)
// x̂_b  = (k_b - conj(L_b) w) * (1/(2 reg))                (:58-62)
template <int DC>
__global__ void __launch_bounds__(kFoldThreads)
    tik_fold_kernel(FoldGeom G, const double2* __restrict__ Yl, const double2* __restrict__ lam,
                    const double2* __restrict__ xbh, double2* __restrict__ xh, double reg2,
                    double shift, double inv2l, double invsqrtd) {
    const long long Nl = G.ml * G.nl * G.sl;
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= Nl) return;
    const LrPos p = lr_pos(G, g);
    const double2 yv = cscale(Yl[g], invsqrtd);
    double2 S = make_double2(0.0, 0.0);
    double gram = 0.0;
    const int d = DC > 0 ? DC : G.d;
    if constexpr (DC > 0) {
        double2 Lc[DC], kc[DC];
        long long fi[DC];
#pragma unroll
        for (int b = 0; b < DC; ++b) {
            long long f1, f2, f3;
            fi[b] = alias_index(G, p, b, &f1, &f2, &f3);
            Lc[b] = __ldg(lam + fi[b]);
        }
#pragma unroll
        for (int b = 0; b < DC; ++b) {
            const double2 X = __ldg(xbh + fi[b]);
            kc[b] = cadd(cmulc(Lc[b], yv), cscale(X, reg2));
            S = cadd(S, cmul(Lc[b], kc[b]));
            gram += cnorm(Lc[b]);
        }
        const double den = gram + shift;
        const double2 w = make_double2(S.x / den, S.y / den);
#pragma unroll
        for (int b = 0; b < DC; ++b)
            xh[fi[b]] = cscale(csub(kc[b], cmulc(Lc[b], w)), inv2l);
    } else {
        for (int b = 0; b < d; ++b) {
            long long f1, f2, f3;
            const long long f = alias_index(G, p, b, &f1, &f2, &f3);
            const double2 L = __ldg(lam + f);
            const double2 k = cadd(cmulc(L, yv), cscale(__ldg(xbh + f), reg2));
            S = cadd(S, cmul(L, k));
            gram += cnorm(L);
        }
        const double den = gram + shift;
        const double2 w = make_double2(S.x / den, S.y / den);
        for (int b = 0; b < d; ++b) {
            long long f1, f2, f3;
            const long long f = alias_index(G, p, b, &f1, &f2, &f3);
            const double2 L = __ldg(lam + f);
            const double2 k = cadd(cmulc(L, yv), cscale(__ldg(xbh + f), reg2));
            xh[f] = cscale(csub(k, cmulc(L, w)), inv2l);
        }
    }
}

// ---------------------------------------------------------------- TV
// k_b = conj(L_b) Yl/sqrt d + mu θ̂_b            (solvers.cpp:342-344,375)
// ĝ_b = Γ_b k_b                                  (:223)
// w   = (sum_b L_b ĝ_b) / (sum_b Γ_b|L_b|^2 + mu d)   (:225-226, :235-241)
// x̂_b = (ĝ_b - (Γ_b conj(L_b)) w) / mu          (:227-231, spectral.cpp:110)
template <int DC, bool GTAB, bool FIT>
__global__ void __launch_bounds__(kFoldThreads)
    tv_fold_kernel(FoldGeom G, const double2* __restrict__ Yl, const double2* __restrict__ lam,
                   const double2* th, double2* xh, const double* __restrict__ gam,
                   GammaTables tabs, double mu, double inv_mu, double shift, double invsqrtd,
                   double* __restrict__ fit_partials) {
    const long long Nl = G.ml * G.nl * G.sl;
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double fit = 0.0;
    if (g < Nl) {
        const LrPos p = lr_pos(G, g);
        const double2 yraw = Yl[g];
        const double2 yv = cscale(yraw, invsqrtd);
        double2 S = make_double2(0.0, 0.0);
        double gram = 0.0;
        double2 acc = make_double2(0.0, 0.0);
        auto gamma_at = [&](long long f, long long f1, long long f2, long long f3) -> double {
            if constexpr (GTAB)
                return 1.0 / (((__ldg(tabs.nr + f1) + __ldg(tabs.nc + f2)) + __ldg(tabs.ns + f3)) +
                              tabs.tau);
            else
                return __ldg(gam + f);
        };
        if constexpr (DC > 0) {
            double2 Lc[DC], gc[DC];
            double Gm[DC];
            long long fi[DC];
#pragma unroll
            for (int b = 0; b < DC; ++b) {
                long long f1, f2, f3;
                fi[b] = alias_index(G, p, b, &f1, &f2, &f3);
                Lc[b] = __ldg(lam + fi[b]);
                Gm[b] = gamma_at(fi[b], f1, f2, f3);
            }
#pragma unroll
            for (int b = 0; b < DC; ++b) {
                const double2 T = th[fi[b]];
                const double2 k = cadd(cmulc(Lc[b], yv), cscale(T, mu));
                gc[b] = cscale(k, Gm[b]);
                S = cadd(S, cmul(Lc[b], gc[b]));
                gram += Gm[b] * cnorm(Lc[b]);
            }
            const double den = gram + shift;
            const double2 w = make_double2(S.x / den, S.y / den);
#pragma unroll
            for (int b = 0; b < DC; ++b) {
                const double2 corr = cmul(make_double2(Gm[b] * Lc[b].x, -(Gm[b] * Lc[b].y)), w);
                const double2 x = cscale(csub(gc[b], corr), inv_mu);
                xh[fi[b]] = x;
                if constexpr (FIT) acc = cadd(acc, cmul(Lc[b], x));
            }
        } else {
            const int d = G.d;
            for (int b = 0; b < d; ++b) {
                long long f1, f2, f3;
                const long long f = alias_index(G, p, b, &f1, &f2, &f3);
                const double2 L = __ldg(lam + f);
                const double Gb = gamma_at(f, f1, f2, f3);
                const double2 k = cadd(cmulc(L, yv), cscale(th[f], mu));
                const double2 gb = cscale(k, Gb);
                S = cadd(S, cmul(L, gb));
                gram += Gb * cnorm(L);
            }
            const double den = gram + shift;
            const double2 w = make_double2(S.x / den, S.y / den);
            for (int b = 0; b < d; ++b) {
                long long f1, f2, f3;
                const long long f = alias_index(G, p, b, &f1, &f2, &f3);
                const double2 L = __ldg(lam + f);
                const double Gb = gamma_at(f, f1, f2, f3);
                const double2 k = cadd(cmulc(L, yv), cscale(th[f], mu));
                const double2 gb = cscale(k, Gb);
                const double2 corr = cmul(make_double2(Gb * L.x, -(Gb * L.y)), w);
                const double2 x = cscale(csub(gb, corr), inv_mu);
                xh[f] = x;
                if constexpr (FIT) acc = cadd(acc, cmul(L, x));
            }
        }
        if constexpr (FIT) {
            const double2 r = csub(yraw, cscale(acc, invsqrtd));
            fit = cnorm(r);
        }
    }
    if constexpr (FIT) {
        __shared__ double red[32];
        double v[1] = {fit};
        block_reduce_sum<1>(v, red);
        if (threadIdx.x == 0) fit_partials[blockIdx.x] = v[0];
    }
}

// Large-d TV fold: a CTA owns 32 consecutive LR frequencies x BG alias groups;
// each thread keeps AP = d / BG aliases in registers (one HBM read each).
// Partial sums over a group are combined in fixed group order through shared
// memory, so results are deterministic (the association differs from the
// reference's single running sum only at rounding level).
template <int BG, int AP, bool GTAB, bool FIT>
__global__ void __launch_bounds__(32 * BG)
    tv_fold_grouped_kernel(FoldGeom G, const double2* __restrict__ Yl, const double2* __restrict__ lam,
                           const double2* th, double2* xh, const double* __restrict__ gam,
                           GammaTables tabs, double mu, double inv_mu, double shift, double invsqrtd,
                           double* __restrict__ fit_partials) {
    __shared__ double2 sS[BG][32];
    __shared__ double sG[BG][32];
    __shared__ double red[32];
    const long long Nl = G.ml * G.nl * G.sl;
    const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
    const long long g = (long long)blockIdx.x * 32 + lane;
    const bool ok = g < Nl;
    const LrPos p = lr_pos(G, ok ? g : 0);
    const double2 yraw = ok ? Yl[g] : make_double2(0.0, 0.0);
    const double2 yv = cscale(yraw, invsqrtd);
    double2 Lc[AP], gc[AP];
    double Gm[AP];
    long long fi[AP];
    double2 S = make_double2(0.0, 0.0);
    double gram = 0.0;
#pragma unroll
    for (int a = 0; a < AP; ++a) {
        long long f1, f2, f3;
        fi[a] = alias_index(G, p, grp * AP + a, &f1, &f2, &f3);
        if (ok) {
            Lc[a] = __ldg(lam + fi[a]);
            if constexpr (GTAB)
                Gm[a] = 1.0 / (((__ldg(tabs.nr + f1) + __ldg(tabs.nc + f2)) + __ldg(tabs.ns + f3)) + tabs.tau);
            else
                Gm[a] = __ldg(gam + fi[a]);
        } else {
            Lc[a] = make_double2(0.0, 0.0);
            Gm[a] = 0.0;
        }
    }
#pragma unroll
    for (int a = 0; a < AP; ++a) {
        const double2 T = ok ? th[fi[a]] : make_double2(0.0, 0.0);
        const double2 k = cadd(cmulc(Lc[a], yv), cscale(T, mu));
        gc[a] = cscale(k, Gm[a]);
        S = cadd(S, cmul(Lc[a], gc[a]));
        gram += Gm[a] * cnorm(Lc[a]);
    }
    sS[grp][lane] = S;
    sG[grp][lane] = gram;
    __syncthreads();
    double2 St = sS[0][lane];
    double Gt = sG[0][lane];
#pragma unroll
    for (int b = 1; b < BG; ++b) {
        St = cadd(St, sS[b][lane]);
        Gt += sG[b][lane];
    }
    const double den = Gt + shift;
    const double2 w = make_double2(St.x / den, St.y / den);
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int a = 0; a < AP; ++a) {
        const double2 corr = cmul(make_double2(Gm[a] * Lc[a].x, -(Gm[a] * Lc[a].y)), w);
        const double2 xv = cscale(csub(gc[a], corr), inv_mu);
        if (ok) xh[fi[a]] = xv;
        if constexpr (FIT) acc = cadd(acc, cmul(Lc[a], xv));
    }
    if constexpr (FIT) {
        __syncthreads();
        sS[grp][lane] = acc;
        __syncthreads();
        double fit = 0.0;
        if (grp == 0 && ok) {
            double2 At = sS[0][lane];
#pragma unroll
            for (int b = 1; b < BG; ++b) At = cadd(At, sS[b][lane]);
            fit = cnorm(csub(yraw, cscale(At, invsqrtd)));
        }
        double v[1] = {fit};
        block_reduce_sum<1>(v, red);
        if (threadIdx.x == 0) fit_partials[blockIdx.x] = v[0];
    }
}

__global__ void __launch_bounds__(kFoldThreads)
    fit_kernel(FoldGeom G, const double2* __restrict__ Yl, const double2* __restrict__ lam,
               const double2* __restrict__ xh, double invsqrtd, double* __restrict__ partials) {
    const long long Nl = G.ml * G.nl * G.sl;
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double fit = 0.0;
    if (g < Nl) {
        const LrPos p = lr_pos(G, g);
        double2 acc = make_double2(0.0, 0.0);
        for (int b = 0; b < G.d; ++b) {
            long long f1, f2, f3;
            const long long f = alias_index(G, p, b, &f1, &f2, &f3);
            acc = cadd(acc, cmul(__ldg(lam + f), __ldg(xh + f)));
        }
        fit = cnorm(csub(Yl[g], cscale(acc, invsqrtd)));
    }
    __shared__ double red[32];
    double v[1] = {fit};
    block_reduce_sum<1>(v, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = v[0];
}

// ---------------------------------------------------------------- primitives
__global__ void fold_apply_kernel(FoldGeom G, const double2* __restrict__ lam,
                                  const double* __restrict__ wts, const double2* __restrict__ in,
                                  double2* __restrict__ out) {
    const long long Nl = G.ml * G.nl * G.sl;
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= Nl) return;
    const LrPos p = lr_pos(G, g);
    double2 acc = make_double2(0.0, 0.0);
    for (int b = 0; b < G.d; ++b) {
        long long f1, f2, f3;
        const long long f = alias_index(G, p, b, &f1, &f2, &f3);
        double2 coef = lam ? lam[f] : make_double2(1.0, 0.0);
        if (wts) coef = cscale(coef, wts[f]);  // (block * w) * v  (spectral.cpp:97)
        acc = cadd(acc, lam || wts ? cmul(coef, in[f]) : in[f]);
    }
    out[g] = acc;
}

__global__ void fold_adjoint_kernel(FoldGeom G, const double2* __restrict__ lam,
                                    const double* __restrict__ wts,
                                    const double2* __restrict__ in, double2* __restrict__ out) {
    const long long N = G.m * G.n * G.s;
    const long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= N) return;
    const long long f1 = f % G.m, f2 = (f / G.m) % G.n, f3 = f / (G.m * G.n);
    const long long g = (f1 % G.ml) + G.ml * ((f2 % G.nl) + G.nl * (f3 % G.sl));
    double2 v = in[g];
    if (lam) {
        double2 c = make_double2(lam[f].x, -lam[f].y);
        if (wts) c = cscale(c, wts[f]);  // (w * conj(block)) * lr  (spectral.cpp:110)
        v = cmul(c, v);
    }
    out[f] = v;
}

__global__ void gram_kernel(FoldGeom G, const double2* __restrict__ lam,
                            const double* __restrict__ wts, double* __restrict__ out) {
    const long long Nl = G.ml * G.nl * G.sl;
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= Nl) return;
    const LrPos p = lr_pos(G, g);
    double acc = 0.0;
    for (int b = 0; b < G.d; ++b) {
        long long f1, f2, f3;
        const long long f = alias_index(G, p, b, &f1, &f2, &f3);
        const double nrm = cnorm(lam[f]);
        acc += wts ? wts[f] * nrm : nrm;
    }
    out[g] = acc;
}

__global__ void swap_blocks_kernel(FoldGeom G, double2* lam) {
    const long long Nl = G.ml * G.nl * G.sl;
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= Nl) return;
    const LrPos p = lr_pos(G, g);
    long long f1, f2, f3;
    const long long a = alias_index(G, p, 0, &f1, &f2, &f3);
    const long long b = alias_index(G, p, 1, &f1, &f2, &f3);
    const double2 t = lam[a];
    lam[a] = lam[b];
    lam[b] = t;
}

__global__ void __launch_bounds__(1024)
    finalize_sum_kernel(const double* __restrict__ partials, int stride, int nvals,
                        long long nblocks, double* __restrict__ out) {
    __shared__ double red[32 * 4];
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (long long i = threadIdx.x; i < nblocks; i += blockDim.x)
        for (int k = 0; k < nvals; ++k) v[k] += partials[i * stride + k];
    block_reduce_sum<4>(v, red);
    if (threadIdx.x == 0)
        for (int k = 0; k < nvals; ++k) out[k] = v[k];
}

unsigned lr_blocks(const FoldGeom& G) {
    const long long Nl = G.ml * G.nl * G.sl;
    return (unsigned)((Nl + kFoldThreads - 1) / kFoldThreads);
}

}  // namespace

void launch_tik_fold(const FoldGeom& G, const double2* Yl, const double2* lam, const double2* xbh,
                     double2* xh, double reg, cudaStream_t st) {
    const double reg2 = 2.0 * reg;
    const double shift = 2.0 * reg * (double)G.d;  // solvers.cpp:43
    const double inv2l = 1.0 / (2.0 * reg);         // solvers.cpp:59
    const double invsqrtd = 1.0 / std::sqrt((double)G.d);
    const unsigned blocks = lr_blocks(G);
#define VSR_TIK(DCV) \
    tik_fold_kernel<DCV><<<blocks, kFoldThreads, 0, st>>>(G, Yl, lam, xbh, xh, reg2, shift, inv2l, invsqrtd)
    switch (G.d) {
        case 1: VSR_TIK(1); break;
        case 2: VSR_TIK(2); break;
        case 4: VSR_TIK(4); break;
        case 8: VSR_TIK(8); break;
        default: VSR_TIK(0); break;
    }
#undef VSR_TIK
    VSR_LAUNCH_CHECK();
}



size_t tv_fold_blocks_for(const FoldGeom& G);
size_t tv_fold_blocks(const FoldGeom& G) { return tv_fold_blocks_for(G); }

void launch_tv_fold(const FoldGeom& G, const double2* Yl, const double2* lam, const double2* th,
                    double2* xh, const double* gam, const GammaTables& tabs, double mu,
                    double* fit_partials, cudaStream_t st) {
    const double inv_mu = 1.0 / mu;                     // solvers.cpp:230
    const double shift = mu * (double)G.d;              // solvers.cpp:238
    const double invsqrtd = 1.0 / std::sqrt((double)G.d);
    const unsigned blocks = lr_blocks(G);
    const bool gtab = gam == nullptr;
    const bool fit = fit_partials != nullptr;
#define VSR_TV(DCV, GT, FT)                                                                  \
    tv_fold_kernel<DCV, GT, FT><<<blocks, kFoldThreads, 0, st>>>(G, Yl, lam, th, xh, gam, tabs, \
                                                                 mu, inv_mu, shift, invsqrtd,   \
                                                                 fit_partials)
#define VSR_TV_D(DCV)                           \
    if (gtab && fit) VSR_TV(DCV, true, true);   \
    else if (gtab) VSR_TV(DCV, true, false);    \
    else if (fit) VSR_TV(DCV, false, true);     \
    else VSR_TV(DCV, false, false);
    const long long Nl = G.ml * G.nl * G.sl;
    const unsigned gblocks = (unsigned)((Nl + 31) / 32);
#define VSR_TVG(BG, GT, FT)                                                                          \
    tv_fold_grouped_kernel<BG, 8, GT, FT><<<gblocks, 32 * BG, 0, st>>>(G, Yl, lam, th, xh, gam, tabs, mu, \
                                                                        inv_mu, shift, invsqrtd, fit_partials)
#define VSR_TVG_B(BG)                            \
    if (gtab && fit) VSR_TVG(BG, true, true);    \
    else if (gtab) VSR_TVG(BG, true, false);     \
    else if (fit) VSR_TVG(BG, false, true);      \
    else VSR_TVG(BG, false, false);
    switch (G.d) {
        case 1: VSR_TV_D(1); break;
        case 2: VSR_TV_D(2); break;
        case 4: VSR_TV_D(4); break;
        case 8: VSR_TV_D(8); break;
        case 16: VSR_TVG_B(2); break;
        case 32: VSR_TVG_B(4); break;
        case 64: VSR_TVG_B(8); break;
        default: VSR_TV_D(0); break;
    }
#undef VSR_TVG_B
#undef VSR_TVG
#undef VSR_TV_D
#undef VSR_TV
    VSR_LAUNCH_CHECK();
}

size_t tv_fold_blocks_for(const FoldGeom& G) {
    const long long Nl = G.ml * G.nl * G.sl;
    if (G.d == 16 || G.d == 32 || G.d == 64) return (size_t)((Nl + 31) / 32);
    return lr_blocks(G);
}

size_t fit_blocks(const FoldGeom& G) { return lr_blocks(G); }

void launch_fit_partials(const FoldGeom& G, const double2* Yl, const double2* lam,
                         const double2* xh, double* fit_partials, cudaStream_t st) {
    fit_kernel<<<lr_blocks(G), kFoldThreads, 0, st>>>(G, Yl, lam, xh,
                                                      1.0 / std::sqrt((double)G.d), fit_partials);
    VSR_LAUNCH_CHECK();
}

void launch_fold_apply(const FoldGeom& G, const double2* lam, const double* weights,
                       const double2* hr_in, double2* lr_out, cudaStream_t st) {
    fold_apply_kernel<<<lr_blocks(G), kFoldThreads, 0, st>>>(G, lam, weights, hr_in, lr_out);
    VSR_LAUNCH_CHECK();
}

void launch_fold_adjoint(const FoldGeom& G, const double2* lam, const double* weights,
                         const double2* lr_in, double2* hr_out, cudaStream_t st) {
    const long long N = G.m * G.n * G.s;
    fold_adjoint_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(G, lam, weights, lr_in, hr_out);
    VSR_LAUNCH_CHECK();
}

void launch_gram(const FoldGeom& G, const double2* lam, const double* weights, double* lr_out,
                 cudaStream_t st) {
    gram_kernel<<<lr_blocks(G), kFoldThreads, 0, st>>>(G, lam, weights, lr_out);
    VSR_LAUNCH_CHECK();
}

void launch_swap_blocks(const FoldGeom& G, double2* lam, cudaStream_t st) {
    swap_blocks_kernel<<<lr_blocks(G), kFoldThreads, 0, st>>>(G, lam);
    VSR_LAUNCH_CHECK();
}

void launch_finalize_sum(const double* partials, int stride, int nvals, size_t nblocks,
                         double* out, cudaStream_t st) {
    finalize_sum_kernel<<<1, 1024, 0, st>>>(partials, stride, nvals, (long long)nblocks, out);
    VSR_LAUNCH_CHECK();
}

namespace {
__global__ void __launch_bounds__(256) sep_dev_kernel(long long m, long long n, long long N,
                                                      const double2* __restrict__ lam,
                                                      unsigned long long* __restrict__ dev_bits,
                                                      unsigned long long* __restrict__ mag_bits) {
    // grid-stride max of |lam L0^2 - a b c| and |lam|; one atomic per block
    // (non-negative doubles order like their bit patterns)
    const double2 L0 = lam[0];
    const double2 L02 = cmul(L0, L0);
    double dev = 0.0, mag = 0.0;
    const long long mn = m * n;
    for (long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x; f < N;
         f += (long long)gridDim.x * blockDim.x) {
        const long long f3 = f / mn, r = f - f3 * mn, f2 = r / m, f1 = r - f2 * m;
        const double2 l = __ldg(lam + f);
        const double2 rhs = cmul(cmul(__ldg(lam + f1), __ldg(lam + m * f2)), __ldg(lam + mn * f3));
        dev = fmax(dev, cnorm(csub(cmul(l, L02), rhs)));
        mag = fmax(mag, cnorm(l));
    }
    for (int o = 16; o > 0; o >>= 1) {
        dev = fmax(dev, __shfl_down_sync(0xffffffffu, dev, o));
        mag = fmax(mag, __shfl_down_sync(0xffffffffu, mag, o));
    }
    __shared__ double sd[8], smg[8];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) sd[w] = dev, smg[w] = mag;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) dev = fmax(dev, sd[i]), mag = fmax(mag, smg[i]);
        atomicMax(dev_bits, (unsigned long long)__double_as_longlong(sqrt(dev)));
        atomicMax(mag_bits, (unsigned long long)__double_as_longlong(sqrt(mag)));
    }
}

__global__ void sep_tables_kernel(long long m, long long n, long long s, const double2* __restrict__ lam,
                                  double2* a, double2* b, double2* c) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const double2 L0 = lam[0];
    const double den = cnorm(L0);
    // x / L0 = x conj(L0) / |L0|^2
    auto divL0 = [&](double2 x) {
        const double2 p = cmul(x, make_double2(L0.x, -L0.y));
        return make_double2(p.x / den, p.y / den);
    };
    if (i < m) a[i] = divL0(lam[i]);
    if (i < n) b[i] = divL0(lam[m * i]);
    if (i < s) c[i] = lam[m * n * i];
}
}  // namespace

bool detect_separable(const Dims& hr, const double2* lam, double2* a, double2* b, double2* c, double tol,
                      cudaStream_t st) {
    const long long N = (long long)hr.count();
    unsigned long long* bits = nullptr;
    VSR_CUDA(cudaMallocAsync(&bits, 2 * sizeof(unsigned long long), st));
    VSR_CUDA(cudaMemsetAsync(bits, 0, 2 * sizeof(unsigned long long), st));
    sep_dev_kernel<<<(unsigned)std::min<long long>((N + 255) / 256, 148LL * 8), 256, 0, st>>>(
        (long long)hr.m, (long long)hr.n, N, lam, bits, bits + 1);
    VSR_LAUNCH_CHECK();
    unsigned long long h[2];
    VSR_CUDA(cudaMemcpyAsync(h, bits, sizeof(h), cudaMemcpyDeviceToHost, st));
    VSR_CUDA(cudaStreamSynchronize(st));
    cudaFreeAsync(bits, st);
    double dev, mag, l0[2];
    std::memcpy(&dev, &h[0], 8);
    std::memcpy(&mag, &h[1], 8);
    VSR_CUDA(cudaMemcpy(l0, lam, sizeof(l0), cudaMemcpyDeviceToHost));
    const double l0m2 = l0[0] * l0[0] + l0[1] * l0[1];
    if (!(l0m2 > 0.0) || !(mag > 0.0) || !(dev <= tol * mag * l0m2)) return false;
    const long long mx = std::max<long long>(hr.m, std::max<long long>(hr.n, hr.s));
    sep_tables_kernel<<<(unsigned)((mx + 255) / 256), 256, 0, st>>>((long long)hr.m, (long long)hr.n,
                                                                  (long long)hr.s, lam, a, b, c);
    VSR_LAUNCH_CHECK();
    return true;
}

// ------------------------------------------------------------ TV gram table
__global__ void __launch_bounds__(256) tv_gram_kernel(FoldGeom G, const double2* __restrict__ lam, SepTables sep,
                                                      GammaTables tabs, double* __restrict__ gw) {
    const long long Nl = G.ml * G.nl * G.sl;
    for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < Nl;
         g += (long long)gridDim.x * blockDim.x) {
        const long long g1 = g % G.ml, r = g / G.ml, g2 = r % G.nl, g3 = r / G.nl;
        double acc = 0.0;
        for (int bs = 0; bs < G.ds; ++bs)
            for (int bc = 0; bc < G.dc; ++bc)
                for (int br = 0; br < G.dr; ++br) {
                    const long long f1 = g1 + br * G.ml, f2 = g2 + bc * G.nl, f3 = g3 + bs * G.sl;
                    const double2 L = sep.a ? cmul(__ldg(sep.a + f1), cmul(__ldg(sep.b + f2), __ldg(sep.c + f3)))
                                            : __ldg(lam + f1 + G.m * (f2 + G.n * f3));
                    const double gam =
                        1.0 / ((__ldg(tabs.nr + f1) + (__ldg(tabs.nc + f2) + __ldg(tabs.ns + f3))) + tabs.tau);
                    acc += gam * cnorm(L);
                }
        gw[g] = acc;
    }
}

void launch_tv_gram(const FoldGeom& G, const double2* lam, const SepTables& sep, const GammaTables& tabs,
                    double* gw, cudaStream_t st) {
    const long long Nl = G.ml * G.nl * G.sl;
    const unsigned blocks = (unsigned)std::min<long long>((Nl + 255) / 256, 148LL * 16);
    tv_gram_kernel<<<blocks, 256, 0, st>>>(G, lam, sep, tabs, gw);
    VSR_LAUNCH_CHECK();
}

}  // namespace vsr
