// Fused spectral-fold + axis-3 FFT kernels (see fused.cuh).
#include "fft.cuh"
#include "fft_core.cuh"
#include "fused.cuh"

namespace vsr {
namespace {

// CTA shape for line length L and A alias lines: T consecutive g1 per tile,
// capped so the exchange buffer (T*A lines of L complex) is <= 64 KB.
constexpr int FR = 8;  // values per thread in the fused kernels (register budget)

template <int L, int A>
struct FShape {
    static constexpr int P = fftc::Plan<L, FR>::P;
    static constexpr int TMAX = (4096 / (L * A)) > 0 ? (4096 / (L * A)) : 1;
    // the A alias lanes of one (g1, t) must sit in one warp: T * A <= 32
    static constexpr int TW = (32 / A) > 0 ? (32 / A) : 1;
    static constexpr int T0 = TMAX > 8 ? 8 : TMAX;
    static constexpr int T = T0 > TW ? TW : T0;
    static constexpr int NLN = T * A;               // lines per CTA
    static constexpr int THREADS = NLN * P;
    static constexpr int SMEM = fftc::Plan<L, FR>::NEEDS_SMEM ? NLN * L : 0;  // double2 elements
};

// xor-butterfly over the A alias lanes (lane stride T): every lane ends with
// the bit-identical total (fp addition is commutative, so each level combines
// identical operand pairs on both partners).
template <int T, int A>
__device__ __forceinline__ double lanes_sum(double v) {
#pragma unroll
    for (int o = T; o < T * A; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int L, int A, int DS, bool TV, bool FIT>
__global__ void __launch_bounds__(FShape<L, A>::THREADS, (512 / FShape<L, A>::THREADS) > 0 ? (512 / FShape<L, A>::THREADS) : 1)
    fold_axis3_kernel(FoldGeom G, const double2* __restrict__ Yl, const double2* __restrict__ lam,
                      const double2* __restrict__ xbh, double2* W, double2* out, GammaTables tabs,
                      double cA /*Tik: 2 reg, TV: mu*/, double shift, double inv_scale,
                      double invsqrtd, double fwd_scale, const double2* __restrict__ tw,
                      double* __restrict__ fit_partials) {
    using Pl = fftc::Plan<L, FR>;
    using Sh = FShape<L, A>;
    constexpr int R = Pl::R, P = Pl::P, T = Sh::T, NLN = Sh::NLN;
    constexpr int RD = R / DS;  // register groups: r = rr + RD * bs holds alias bs of g3 = t + P rr
    static_assert(R % DS == 0, "ds must divide R");
    extern __shared__ double2 sm[];

    const int tid = threadIdx.x;
    const int ln = tid % NLN, t = tid / NLN;
    const int ti = ln % T, a = ln / T;
    const int br = a % G.dr, bc = a / G.dr;
    const long long tpr = G.ml / T;
    const long long tile = blockIdx.x;
    const long long g1 = (tile % tpr) * T + ti, g2 = tile / tpr;
    const long long f1 = g1 + br * G.ml, f2 = g2 + bc * G.nl;
    const long long base = f1 + G.m * f2, stride = G.m * G.n;
    auto sidx = [&](int q) { return q * NLN + ln; };

    double2 v[R];
    if constexpr (TV) {
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = W[base + stride * (t + P * r)];
        fftc::stockham<L, false, decltype(sidx), FR>(v, t, sm, sidx, tw);
        fftc::to_natural<L, FR>(v);
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = cscale(v[r], fwd_scale);
    }
    // ---- fold in registers: thread holds q = t + P r, i.e. g3 = t + P (r % RD), bs = r / RD.
    // All operand loads are issued up front (memory-level parallelism), then
    // one g3 group (its DS axis-3 aliases) is folded at a time.
    double2 Lm[R];
#pragma unroll
    for (int r = 0; r < R; ++r) Lm[r] = __ldg(lam + base + stride * (t + P * r));
    if constexpr (!TV) {
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = __ldg(xbh + base + stride * (t + P * r));
    }
    double2 Yg[RD];
#pragma unroll
    for (int rr = 0; rr < RD; ++rr) Yg[rr] = __ldg(Yl + g1 + G.ml * (g2 + G.nl * (long long)(t + P * rr)));
    double base_g = 0.0;
    if constexpr (TV) base_g = __ldg(tabs.nr + f1) + __ldg(tabs.nc + f2);
    double fit = 0.0;
#pragma unroll
    for (int rr = 0; rr < RD; ++rr) {
        const double2 yv = cscale(Yg[rr], invsqrtd);
        double Gg[DS];
        double Sx = 0.0, Sy = 0.0, gram = 0.0;
#pragma unroll
        for (int bs = 0; bs < DS; ++bs) {
            const int r = rr + RD * bs;
            if constexpr (TV) {
                // k = conj(L) F D^H y + mu theta_hat (solvers.cpp:342-344,375); ĝ = Γ k (:223)
                Gg[bs] = 1.0 / ((base_g + __ldg(tabs.ns + (t + P * r))) + tabs.tau);
                v[r] = cscale(cadd(cmulc(Lm[r], yv), cscale(v[r], cA)), Gg[bs]);
                gram += Gg[bs] * cnorm(Lm[r]);
            } else {
                // k = conj(L) F D^H y + 2 reg X̄ (solvers.cpp:53-54)
                v[r] = cadd(cmulc(Lm[r], yv), cscale(v[r], cA));
                gram += cnorm(Lm[r]);
            }
            const double2 pr = cmul(Lm[r], v[r]);
            Sx += pr.x;
            Sy += pr.y;
        }
        Sx = lanes_sum<T, A>(Sx);
        Sy = lanes_sum<T, A>(Sy);
        gram = lanes_sum<T, A>(gram);
        const double den = gram + shift;
        const double2 w = make_double2(Sx / den, Sy / den);
        double ax = 0.0, ay = 0.0;
#pragma unroll
        for (int bs = 0; bs < DS; ++bs) {
            const int r = rr + RD * bs;
            double2 c;
            if constexpr (TV)
                c = cmul(make_double2(Gg[bs] * Lm[r].x, -(Gg[bs] * Lm[r].y)), w);  // spectral.cpp:110
            else
                c = cmulc(Lm[r], w);
            v[r] = cscale(csub(v[r], c), inv_scale);  // x̂ (solvers.cpp:60-62 / :230-231)
            if constexpr (FIT) {
                const double2 pr = cmul(Lm[r], v[r]);
                ax += pr.x;
                ay += pr.y;
            }
        }
        if constexpr (FIT) {
            ax = lanes_sum<T, A>(ax);
            ay = lanes_sum<T, A>(ay);
            if (a == 0) {
                const double rx = Yg[rr].x - invsqrtd * ax, ry = Yg[rr].y - invsqrtd * ay;
                fit += rx * rx + ry * ry;
            }
        }
    }
    // ---- inverse axis-3 FFT of x̂ (natural order in v)
    if constexpr (TV) __syncthreads();  // the forward transform's exchange buffer is reused
    fftc::stockham<L, true, decltype(sidx), FR>(v, t, sm, sidx, tw);
    double2* dst = TV ? W : out;
#pragma unroll
    for (int j = 0; j < R; ++j) dst[base + stride * Pl::out_q(t, j)] = v[j];
    if constexpr (FIT) {
        __shared__ double red[32];
        double vv[1] = {fit};
        block_reduce_sum<1>(vv, red);
        if (tid == 0) fit_partials[blockIdx.x] = vv[0];
    }
}

// ---------------------------------------------------------------- dispatch
struct Key {
    int L, A, DS;
};

template <int L, int A, int DS, bool TV, bool FIT>
void launch_one(const FoldGeom& G, const double2* Yl, const double2* lam, const double2* xbh,
                double2* W, double2* out, const GammaTables& tabs, double cA, double shift,
                double inv_scale, double fwd_scale, double* fit, cudaStream_t st) {
    using Sh = FShape<L, A>;
    auto kern = fold_axis3_kernel<L, A, DS, TV, FIT>;
    const size_t smem = (size_t)Sh::SMEM * sizeof(double2);
    if (smem > 48 * 1024)
        VSR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const unsigned grid = (unsigned)((G.ml / Sh::T) * G.nl);
    kern<<<grid, Sh::THREADS, smem, st>>>(G, Yl, lam, xbh, W, out, tabs, cA, shift, inv_scale,
                                          1.0 / std::sqrt((double)G.d), fwd_scale,
                                          fft_engine().twiddles((size_t)L), fit);
    VSR_LAUNCH_CHECK();
}

// Supported (L, A = dr*dc, DS) triples; others take the unfused path.
#define VSR_FUSED_TABLE(X) \
    X(32, 4, 2) X(32, 4, 4) X(32, 16, 4) X(32, 1, 1)                    \
    X(64, 4, 2) X(128, 4, 2) X(256, 4, 2) X(512, 4, 2) X(1024, 4, 2)  \
    X(64, 4, 4) X(128, 4, 4) X(256, 4, 4) X(512, 4, 4) X(1024, 4, 4)  \
    X(64, 16, 4) X(128, 16, 4) X(256, 16, 4)                           \
    X(64, 1, 1) X(128, 1, 1) X(256, 1, 1) X(512, 1, 1) X(1024, 1, 1)

template <bool TV, bool FIT>
bool dispatch(const FoldGeom& G, const double2* Yl, const double2* lam, const double2* xbh,
              double2* W, double2* out, const GammaTables& tabs, double cA, double shift,
              double inv_scale, double fwd_scale, double* fit, cudaStream_t st) {
    const int A = G.dr * G.dc;
#define VSR_X(LL, AA, DD)                                                                           \
    if (G.s == LL && A == AA && G.ds == DD && G.ml % FShape<LL, AA>::T == 0) {                      \
        launch_one<LL, AA, DD, TV, FIT>(G, Yl, lam, xbh, W, out, tabs, cA, shift, inv_scale,        \
                                        fwd_scale, fit, st);                                        \
        return true;                                                                                \
    }
    VSR_FUSED_TABLE(VSR_X)
#undef VSR_X
    return false;
}

}  // namespace

bool fused_axis3_ok(const FoldGeom& G) {
    const int A = G.dr * G.dc;
#define VSR_X(LL, AA, DD) \
    if (G.s == LL && A == AA && G.ds == DD && G.ml % FShape<LL, AA>::T == 0) return true;
    VSR_FUSED_TABLE(VSR_X)
#undef VSR_X
    return false;
}

void launch_tik_fold_ifft3(const FoldGeom& G, const double2* Yl, const double2* lam,
                           const double2* xbh, double2* out, double reg, cudaStream_t st) {
    GammaTables none{nullptr, nullptr, nullptr, 0.0};
    const double shift = 2.0 * reg * (double)G.d;  // solvers.cpp:43
    const double inv2l = 1.0 / (2.0 * reg);         // solvers.cpp:59
    if (!dispatch<false, false>(G, Yl, lam, xbh, nullptr, out, none, 2.0 * reg, shift, inv2l, 1.0,
                                nullptr, st))
        throw std::logic_error("launch_tik_fold_ifft3: unsupported geometry");
}

size_t tv_sandwich_blocks(const FoldGeom& G) {
    const int A = G.dr * G.dc;
#define VSR_X(LL, AA, DD) \
    if (G.s == LL && A == AA && G.ds == DD) return (size_t)((G.ml / FShape<LL, AA>::T) * G.nl);
    VSR_FUSED_TABLE(VSR_X)
#undef VSR_X
    return 0;
}

void launch_tv_sandwich(const FoldGeom& G, const double2* Yl, const double2* lam, double2* W,
                        const GammaTables& tabs, double mu, double fwd_scale, double* fit_partials,
                        cudaStream_t st) {
    const double shift = mu * (double)G.d;  // solvers.cpp:238
    const double inv_mu = 1.0 / mu;         // solvers.cpp:230
    const bool ok = fit_partials
                        ? dispatch<true, true>(G, Yl, lam, nullptr, W, nullptr, tabs, mu, shift, inv_mu,
                                               fwd_scale, fit_partials, st)
                        : dispatch<true, false>(G, Yl, lam, nullptr, W, nullptr, tabs, mu, shift, inv_mu,
                                                fwd_scale, nullptr, st);
    if (!ok) throw std::logic_error("launch_tv_sandwich: unsupported geometry");
}

}  // namespace vsr
