// Fused spectral-fold + axis-3 FFT kernels (see fused.cuh).
#include "fft.cuh"
#include "fft_core.cuh"
#include "fused.cuh"

#include <cstdlib>

namespace vsr {
namespace {

// CTA shape for line length L and A alias lines: T consecutive g1 per tile,
// capped so the exchange buffer (T*A lines of L complex) is <= 64 KB.
constexpr int FR = 8;  // values per thread in the fused kernels (register budget)
#ifndef VSR_FUSED_TMAX
#define VSR_FUSED_TMAX 8
#endif

template <int L, int A>
struct FShape {
    static constexpr int P = fftc::Plan<L, FR>::P;
    static constexpr int TMAX = (4096 / (L * A)) > 0 ? (4096 / (L * A)) : 1;
    // the A alias lanes of one (g1, t) must sit in one warp: T * A <= 32
    static constexpr int TW = (32 / A) > 0 ? (32 / A) : 1;
    static constexpr int T0 = TMAX > VSR_FUSED_TMAX ? VSR_FUSED_TMAX : TMAX;
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
                      SepTables sep,
                      const double2* __restrict__ xbh, const double2* __restrict__ Zl, double2* W, double2* out,
                      GammaTables tabs,
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
    if (sep.a) {
        const double2 ab = cmul(__ldg(sep.a + f1), __ldg(sep.b + f2));
#pragma unroll
        for (int r = 0; r < R; ++r) Lm[r] = cmul(ab, __ldg(sep.c + (t + P * r)));
    } else {
#pragma unroll
        for (int r = 0; r < R; ++r) Lm[r] = __ldg(lam + base + stride * (t + P * r));
    }
    if constexpr (!TV) {
        if (Zl) {  // prior on the decimation lattice: fft3(xbar) = LR spectrum replicated over the aliases
#pragma unroll
            for (int rr = 0; rr < RD; ++rr) {
                const double2 z = __ldg(Zl + g1 + G.ml * (g2 + G.nl * (long long)(t + P * rr)));
#pragma unroll
                for (int bs = 0; bs < DS; ++bs) v[rr + RD * bs] = z;
            }
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) v[r] = __ldg(xbh + base + stride * (t + P * r));
        }
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
                Gg[bs] = rcp_pos((base_g + __ldg(tabs.ns + (t + P * r))) + tabs.tau);
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
        double2 w;
        if constexpr (TV) {
            const double iden = rcp_pos(den);
            w = make_double2(Sx * iden, Sy * iden);
        } else {
            const double iden = rcp_pos(den);
            w = make_double2(Sx * iden, Sy * iden);
        }
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

// ---------------------------------------------------------------- fold + axis 1
// The fold fused with the contiguous axis-1 pass.  A CTA owns T consecutive
// g2 x the A = dc*ds alias rows (g2 + bc nl, g3 + bs sl) of one g3, full rows
// of length m: the br aliases of every g1 sit in one thread (positions q and
// q + br*ml, ml a multiple of P) and the (bc, bs) aliases in adjacent lanes,
// and every HBM access is a 128-byte-plus row segment.
//   TV = false: Tikhonov fold (solvers.cpp:53-62) -> inverse axis-1 FFT -> out
//   TV = true : W -> forward axis-1 FFT (scaled) -> TV fold (:219-233) -> inverse
//               axis-1 FFT -> W (in place), + LR-Parseval data-fit partials
// Lambda waits in the thread's own slots of the exchange buffer during the fold.
template <int L, int A, int DR, int T, bool TV, bool FIT, int RM>
__device__ __forceinline__ void fold_axis1_tile(int tile, FoldGeom G, const double2* __restrict__ Yl, const double2* __restrict__ lam,
                      SepTables sep,
                      const double2* __restrict__ xbh, const double2* __restrict__ Zl, double2* W, double2* out,
                      GammaTables tabs, double cA,
                      double shift, double inv_scale, double invsqrtd, double fwd_scale,
                      const double2* __restrict__ tw, double* __restrict__ fit_partials) {
    using Pl = fftc::Plan<L, RM>;
    constexpr int R = Pl::R, P = Pl::P, NLN = T * A;
    constexpr int RD = R / DR;  // r = rr + RD * br: alias br of g1 = t + P rr
    static_assert(R % DR == 0, "dr must divide the radix");
    extern __shared__ double2 sm[];
    const int tid = threadIdx.x;
    const int ln = tid % NLN, t = tid / NLN;
    const int a = ln % A, ti = ln / A;
    const int bc = a % G.dc, bs = a / G.dc;
    const int ng2 = (int)(G.nl / T);
    int bx2 = tile % ng2, bx3 = tile / ng2;
    if (TV && tabs.tiles) {  // slab-sharded: this rank's tile list
        const int2 tt = tabs.tiles[tile];
        bx2 = tt.x, bx3 = tt.y;
    }
    const long long g2 = (long long)bx2 * T + ti, g3 = bx3;
    const long long f2 = g2 + bc * G.nl, f3 = g3 + bs * G.sl;
    // W / output rows live on local planes (wplane), dense Lambda rows on lplane
    auto wpl = [&](long long z) -> long long { return (TV && tabs.wplane) ? (long long)tabs.wplane[z] : z; };
    const long long rowb = (TV && tabs.lplane) ? G.m * (f2 + G.n * (long long)tabs.lplane[f3]) : G.m * (f2 + G.n * f3);
    // half-spectrum W (tabs.half3): rows past the Nyquist plane are mirrors
    const bool mir = TV && tabs.half3 && 2 * f3 > G.s;
    const long long nf2 = f2 == 0 ? 0 : G.n - f2;  // -f2 mod n (0 <= f2 < n)
    const long long roww = mir ? 0 : G.m * (f2 + G.n * wpl(f3));
    const long long rowb_rd = mir ? G.m * (nf2 + G.n * wpl(G.s - f3)) : roww;
    // Mirror pairing (half3, one LR column per tile): the alias set of LR
    // (g2, g3) and that of (-g2, -g3) give conjugate rows, so only one of the
    // pair runs (role 1) and also stores the other's rows, conjugated; a
    // self-mirror set (role 0) stores its direct rows; role 2 returns at once.
    int role = 0;
    if (TV && tabs.half3 && T == 1) {
        const int mg2 = bx2 == 0 ? 0 : (int)G.nl - bx2, mg3 = bx3 == 0 ? 0 : (int)G.sl - bx3;
        if (mg2 == bx2 && mg3 == bx3)
            role = 0;
        else if (bx3 < mg3 || (bx3 == mg3 && bx2 < mg2))
            role = 1;
        else
            role = 2;
    }
    if (role == 2) {
        if (FIT && tid == 0) fit_partials[tile] = 0.0;
        return;
    }
    // second copy of a row on the Nyquist/zero planes (its mirror is also <= s/2)
    const long long mrow = G.m * (nf2 + G.n * wpl(f3));
    const long long sec = (role == 1 && !mir && (f3 == 0 || 2 * f3 == G.s) && mrow != roww) ? mrow : -1;
    // line-interleaved: a quarter-warp (8 lines at one position) is one 128-B row
    auto sidx = [&](int q) { return q * NLN + ln; };
    // Staged HBM I/O: whole rows move through shared memory (pitch L + 1, bank-
    // conflict free both ways) so every warp access is a contiguous row segment
    // instead of NLN rows x 32 B.
    constexpr int THREADS = NLN * P;
    constexpr bool STAGED = NLN >= 8 && L >= 32 && THREADS % L == 0;
    constexpr int PITCH = L + 1;
    __shared__ long long rowbase_s[NLN];  // HBM offset each line of the tile is read from
    __shared__ bool mir_s[NLN];           // line read as a conjugate mirror
    __shared__ long long sec_s[NLN];      // extra conjugate copy location, -1 if none
    if (tid < NLN) {                      // thread tid owns line ln = tid
        rowbase_s[tid] = rowb_rd;
        mir_s[tid] = mir;
        sec_s[tid] = sec;
    }
    __syncthreads();
    auto row_base = [&](int j) { return rowbase_s[j]; };
    // TV: the per-position tables (blur factor a, Gamma row term, Gw row) go to
    // shared memory by cp.async now, and the per-line scalars to registers, so
    // their latency hides under the W load and the forward FFT
    __shared__ __align__(16) double2 sa_s[TV ? L : 1];
    __shared__ __align__(16) double nr_s[TV ? L : 1];
    __shared__ __align__(16) double gw_s[TV ? T * (L / DR) : 1];  // one Gw row per LR g2 of the tile
    double2 bc_ = make_double2(0.0, 0.0);
    double base_g = 0.0;
    if constexpr (TV) {
        if (sep.a) {
            for (int i = tid; i < L; i += THREADS)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(sa_s + i)),
                             "l"(sep.a + i) : "memory");
            bc_ = cmul(__ldg(sep.b + f2), __ldg(sep.c + f3));
        }
        for (int i = tid; i < L; i += THREADS)
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(nr_s + i)),
                         "l"(tabs.nr + i) : "memory");
        if (tabs.gw)
            for (int i = tid; i < T * (L / DR); i += THREADS) {
                const long long gi2 = (long long)bx2 * T + i / (L / DR);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(gw_s + i)),
                             "l"(tabs.gw + G.ml * (gi2 + G.nl * g3) + i % (L / DR)) : "memory");
            }
        asm volatile("cp.async.commit_group;" ::: "memory");
        base_g = __ldg(tabs.nc + f2) + __ldg(tabs.ns + f3);
    }
    double2 v[R];
    // LR spectrum of y for this row: issued first so its latency overlaps the
    // forward transform
    const double2* Yrow = Yl + G.ml * (g2 + G.nl * g3);
    double2 yr[RD];
#pragma unroll
    for (int rr = 0; rr < RD; ++rr) yr[rr] = __ldg(Yrow + t + P * rr);
    if constexpr (TV) {
        if constexpr (STAGED) {
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const int e = tid + THREADS * k, j = e / L, q = e % L;
                v[k] = W[row_base(j) + q];
                if (mir_s[j]) v[k].y = -v[k].y;
            }
#pragma unroll
            for (int k = 0; k < R; ++k) {
                const int e = tid + THREADS * k, j = e / L, q = e % L;
                sm[j * PITCH + q] = v[k];
            }
            __syncthreads();
#pragma unroll
            for (int r = 0; r < R; ++r) v[r] = sm[ln * PITCH + t + P * r];
            __syncthreads();
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                v[r] = W[rowb_rd + t + P * r];
                if (mir) v[r].y = -v[r].y;
            }
        }
        fftc::stockham<L, false, decltype(sidx), RM>(v, t, sm, sidx, tw);
        fftc::to_natural<L, RM>(v);
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = cscale(v[r], fwd_scale);
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();  // exchange buffer reused for Lambda below; tables landed
    } else if (Zl) {
        const double2* zrow = Zl + G.ml * (g2 + G.nl * g3);
#pragma unroll
        for (int rr = 0; rr < RD; ++rr) {
            const double2 z = __ldg(zrow + t + P * rr);
#pragma unroll
            for (int br = 0; br < DR; ++br) v[rr + RD * br] = z;
        }
    } else {
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = __ldg(xbh + rowb + t + P * r);
    }
#pragma unroll
    if (sep.a) {
        if constexpr (TV) {
#pragma unroll
            for (int r = 0; r < R; ++r) sm[sidx(t + P * r)] = cmul(sa_s[t + P * r], bc_);
        } else {
            const double2 bcv = cmul(__ldg(sep.b + f2), __ldg(sep.c + f3));
#pragma unroll
            for (int r = 0; r < R; ++r) sm[sidx(t + P * r)] = cmul(__ldg(sep.a + (t + P * r)), bcv);
        }
    } else {
#pragma unroll
        for (int r = 0; r < R; ++r) sm[sidx(t + P * r)] = __ldg(lam + rowb + t + P * r);
    }
    double fit = 0.0;
    if constexpr (TV && FIT) {
        if (tabs.fit_only) {  // data fit of the input spectrum only (uniform per launch)
#pragma unroll
            for (int rr = 0; rr < RD; ++rr) {
                double ax = 0.0, ay = 0.0;
#pragma unroll
                for (int br = 0; br < DR; ++br) {
                    const int r = rr + RD * br;
                    const double2 pr = cmul(sm[sidx(t + P * r)], v[r]);
                    ax += pr.x;
                    ay += pr.y;
                }
                ax = lanes_sum<1, A>(ax);
                ay = lanes_sum<1, A>(ay);
                if (a == 0) {
                    const double rx = yr[rr].x - invsqrtd * ax, ry = yr[rr].y - invsqrtd * ay;
                    fit += rx * rx + ry * ry;
                }
            }
            if (role == 1) fit *= 2.0;
            __shared__ double red0[32];
            double vv[1] = {fit};
            block_reduce_sum<1>(vv, red0);
            if (tid == 0) fit_partials[tile] = vv[0];
            return;
        }
    }
    if constexpr (TV) {
        if (tabs.gw) {
            // one cross-alias sum: S = sum_b Lambda_b g_b with g_b = Gamma_b k_b; the
            // denominator Gw + mu d is tabled and the data fit follows from S and w:
            // sum_b Lambda_b x̂_b = (S - Gw w) / mu
            double gwv[RD];
#pragma unroll
            for (int rr = 0; rr < RD; ++rr) gwv[rr] = gw_s[ti * (L / DR) + t + P * rr];
#pragma unroll
            for (int rr = 0; rr < RD; ++rr) {
                const double2 yraw = yr[rr];
                const double2 yv = cscale(yraw, invsqrtd);
                double Gg[DR];
                double Sx = 0.0, Sy = 0.0;
#pragma unroll
                for (int br = 0; br < DR; ++br) {
                    const int r = rr + RD * br;
                    const double2 Lr = sm[sidx(t + P * r)];
                    Gg[br] = rcp_pos((nr_s[t + P * r] + base_g) + tabs.tau);
                    v[r] = cscale(cadd(cmulc(Lr, yv), cscale(v[r], cA)), Gg[br]);
                    const double2 pr = cmul(Lr, v[r]);
                    Sx += pr.x;
                    Sy += pr.y;
                }
                Sx = lanes_sum<1, A>(Sx);
                Sy = lanes_sum<1, A>(Sy);
                const double iden = rcp_pos(gwv[rr] + shift);
                const double2 w = make_double2(Sx * iden, Sy * iden);
#pragma unroll
                for (int br = 0; br < DR; ++br) {
                    const int r = rr + RD * br;
                    const double2 Lr = sm[sidx(t + P * r)];
                    const double2 c = cmul(make_double2(Gg[br] * Lr.x, -(Gg[br] * Lr.y)), w);
                    v[r] = cscale(csub(v[r], c), inv_scale);
                }
                if constexpr (FIT) {
                    if (a == 0) {
                        const double ax = (Sx - gwv[rr] * w.x) * inv_scale, ay = (Sy - gwv[rr] * w.y) * inv_scale;
                        const double rx = yraw.x - invsqrtd * ax, ry = yraw.y - invsqrtd * ay;
                        fit += rx * rx + ry * ry;
                    }
                }
            }
            goto folded;
        }
    }
#pragma unroll
    for (int rr = 0; rr < RD; ++rr) {
        const double2 yraw = yr[rr];
        const double2 yv = cscale(yraw, invsqrtd);
        double Gg[DR];
        double Sx = 0.0, Sy = 0.0, gram = 0.0;
#pragma unroll
        for (int br = 0; br < DR; ++br) {
            const int r = rr + RD * br;
            const double2 Lr = sm[sidx(t + P * r)];
            if constexpr (TV) {
                Gg[br] = 1.0 / ((nr_s[t + P * r] + base_g) + tabs.tau);
                v[r] = cscale(cadd(cmulc(Lr, yv), cscale(v[r], cA)), Gg[br]);
                gram += Gg[br] * cnorm(Lr);
            } else {
                v[r] = cadd(cmulc(Lr, yv), cscale(v[r], cA));
                gram += cnorm(Lr);
            }
            const double2 pr = cmul(Lr, v[r]);
            Sx += pr.x;
            Sy += pr.y;
        }
        Sx = lanes_sum<1, A>(Sx);
        Sy = lanes_sum<1, A>(Sy);
        gram = lanes_sum<1, A>(gram);
        const double den = gram + shift;
        const double2 w = make_double2(Sx / den, Sy / den);
        double ax = 0.0, ay = 0.0;
#pragma unroll
        for (int br = 0; br < DR; ++br) {
            const int r = rr + RD * br;
            const double2 Lr = sm[sidx(t + P * r)];
            double2 c;
            if constexpr (TV)
                c = cmul(make_double2(Gg[br] * Lr.x, -(Gg[br] * Lr.y)), w);
            else
                c = cmulc(Lr, w);
            v[r] = cscale(csub(v[r], c), inv_scale);
            if constexpr (FIT) {
                const double2 pr = cmul(Lr, v[r]);
                ax += pr.x;
                ay += pr.y;
            }
        }
        if constexpr (FIT) {
            ax = lanes_sum<1, A>(ax);
            ay = lanes_sum<1, A>(ay);
            if (a == 0) {
                const double rx = yraw.x - invsqrtd * ax, ry = yraw.y - invsqrtd * ay;
                fit += rx * rx + ry * ry;
            }
        }
    }
folded:
    __syncthreads();
    fftc::stockham<L, true, decltype(sidx), RM>(v, t, sm, sidx, tw);
    double2* dst = (TV && out == nullptr) ? W : out;  // TV: in place unless a separate output is given
    if constexpr (STAGED) {
#pragma unroll
        for (int j = 0; j < R; ++j) sm[ln * PITCH + Pl::out_q(t, j)] = v[j];
        __syncthreads();
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const int e = tid + THREADS * k, j = e / L, q = e % L;
            const double2 val = sm[j * PITCH + q];
            if (!mir_s[j])
                dst[row_base(j) + q] = val;
            else if (role == 1)
                dst[row_base(j) + q] = make_double2(val.x, -val.y);
            if (sec_s[j] >= 0) dst[sec_s[j] + q] = make_double2(val.x, -val.y);
        }
    } else {
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const double2 val = v[j];
            if (!mir)
                dst[(TV ? roww : rowb) + Pl::out_q(t, j)] = val;
            else if (role == 1)
                dst[rowb_rd + Pl::out_q(t, j)] = make_double2(val.x, -val.y);
            if (sec >= 0) dst[sec + Pl::out_q(t, j)] = make_double2(val.x, -val.y);
        }
    }
    if (role == 1) fit *= 2.0;  // the skipped mirror set has the same |residual|^2
    if constexpr (FIT) {
        __shared__ double red[32];
        double vv[1] = {fit};
        block_reduce_sum<1>(vv, red);
        if (tid == 0) fit_partials[tile] = vv[0];
    }
}


// Persistent wrapper: a CTA walks tiles tile0, tile0 + grid, ... and, for the
// TV sandwich, asks the TMA unit to pull the next tile's rows into L2
// (cp.async.bulk.prefetch) while the current tile computes.
template <int L, int A, int DR, int T, bool TV, bool FIT, int RM>
__global__ void __launch_bounds__(T * A * (L / RM), ((RM == 8 ? 1024 : 512) / (T * A * (L / RM))) > 0 ? (RM == 8 ? 1024 : 512) / (T * A * (L / RM)) : 1)
    fold_axis1_kernel(int ntiles, FoldGeom G, const double2* __restrict__ Yl, const double2* __restrict__ lam,
                      SepTables sep, const double2* __restrict__ xbh, const double2* __restrict__ Zl, double2* W,
                      double2* out, GammaTables tabs, double cA, double shift, double inv_scale, double invsqrtd,
                      double fwd_scale, const double2* __restrict__ tw, double* __restrict__ fit_partials) {
    constexpr int NLN = T * A;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int next = tile + gridDim.x;
        if (TV && next < ntiles && threadIdx.x < NLN) {
            const int ln = threadIdx.x, a = ln % A, ti = ln / A;
            const int ng2 = (int)(G.nl / T);
            const long long f2 = (long long)(next % ng2) * T + ti + (a % G.dc) * G.nl;
            const long long f3 = (long long)(next / ng2) + (a / G.dc) * G.sl;
            const double2* row = W + G.m * (f2 + G.n * f3);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(row), "r"((unsigned)(L * sizeof(double2)))
                         : "memory");
        }
        fold_axis1_tile<L, A, DR, T, TV, FIT, RM>(tile, G, Yl, lam, sep, xbh, Zl, W, out, tabs, cA, shift, inv_scale,
                                                   invsqrtd, fwd_scale, tw, fit_partials);
        __syncthreads();  // shared buffers are reused by the next tile
    }
}

template <int L, int A, int DR, int RM = 16>
struct A1Shape {
    static constexpr int PP = L / (L < RM ? L : RM);              // threads per line
    static constexpr int T0 = 32 / A > 0 ? 32 / A : 1;          // NLN <= 32 (alias lanes in a warp)
    static constexpr int TT = (T0 * A * PP) > 256 ? (256 / (A * PP) > 0 ? 256 / (A * PP) : 1) : T0;
    static constexpr int T = TT > 2 ? 2 : TT;                    // 2 consecutive g2 per tile
    static constexpr int THREADS = T * A * PP;
    static constexpr bool STAGED = T * A >= 8 && L >= 32 && THREADS % L == 0;  // fold_axis1_kernel
    static constexpr size_t SMEM = (size_t)T * A * (STAGED ? L + 1 : L) * sizeof(double2);
};

template <int L, int A, int DR, bool TV, bool FIT, int RM = 16>
void launch_a1(const FoldGeom& G, const double2* Yl, const double2* lam, const SepTables& sep, const double2* xbh,
               const double2* Zl, double2* W, double2* out, const GammaTables& tabs, double cA, double shift, double inv_scale,
               double fwd_scale, double* fit, cudaStream_t st) {
    using Sh = A1Shape<L, A, DR, RM>;
    auto kern = fold_axis1_kernel<L, A, DR, Sh::T, TV, FIT, RM>;
    if (Sh::SMEM > 48 * 1024)
        VSR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sh::SMEM));
    const int ntiles = (TV && tabs.tiles) ? tabs.ntiles : (int)((G.nl / Sh::T) * G.sl);
    if (ntiles == 0) return;
    const unsigned grid = (unsigned)ntiles;
    kern<<<grid, Sh::THREADS, Sh::SMEM, st>>>(ntiles, G, Yl, lam, sep, xbh, Zl, W, out, tabs, cA, shift, inv_scale,
                                              1.0 / std::sqrt((double)G.d), fwd_scale,
                                              fft_engine().twiddles((size_t)L), fit);
    VSR_LAUNCH_CHECK();
}

// (L = m, A = dc*ds, DR = dr) triples served by fold_axis1_kernel
#define VSR_A1_TABLE(X)                                                                 \
    X(64, 4, 2) X(128, 4, 2) X(256, 4, 2) X(512, 4, 2) X(1024, 4, 2)                      \
    X(64, 8, 2) X(128, 8, 2) X(256, 8, 2) X(512, 8, 2) X(1024, 8, 2)                      \
    X(64, 16, 4) X(128, 16, 4) X(256, 16, 4) X(512, 16, 4)                               \
    X(64, 1, 1) X(128, 1, 1) X(256, 1, 1) X(512, 1, 1) X(1024, 1, 1)

template <bool TV, bool FIT>
bool dispatch_a1(const FoldGeom& G, const double2* Yl, const double2* lam, const SepTables& sep,
                 const double2* xbh, const double2* Zl, double2* W, double2* out, const GammaTables& tabs, double cA, double shift,
                 double inv_scale, double fwd_scale, double* fit, cudaStream_t st) {
    const int A = G.dc * G.ds;
#define VSR_X(LL, AA, DD)                                                                           \
    if (G.m == LL && A == AA && G.dr == DD && G.nl % A1Shape<LL, AA, DD>::T == 0) {                  \
        launch_a1<LL, AA, DD, TV, FIT>(G, Yl, lam, sep, xbh, Zl, W, out, tabs, cA, shift, inv_scale,   \
                                       fwd_scale, fit, st);                                         \
        return true;                                                                                \
    }
    VSR_A1_TABLE(VSR_X)
#undef VSR_X
    return false;
}

// ---------------------------------------------------------------- dispatch
struct Key {
    int L, A, DS;
};

template <int L, int A, int DS, bool TV, bool FIT>
void launch_one(const FoldGeom& G, const double2* Yl, const double2* lam, const SepTables& sep,
                const double2* xbh, const double2* Zl, double2* W, double2* out, const GammaTables& tabs, double cA, double shift,
                double inv_scale, double fwd_scale, double* fit, cudaStream_t st) {
    using Sh = FShape<L, A>;
    auto kern = fold_axis3_kernel<L, A, DS, TV, FIT>;
    const size_t smem = (size_t)Sh::SMEM * sizeof(double2);
    if (smem > 48 * 1024)
        VSR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const unsigned grid = (unsigned)((G.ml / Sh::T) * G.nl);
    kern<<<grid, Sh::THREADS, smem, st>>>(G, Yl, lam, sep, xbh, Zl, W, out, tabs, cA, shift, inv_scale,
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
bool dispatch(const FoldGeom& G, const double2* Yl, const double2* lam, const SepTables& sep,
              const double2* xbh, const double2* Zl, double2* W, double2* out, const GammaTables& tabs, double cA, double shift,
              double inv_scale, double fwd_scale, double* fit, cudaStream_t st) {
    const int A = G.dr * G.dc;
#define VSR_X(LL, AA, DD)                                                                           \
    if (G.s == LL && A == AA && G.ds == DD && G.ml % FShape<LL, AA>::T == 0) {                      \
        launch_one<LL, AA, DD, TV, FIT>(G, Yl, lam, sep, xbh, Zl, W, out, tabs, cA, shift, inv_scale, \
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
                           const double2* xbh, double2* out, double reg, cudaStream_t st, const SepTables& sep,
                           const double2* Zl) {
    GammaTables none{nullptr, nullptr, nullptr, 0.0};
    const double shift = 2.0 * reg * (double)G.d;  // solvers.cpp:43
    const double inv2l = 1.0 / (2.0 * reg);         // solvers.cpp:59
    if (!dispatch<false, false>(G, Yl, lam, sep, xbh, Zl, nullptr, out, none, 2.0 * reg, shift, inv2l, 1.0,
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
                        cudaStream_t st, const SepTables& sep) {
    const double shift = mu * (double)G.d;  // solvers.cpp:238
    const double inv_mu = 1.0 / mu;         // solvers.cpp:230
    const bool ok = fit_partials
                        ? dispatch<true, true>(G, Yl, lam, sep, nullptr, nullptr, W, nullptr, tabs, mu, shift, inv_mu,
                                               fwd_scale, fit_partials, st)
                        : dispatch<true, false>(G, Yl, lam, sep, nullptr, nullptr, W, nullptr, tabs, mu, shift, inv_mu,
                                                fwd_scale, nullptr, st);
    if (!ok) throw std::logic_error("launch_tv_sandwich: unsupported geometry");
}

bool fused_axis1_ok(const FoldGeom& G) {
    const int A = G.dc * G.ds;
#define VSR_X(LL, AA, DD) \
    if (G.m == LL && A == AA && G.dr == DD && G.nl % A1Shape<LL, AA, DD>::T == 0) return true;
    VSR_A1_TABLE(VSR_X)
#undef VSR_X
    return false;
}

void launch_tik_fold_ifft1(const FoldGeom& G, const double2* Yl, const double2* lam, const double2* xbh,
                           double2* out, double reg, cudaStream_t st, const SepTables& sep, const double2* Zl) {
    GammaTables none{nullptr, nullptr, nullptr, 0.0};
    if (!dispatch_a1<false, false>(G, Yl, lam, sep, xbh, Zl, nullptr, out, none, 2.0 * reg, 2.0 * reg * (double)G.d,
                                   1.0 / (2.0 * reg), 1.0, nullptr, st))
        throw std::logic_error("launch_tik_fold_ifft1: unsupported geometry");
}

int tv_sandwich1_tile_g2(const FoldGeom& G) {
    const int A = G.dc * G.ds;
#define VSR_X(LL, AA, DD) \
    if (G.m == LL && A == AA && G.dr == DD) return A1Shape<LL, AA, DD>::T;
    VSR_A1_TABLE(VSR_X)
#undef VSR_X
    return 0;
}

size_t tv_sandwich1_blocks(const FoldGeom& G) {
    const int A = G.dc * G.ds;
#define VSR_X(LL, AA, DD) \
    if (G.m == LL && A == AA && G.dr == DD) return (size_t)((G.nl / A1Shape<LL, AA, DD>::T) * G.sl);
    VSR_A1_TABLE(VSR_X)
#undef VSR_X
    return 0;
}

void launch_tv_sandwich1(const FoldGeom& G, const double2* Yl, const double2* lam, double2* W,
                         const GammaTables& tabs, double mu, double fwd_scale, double* fit_partials,
                         cudaStream_t st, const SepTables& sep, double2* Wout) {
    const double shift = mu * (double)G.d, inv_mu = 1.0 / mu;
    static const bool no_pipe = std::getenv("VSR_NO_PIPE") != nullptr;
    if (!no_pipe && tv_sandwich_pipe(G, Yl, sep, W, Wout, tabs, mu, shift, inv_mu, fwd_scale, fit_partials, st))
        return;
    const bool ok = fit_partials ? dispatch_a1<true, true>(G, Yl, lam, sep, nullptr, nullptr, W, Wout, tabs, mu, shift,
                                                           inv_mu, fwd_scale, fit_partials, st)
                                 : dispatch_a1<true, false>(G, Yl, lam, sep, nullptr, nullptr, W, Wout, tabs, mu, shift,
                                                            inv_mu, fwd_scale, nullptr, st);
    if (!ok) throw std::logic_error("launch_tv_sandwich1: unsupported geometry");
}

}  // namespace vsr
