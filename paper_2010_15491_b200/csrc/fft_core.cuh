// Register/shared-memory Stockham core of the fp64 FFT engine, shared by the
// plain axis-pass kernels (fft.cu) and the fused fold kernels (fused.cu).
//
// A line of length L (power of two, 2..2048) is served by P = L / R threads
// (R = min(L, 16) values per thread).  On entry thread t holds the line in
// natural order, v[r] = x[t + P r]; stages are radix-R Stockham steps with
// shared-memory exchanges, then an optional final radix RL < R stage.  On
// exit v is in "output order": v[vv * RSL + r] = X[t + P vv + (L / RSL) r].
// to_natural() permutes that back to v[k] = X[t + P k] (register renaming).
#pragma once

#include "vsr_common.cuh"

namespace vsr {
namespace fftc {

__device__ constexpr double kC8[8] = {1.0,
                                      0.9807852804032304,
                                      0.9238795325112867,
                                      0.8314696123025452,
                                      0.7071067811865476,
                                      0.5555702330196022,
                                      0.3826834323650898,
                                      0.19509032201612828};

// exp(-+2 pi i k / 32) * v, k in [0, 16); k is a compile-time constant after
// unrolling so every branch folds away.  C = double2 or float2 (fp32 mode).
template <bool INV, class C>
__device__ __forceinline__ C twiddle32(C v, int k) {
    using T = typename CplxT<C>::real;
    if (k == 0) return v;
    if (k == 8) return INV ? cmake<C>(-v.y, v.x) : cmake<C>(v.y, -v.x);
    T c, s;  // cos, sin of 2*pi*k/32
    if (k < 8) {
        c = (T)kC8[k];
        s = (T)kC8[8 - k];
    } else {
        c = -(T)kC8[16 - k];
        s = (T)kC8[k - 8];
    }
    if (INV) return cmake<C>(v.x * c - v.y * s, v.y * c + v.x * s);
    return cmake<C>(v.x * c + v.y * s, v.y * c - v.x * s);
}

template <int R>
__host__ __device__ constexpr int bitrev(int i) {
    int r = 0;
    for (int b = 1; b < R; b <<= 1) {
        r = (r << 1) | (i & 1);
        i >>= 1;
    }
    return r;
}

// In-register radix-R DFT (R = 1..32, power of two), natural order in/out.
template <int R, bool INV, class C>
__device__ __forceinline__ void dft_reg(C* a) {
    if constexpr (R > 1) {
        C b[R];
#pragma unroll
        for (int i = 0; i < R; ++i) b[bitrev<R>(i)] = a[i];
#pragma unroll
        for (int h = 1; h < R; h <<= 1) {
#pragma unroll
            for (int i = 0; i < R; i += 2 * h) {
#pragma unroll
                for (int j = 0; j < h; ++j) {
                    const C u = b[i + j];
                    const C t = twiddle32<INV>(b[i + j + h], j * (16 / h));
                    b[i + j] = cadd(u, t);
                    b[i + j + h] = csub(u, t);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < R; ++i) a[i] = b[i];
    }
}

__host__ __device__ constexpr int ilog2(int v) { return v <= 1 ? 0 : 1 + ilog2(v >> 1); }

// Barrier used between Stockham stages: the whole CTA by default; the
// pipelined sandwich (sandwich.cu) passes a named barrier per thread group.
struct CtaSync {
    __device__ __forceinline__ void operator()() const { __syncthreads(); }
};

// Twiddle table access: a global table through the read-only path, or a
// copy in shared memory (TwShared).
template <class C = double2>
struct TwShared {
    const C* p;
};
__device__ __forceinline__ double2 tw_at(const double2* __restrict__ p, int i) { return __ldg(p + i); }
__device__ __forceinline__ float2 tw_at(const float2* __restrict__ p, int i) { return __ldg(p + i); }
template <class C>
__device__ __forceinline__ C tw_at(const TwShared<C>& s, int i) { return s.p[i]; }

template <int L, int RMAX = 16>
struct Plan {
    static constexpr int R = L < RMAX ? L : RMAX;
    static constexpr int P = L / R;
    static constexpr int LOGL = ilog2(L), LOGR = ilog2(R);
    static constexpr int K = LOGL / LOGR;               // full radix-R stages
    static constexpr int RL = 1 << (LOGL - K * LOGR);  // final small radix (1 = none)
    static constexpr int NSTAGE = K + (RL > 1 ? 1 : 0);
    static constexpr int RSL = RL > 1 ? RL : R;        // radix of the last stage
    static constexpr int NBL = R / RSL;                // butterflies per thread, last stage
    static constexpr bool NEEDS_SMEM = NSTAGE > 1;
    // line position held in output-order slot j
    __device__ static __forceinline__ int out_q(int t, int j) {
        return t + P * (j / RSL) + (L / RSL) * (j % RSL);
    }
};

// Full line transform.  All threads of the CTA must call it (it syncs when
// NSTAGE > 1).  sidx(q) maps a line position to this thread's line slot in sm.
template <int L, bool INV, class SIdx, int RMAX = 16, class Sync = CtaSync, class Tw = const double2*, class C>
__device__ __forceinline__ void stockham(C* v, int t, C* sm, const SIdx& sidx, Tw tw, const Sync& sync = Sync()) {
    using Pl = Plan<L, RMAX>;
    constexpr int R = Pl::R, P = Pl::P;
    int Ns = 1;
#pragma unroll
    for (int stage = 0; stage < Pl::NSTAGE; ++stage) {
        const bool last = stage == Pl::NSTAGE - 1;
        const int RS = (stage < Pl::K) ? R : Pl::RL;
        const int NB = R / RS;
#pragma unroll
        for (int vv = 0; vv < NB; ++vv) {
            const int u = t + P * vv;
            const int k = u & (Ns - 1);
            if (stage > 0) {
                const int tstride = L / (Ns * RS);
#pragma unroll
                for (int r = 1; r < R; ++r) {
                    if (r < RS) {
                        const C w = tw_at(tw, (r * k * tstride) & (L - 1));
                        const C a = v[vv * RS + r];
                        v[vv * RS + r] = INV ? cmulc(w, a) : cmul(w, a);
                    }
                }
            }
            if (RS == R)
                dft_reg<R, INV>(v);
            else if (RS == Pl::RL)
                dft_reg<(Pl::RL > 1 ? Pl::RL : 1), INV>(v + vv * RS);
        }
        if (!last) {
#pragma unroll
            for (int vv = 0; vv < NB; ++vv) {
                const int u = t + P * vv;
                const int k = u & (Ns - 1);
                const int ob = (u - k) * RS + k;
#pragma unroll
                for (int r = 0; r < R; ++r)
                    if (r < RS) sm[sidx(ob + r * Ns)] = v[vv * RS + r];
            }
            sync();
            Ns *= RS;
            const int RSn = (stage + 1 < Pl::K) ? R : Pl::RL;
            const int NBn = R / RSn;
#pragma unroll
            for (int vv = 0; vv < NBn; ++vv) {
                const int u = t + P * vv;
#pragma unroll
                for (int r = 0; r < R; ++r)
                    if (r < RSn) v[vv * RSn + r] = sm[sidx(u + (L / RSn) * r)];
            }
            sync();
        } else {
            Ns *= RS;
        }
    }
}

// The same transform with the exchanges split into a real and an imaginary
// round through a buffer of REALS (half the shared memory of stockham(), four
// barriers per exchange instead of two).  sidx(q) maps a line position to this
// thread's line slot in smr.  Used by the wide-tile passes of long lines, where
// the full complex exchange buffer would leave no room for the prefetch stage.
template <int L, bool INV, class SIdx, int RMAX = 16, class Sync = CtaSync, class Tw = const double2*, class C>
__device__ __forceinline__ void stockham_split(C* v, int t, typename CplxT<C>::real* smr, const SIdx& sidx, Tw tw,
                                               const Sync& sync = Sync()) {
    using Pl = Plan<L, RMAX>;
    constexpr int R = Pl::R, P = Pl::P;
    int Ns = 1;
#pragma unroll
    for (int stage = 0; stage < Pl::NSTAGE; ++stage) {
        const bool last = stage == Pl::NSTAGE - 1;
        const int RS = (stage < Pl::K) ? R : Pl::RL;
        const int NB = R / RS;
#pragma unroll
        for (int vv = 0; vv < NB; ++vv) {
            const int u = t + P * vv;
            const int k = u & (Ns - 1);
            if (stage > 0) {
                const int tstride = L / (Ns * RS);
#pragma unroll
                for (int r = 1; r < R; ++r) {
                    if (r < RS) {
                        const C w = tw_at(tw, (r * k * tstride) & (L - 1));
                        const C a = v[vv * RS + r];
                        v[vv * RS + r] = INV ? cmulc(w, a) : cmul(w, a);
                    }
                }
            }
            if (RS == R)
                dft_reg<R, INV>(v);
            else if (RS == Pl::RL)
                dft_reg<(Pl::RL > 1 ? Pl::RL : 1), INV>(v + vv * RS);
        }
        if (!last) {
            const int RSn = (stage + 1 < Pl::K) ? R : Pl::RL;
            const int NBn = R / RSn;
#pragma unroll
            for (int comp = 0; comp < 2; ++comp) {
#pragma unroll
                for (int vv = 0; vv < NB; ++vv) {
                    const int u = t + P * vv;
                    const int k = u & (Ns - 1);
                    const int ob = (u - k) * RS + k;
#pragma unroll
                    for (int r = 0; r < R; ++r)
                        if (r < RS) smr[sidx(ob + r * Ns)] = comp ? v[vv * RS + r].y : v[vv * RS + r].x;
                }
                sync();
#pragma unroll
                for (int vv = 0; vv < NBn; ++vv) {
                    const int u = t + P * vv;
#pragma unroll
                    for (int r = 0; r < R; ++r)
                        if (r < RSn) {
                            // (the other component of this slot still holds its
                            // pre-exchange value until its own round)
                            if (comp)
                                v[vv * RSn + r].y = smr[sidx(u + (L / RSn) * r)];
                            else
                                v[vv * RSn + r].x = smr[sidx(u + (L / RSn) * r)];
                        }
                }
                sync();
            }
            Ns *= RS;
        } else {
            Ns *= RS;
        }
    }
}

// Output order -> natural order (v[k] = X[t + P k]); compile-time permutation.
template <int L, int RMAX = 16, class C>
__device__ __forceinline__ void to_natural(C* v) {
    using Pl = Plan<L, RMAX>;
    if constexpr (Pl::RL > 1) {
        C o[Pl::R];
#pragma unroll
        for (int j = 0; j < Pl::R; ++j) o[(j / Pl::RSL) + Pl::NBL * (j % Pl::RSL)] = v[j];
#pragma unroll
        for (int j = 0; j < Pl::R; ++j) v[j] = o[j];
    }
}

}  // namespace fftc
}  // namespace vsr
