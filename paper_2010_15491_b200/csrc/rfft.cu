// Real <-> half-spectrum transforms along axis 1 (contiguous rows), used by
// the spatial-expansion Tikhonov path's LR stage (spatial.cuh).
//
// A real row x of even length L = 2M is viewed as M complex z[n] = x[2n] +
// i x[2n+1] and transformed by the same register/shared-memory Stockham core
// as the axis passes (fft_core.cuh), then split:
//   E[k] = (Z[k] + conj(Z[M-k])) / 2,  O[k] = -i (Z[k] - conj(Z[M-k])) / 2
//   X[k] = E[k] + e^{-2 pi i k / L} O[k],   k = 0..M      (X[M] = E[0] - O[0])
// The inverse forms C[k] = (X[k] + conj(X[M-k])) + i e^{+2 pi i k / L}
// (X[k] - conj(X[M-k])) and returns x[2n] + i x[2n+1] = IDFT_M(C)[n]: the
// unnormalised length-L inverse of the Hermitian extension of X.
// Half-spectrum rows are stored with pitch Mp >= M + 1 (a multiple of 8 so the
// strided axis-2/3 passes tile it); the pad columns are written as zero.
#include "fft.cuh"
#include "fft_core.cuh"
#include "rfft.cuh"

namespace vsr {
namespace {

template <int M>
struct RowShape {
    using Pl = fftc::Plan<M>;
    static constexpr int R = Pl::R, P = Pl::P;
    static constexpr int TG = P >= 128 ? 1 : 128 / P;  // rows per CTA
    static constexpr int THREADS = TG * P;
    static constexpr int LPAD = M + M / R;            // exchange pitch (bank spread)
    static constexpr int XPITCH = M + 2;              // split/merge row buffer pitch
    static constexpr int SMEM = TG * (LPAD > XPITCH ? LPAD : XPITCH);
};

template <int M>
__global__ void __launch_bounds__(RowShape<M>::THREADS)
    r2c_rows_kernel(const double* __restrict__ x, double2* __restrict__ X, long long rows, int Mp,
                    const double2* __restrict__ twM, const double2* __restrict__ twL) {
    using Sh = RowShape<M>;
    constexpr int R = Sh::R, P = Sh::P;
    extern __shared__ double2 smr[];
    const int tid = threadIdx.x, ls = tid / P, t = tid % P;
    const long long row = (long long)blockIdx.x * Sh::TG + ls;
    const bool active = row < rows;
    const double2* z = reinterpret_cast<const double2*>(x) + row * M;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = active ? __ldg(z + t + P * r) : make_double2(0.0, 0.0);
    fftc::stockham<M, false>(v, t, smr, [&](int q) { return ls * Sh::LPAD + q + q / R; }, twM);
    __syncthreads();  // exchange buffer -> split buffer
    double2* buf = smr + ls * Sh::XPITCH;
#pragma unroll
    for (int j = 0; j < R; ++j) buf[fftc::Plan<M>::out_q(t, j)] = v[j];
    __syncthreads();
    if (!active) return;
    double2* out = X + row * Mp;
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int k = t + P * j;
        const double2 a = buf[k], b = buf[(M - k) & (M - 1)];
        const double2 e = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
        const double2 o = make_double2(0.5 * (a.y + b.y), -0.5 * (a.x - b.x));  // -i (a - conj b) / 2
        out[k] = cadd(e, cmul(__ldg(twL + k), o));
    }
    if (t == 0) {
        const double2 a = buf[0];
        out[M] = make_double2(a.x - a.y, 0.0);  // E[0] - O[0] with E[0] = Re a, O[0] = Im a
    }
    for (int k = M + 1 + t; k < Mp; k += P) out[k] = make_double2(0.0, 0.0);
}

template <int M>
__global__ void __launch_bounds__(RowShape<M>::THREADS)
    c2r_rows_kernel(const double2* __restrict__ X, double* __restrict__ x, long long rows, int Mp, double scale,
                    const double* __restrict__ sub, const double2* __restrict__ twM,
                    const double2* __restrict__ twL) {
    using Sh = RowShape<M>;
    constexpr int R = Sh::R, P = Sh::P;
    extern __shared__ double2 smr[];
    const int tid = threadIdx.x, ls = tid / P, t = tid % P;
    const long long row = (long long)blockIdx.x * Sh::TG + ls;
    const bool active = row < rows;
    double2* buf = smr + ls * Sh::XPITCH;
    const double2* in = X + row * Mp;
#pragma unroll
    for (int j = 0; j < R; ++j) buf[t + P * j] = active ? __ldg(in + t + P * j) : make_double2(0.0, 0.0);
    if (t == 0) buf[M] = active ? __ldg(in + M) : make_double2(0.0, 0.0);
    __syncthreads();
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int k = t + P * r;
        const double2 a = buf[k], b = buf[M - k];
        const double2 s = make_double2(a.x + b.x, a.y - b.y);   // a + conj b
        const double2 d = make_double2(a.x - b.x, a.y + b.y);   // a - conj b
        const double2 w = __ldg(twL + k);                       // e^{-2 pi i k / L}
        const double2 wd = cmulc(w, d);                         // e^{+2 pi i k / L} d
        v[r] = make_double2(s.x - wd.y, s.y + wd.x);            // s + i wd
    }
    __syncthreads();  // split buffer -> exchange buffer
    fftc::stockham<M, true>(v, t, smr, [&](int q) { return ls * Sh::LPAD + q + q / R; }, twM);
    if (!active) return;
    double2* outz = reinterpret_cast<double2*>(x) + row * M;
    const double2* subz = reinterpret_cast<const double2*>(sub) + row * M;
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int n = fftc::Plan<M>::out_q(t, j);
        double2 r = cscale(v[j], scale);
        if (sub) {
            const double2 q = __ldg(subz + n);
            r = csub(r, q);
        }
        outz[n] = r;
    }
}

template <int M>
void launch_r2c(const double* x, double2* X, long long rows, int Mp, cudaStream_t st) {
    using Sh = RowShape<M>;
    const size_t smem = (size_t)Sh::SMEM * sizeof(double2);
    auto kern = r2c_rows_kernel<M>;
    if (smem > 48 * 1024) VSR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const unsigned blocks = (unsigned)((rows + Sh::TG - 1) / Sh::TG);
    kern<<<blocks, Sh::THREADS, smem, st>>>(x, X, rows, Mp, fft_engine().twiddles(M), fft_engine().twiddles(2 * M));
    VSR_LAUNCH_CHECK();
}

template <int M>
void launch_c2r(const double2* X, double* x, long long rows, int Mp, double scale, const double* sub,
                cudaStream_t st) {
    using Sh = RowShape<M>;
    const size_t smem = (size_t)Sh::SMEM * sizeof(double2);
    auto kern = c2r_rows_kernel<M>;
    if (smem > 48 * 1024) VSR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const unsigned blocks = (unsigned)((rows + Sh::TG - 1) / Sh::TG);
    kern<<<blocks, Sh::THREADS, smem, st>>>(X, x, rows, Mp, scale, sub, fft_engine().twiddles(M),
                                            fft_engine().twiddles(2 * M));
    VSR_LAUNCH_CHECK();
}

// ------------------------------------------------------------ plane kernels
// One CTA per z-plane of an LR volume (NY rows of length L = 2M): the row
// r2c transform and the axis-2 (column) transform of the half spectrum run
// back to back in shared memory, so the intermediate never touches L2/HBM.
// The plane lives in smem as NY rows x PITCH = M + 1 (odd: column accesses
// are bank-conflict free); threads without a row/column of their own point
// their exchange slots at a scratch row.
template <int M, int NY>
struct PlaneShape {
    using P1l = fftc::Plan<M>;
    using P2l = fftc::Plan<NY>;
    static constexpr int R1 = P1l::R, P1 = P1l::P, R2 = P2l::R, P2 = P2l::P;
    static constexpr int PITCH = M + 1;
    static constexpr int T1 = NY * P1;                         // row phase threads
    static constexpr int COLS = (M + 1 + 3) / 4 * 4;
    static constexpr int T2 = COLS * P2;                       // column phase threads
    static constexpr int THREADS = ((T1 > T2 ? T1 : T2) + 31) / 32 * 32;
    static constexpr int SCRATCH = (NY > M ? NY : M) + 1;
    static constexpr int SMEM = NY * PITCH + SCRATCH;           // double2 elements
};

template <int M, int NY>
__global__ void __launch_bounds__(PlaneShape<M, NY>::THREADS, 1)
    lr_plane_fwd_kernel(const double* __restrict__ y, double2* __restrict__ Yh, int Mp,
                        const double2* __restrict__ twM, const double2* __restrict__ twL,
                        const double2* __restrict__ twN) {
    using Sh = PlaneShape<M, NY>;
    constexpr int R1 = Sh::R1, P1 = Sh::P1, R2 = Sh::R2, P2 = Sh::P2, PITCH = Sh::PITCH;
    extern __shared__ double2 pl[];
    double2* scratch = pl + NY * PITCH;
    const int tid = threadIdx.x;
    const long long plane = blockIdx.x;
    // ---- rows: z = x[2n] + i x[2n+1], M-point FFT, Hermitian split
    {
        const int row = tid / P1, t = tid % P1;
        const bool act = row < NY;
        const double2* zr = reinterpret_cast<const double2*>(y) + (plane * NY + row) * M;
        double2 v[R1];
#pragma unroll
        for (int r = 0; r < R1; ++r) v[r] = act ? __ldg(zr + t + P1 * r) : make_double2(0.0, 0.0);
        fftc::stockham<M, false>(v, t, pl, [&](int q) { return act ? row * PITCH + q : (int)(scratch - pl) + (q % Sh::SCRATCH); }, twM);
        __syncthreads();
        if (act) {
#pragma unroll
            for (int j = 0; j < R1; ++j) pl[row * PITCH + fftc::Plan<M>::out_q(t, j)] = v[j];
        }
        __syncthreads();
        if (act) {
            double2* rz = pl + row * PITCH;
            for (int k = t; k <= M / 2; k += P1) {
                const double2 a = rz[k], b = rz[(M - k) & (M - 1)];
                const double2 e = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
                const double2 o = make_double2(0.5 * (a.y + b.y), -0.5 * (a.x - b.x));
                const double2 xk = cadd(e, cmul(__ldg(twL + k), o));
                if (k == 0) {
                    rz[0] = make_double2(a.x + a.y, 0.0);
                    rz[M] = make_double2(a.x - a.y, 0.0);
                } else if (2 * k == M) {
                    rz[k] = xk;
                } else {
                    // X[M-k] = conj(E_k) + e^{-2 pi i (M-k)/L} conj(O_k)
                    const double2 xm = cadd(make_double2(e.x, -e.y),
                                            cmul(__ldg(twL + (M - k)), make_double2(o.x, -o.y)));
                    rz[k] = xk;
                    rz[M - k] = xm;
                }
            }
        }
        __syncthreads();
    }
    // ---- columns: NY-point FFT of each of the M + 1 columns, in place
    {
        const int col = tid / P2, t = tid % P2;
        const bool act = col <= M;
        double2 v[R2];
#pragma unroll
        for (int r = 0; r < R2; ++r) v[r] = act ? pl[(t + P2 * r) * PITCH + col] : make_double2(0.0, 0.0);
        __syncthreads();
        fftc::stockham<NY, false>(v, t, pl, [&](int q) { return act ? q * PITCH + col : (int)(scratch - pl) + (q % Sh::SCRATCH); }, twN);
        __syncthreads();
        if (act) {
#pragma unroll
            for (int j = 0; j < R2; ++j) pl[fftc::Plan<NY>::out_q(t, j) * PITCH + col] = v[j];
        }
        __syncthreads();
    }
    // ---- coalesced store of the half-spectrum plane (pad columns zero)
    double2* out = Yh + plane * NY * Mp;
    for (int e = tid; e < NY * Mp; e += Sh::THREADS) {
        const int row = e / Mp, k = e - row * Mp;
        out[e] = k <= M ? pl[row * PITCH + k] : make_double2(0.0, 0.0);
    }
}

template <int M, int NY>
__global__ void __launch_bounds__(PlaneShape<M, NY>::THREADS, 1)
    lr_plane_inv_kernel(const double2* __restrict__ Yh, double* __restrict__ u, int Mp, double scale,
                        const double* __restrict__ sub, const double2* __restrict__ twM,
                        const double2* __restrict__ twL, const double2* __restrict__ twN) {
    using Sh = PlaneShape<M, NY>;
    constexpr int R1 = Sh::R1, P1 = Sh::P1, R2 = Sh::R2, P2 = Sh::P2, PITCH = Sh::PITCH;
    extern __shared__ double2 pl[];
    double2* scratch = pl + NY * PITCH;
    const int tid = threadIdx.x;
    const long long plane = blockIdx.x;
    const double2* in = Yh + plane * NY * Mp;
    for (int e = tid; e < NY * Mp; e += Sh::THREADS) {
        const int row = e / Mp, k = e - row * Mp;
        if (k <= M) pl[row * PITCH + k] = __ldg(in + e);
    }
    __syncthreads();
    // ---- columns: inverse NY-point FFT in place
    {
        const int col = tid / P2, t = tid % P2;
        const bool act = col <= M;
        double2 v[R2];
#pragma unroll
        for (int r = 0; r < R2; ++r) v[r] = act ? pl[(t + P2 * r) * PITCH + col] : make_double2(0.0, 0.0);
        __syncthreads();
        fftc::stockham<NY, true>(v, t, pl, [&](int q) { return act ? q * PITCH + col : (int)(scratch - pl) + (q % Sh::SCRATCH); }, twN);
        __syncthreads();
        if (act) {
#pragma unroll
            for (int j = 0; j < R2; ++j) pl[fftc::Plan<NY>::out_q(t, j) * PITCH + col] = v[j];
        }
        __syncthreads();
    }
    // ---- rows: Hermitian merge, inverse M-point FFT, x[2n] + i x[2n+1]
    {
        const int row = tid / P1, t = tid % P1;
        const bool act = row < NY;
        double2 v[R1];
        if (act) {
            const double2* rz = pl + row * PITCH;
#pragma unroll
            for (int r = 0; r < R1; ++r) {
                const int k = t + P1 * r;
                const double2 a = rz[k], b = rz[M - k];
                const double2 sm_ = make_double2(a.x + b.x, a.y - b.y);
                const double2 d = make_double2(a.x - b.x, a.y + b.y);
                const double2 wd = cmulc(__ldg(twL + k), d);
                v[r] = make_double2(sm_.x - wd.y, sm_.y + wd.x);
            }
        } else {
#pragma unroll
            for (int r = 0; r < R1; ++r) v[r] = make_double2(0.0, 0.0);
        }
        __syncthreads();
        fftc::stockham<M, true>(v, t, pl, [&](int q) { return act ? row * PITCH + q : (int)(scratch - pl) + (q % Sh::SCRATCH); }, twM);
        if (act) {
            double2* oz = reinterpret_cast<double2*>(u) + (plane * NY + row) * M;
            const double2* sz = reinterpret_cast<const double2*>(sub) + (plane * NY + row) * M;
#pragma unroll
            for (int j = 0; j < R1; ++j) {
                const int n = fftc::Plan<M>::out_q(t, j);
                double2 r = cscale(v[j], scale);
                if (sub) r = csub(r, __ldg(sz + n));
                oz[n] = r;
            }
        }
    }
}

template <int M, int NY>
void launch_plane(bool fwd, const double* y, double2* Yh, double* u, long long planes, int Mp, double scale,
                  const double* sub, cudaStream_t st) {
    using Sh = PlaneShape<M, NY>;
    const size_t smem = (size_t)Sh::SMEM * sizeof(double2);
    const double2 *twM = fft_engine().twiddles(M), *twL = fft_engine().twiddles(2 * M),
                  *twN = fft_engine().twiddles(NY);
    if (fwd) {
        auto kern = lr_plane_fwd_kernel<M, NY>;
        VSR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<(unsigned)planes, Sh::THREADS, smem, st>>>(y, Yh, Mp, twM, twL, twN);
    } else {
        auto kern = lr_plane_inv_kernel<M, NY>;
        VSR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<(unsigned)planes, Sh::THREADS, smem, st>>>(Yh, u, Mp, scale, sub, twM, twL, twN);
    }
    VSR_LAUNCH_CHECK();
}

#define VSR_PLANE_TABLE(X) X(16, 32) X(32, 32) X(32, 64) X(64, 64) X(64, 128) X(128, 64)

}  // namespace

bool rfft_rows_ok(size_t L) { return L >= 16 && L <= 2048 && is_pow2(L); }

int half_pitch(size_t L) { return (int)(((L / 2 + 1) + 7) / 8 * 8); }

void rfft_rows_forward(size_t L, const double* x, double2* X, long long rows, cudaStream_t st) {
    const int Mp = half_pitch(L);
    switch (L / 2) {
        case 8: launch_r2c<8>(x, X, rows, Mp, st); break;
        case 16: launch_r2c<16>(x, X, rows, Mp, st); break;
        case 32: launch_r2c<32>(x, X, rows, Mp, st); break;
        case 64: launch_r2c<64>(x, X, rows, Mp, st); break;
        case 128: launch_r2c<128>(x, X, rows, Mp, st); break;
        case 256: launch_r2c<256>(x, X, rows, Mp, st); break;
        case 512: launch_r2c<512>(x, X, rows, Mp, st); break;
        case 1024: launch_r2c<1024>(x, X, rows, Mp, st); break;
        default: throw std::logic_error("rfft_rows_forward: unsupported length");
    }
}

void rfft_rows_inverse(size_t L, const double2* X, double* x, long long rows, double scale, const double* sub,
                       cudaStream_t st) {
    const int Mp = half_pitch(L);
    switch (L / 2) {
        case 8: launch_c2r<8>(X, x, rows, Mp, scale, sub, st); break;
        case 16: launch_c2r<16>(X, x, rows, Mp, scale, sub, st); break;
        case 32: launch_c2r<32>(X, x, rows, Mp, scale, sub, st); break;
        case 64: launch_c2r<64>(X, x, rows, Mp, scale, sub, st); break;
        case 128: launch_c2r<128>(X, x, rows, Mp, scale, sub, st); break;
        case 256: launch_c2r<256>(X, x, rows, Mp, scale, sub, st); break;
        case 512: launch_c2r<512>(X, x, rows, Mp, scale, sub, st); break;
        case 1024: launch_c2r<1024>(X, x, rows, Mp, scale, sub, st); break;
        default: throw std::logic_error("rfft_rows_inverse: unsupported length");
    }
}

bool lr_plane_ok(size_t L, size_t ny) {
#define VSR_X(MM, NN) \
    if (L == 2 * MM && ny == NN) return true;
    VSR_PLANE_TABLE(VSR_X)
#undef VSR_X
    return false;
}

void lr_plane_forward(size_t L, size_t ny, const double* y, double2* Yh, long long planes, cudaStream_t st) {
#define VSR_X(MM, NN)                                                                       \
    if (L == 2 * MM && ny == NN) {                                                          \
        launch_plane<MM, NN>(true, y, Yh, nullptr, planes, half_pitch(L), 1.0, nullptr, st); \
        return;                                                                             \
    }
    VSR_PLANE_TABLE(VSR_X)
#undef VSR_X
    throw std::logic_error("lr_plane_forward: unsupported plane");
}

void lr_plane_inverse(size_t L, size_t ny, const double2* Yh, double* u, long long planes, double scale,
                      const double* sub, cudaStream_t st) {
#define VSR_X(MM, NN)                                                                                        \
    if (L == 2 * MM && ny == NN) {                                                                           \
        launch_plane<MM, NN>(false, nullptr, const_cast<double2*>(Yh), u, planes, half_pitch(L), scale, sub, st); \
        return;                                                                                              \
    }
    VSR_PLANE_TABLE(VSR_X)
#undef VSR_X
    throw std::logic_error("lr_plane_inverse: unsupported plane");
}

}  // namespace vsr
