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

// values per thread of a row transform: radix 8 for the short rows of the
// latency-bound LR stages (M <= 64: 128^3 LR grids), 16 for longer rows
template <int M>
constexpr int row_r() { return M <= 64 ? 8 : 16; }

template <int M>
struct RowShape {
    using Pl = fftc::Plan<M, row_r<M>()>;
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
    double2 wl[R];  // split twiddles, fetched under the transform
#pragma unroll
    for (int j = 0; j < R; ++j) wl[j] = __ldg(twL + fftc::Plan<M, row_r<M>()>::out_q(t, j));
    auto sidx_r = [&](int q) { return ls * Sh::LPAD + q + q / R; };
    fftc::stockham<M, false, decltype(sidx_r), row_r<M>()>(v, t, smr, sidx_r, twM);
    // (the transform's last exchange ends with a barrier: the buffer is free)
    double2* buf = smr + ls * Sh::XPITCH;
#pragma unroll
    for (int j = 0; j < R; ++j) buf[fftc::Plan<M, row_r<M>()>::out_q(t, j)] = v[j];
    __syncthreads();
    if (!active) return;
    double2* out = X + row * Mp;
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int k = fftc::Plan<M, row_r<M>()>::out_q(t, j);
        const double2 a = v[j], b = buf[(M - k) & (M - 1)];  // Z[k] is still in registers
        const double2 e = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
        const double2 o = make_double2(0.5 * (a.y + b.y), -0.5 * (a.x - b.x));  // -i (a - conj b) / 2
        out[k] = cadd(e, cmul(wl[j], o));
    }
    if (t == 0) {
        const double2 a = v[0];  // position 0 (out_q(0, 0) = 0)
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
    double2 wl[R];
#pragma unroll
    for (int r = 0; r < R; ++r) wl[r] = __ldg(twL + t + P * r);
    // the subtrahend (cold in HBM) is fetched now, its latency hidden under the transform
    double2 qv[R];
    const double2* subz = reinterpret_cast<const double2*>(sub) + row * M;
#pragma unroll
    for (int j = 0; j < R; ++j)
        qv[j] = (sub && active) ? __ldg(subz + fftc::Plan<M, row_r<M>()>::out_q(t, j)) : make_double2(0.0, 0.0);
    __syncthreads();
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int k = t + P * r;
        const double2 a = buf[k], b = buf[M - k];
        const double2 s = make_double2(a.x + b.x, a.y - b.y);   // a + conj b
        const double2 d = make_double2(a.x - b.x, a.y + b.y);   // a - conj b
        const double2 w = wl[r];                                // e^{-2 pi i k / L}
        const double2 wd = cmulc(w, d);                         // e^{+2 pi i k / L} d
        v[r] = make_double2(s.x - wd.y, s.y + wd.x);            // s + i wd
    }
    __syncthreads();  // split buffer -> exchange buffer
    auto sidx_r = [&](int q) { return ls * Sh::LPAD + q + q / R; };
    fftc::stockham<M, true, decltype(sidx_r), row_r<M>()>(v, t, smr, sidx_r, twM);
    if (!active) return;
    double2* outz = reinterpret_cast<double2*>(x) + row * M;
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int n = fftc::Plan<M, row_r<M>()>::out_q(t, j);
        outz[n] = csub(cscale(v[j], scale), qv[j]);
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

}  // namespace vsr
