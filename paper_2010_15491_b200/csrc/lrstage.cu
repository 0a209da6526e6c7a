// Persistent LR stage of the spatial-expansion Tikhonov solve (spatial.cuh):
// the five half-spectrum LR steps of one solve in ONE cooperative kernel,
//   1. r2c rows (axis 1)                      y -> Yh   (rfft.cu semantics)
//   2. forward axis-2 FFT of Yh               (in place)
//   3. axis-3 forward FFT, x 1/(G2 + 2 reg d) x cfac, inverse FFT (in place)
//   4. inverse axis-2 FFT                     (in place)
//   5. c2r rows minus the constant prior term q -> u
// with a grid-wide barrier between steps.  The LR volume is L2-resident, so
// each step is a few microseconds of work; as five separate launches the
// per-kernel ramp-up and tail dominated (~77 us at 128^3).  Every CTA has 128
// threads and walks the step's work units grid-stride; the unit bodies are the
// same Stockham register/shared-memory code as the standalone kernels.
#include <cooperative_groups.h>

#include "fft.cuh"
#include "fft_core.cuh"
#include "lrstage.cuh"
#include "rfft.cuh"

namespace cg = cooperative_groups;

namespace vsr {
namespace {

constexpr int LS_THREADS = 128;

struct LrArgs {
    const double* y;       // LR real input (ml x nl x sl)
    double2* Yh;           // half spectrum (Mp x nl x sl)
    double* u;             // LR real output
    const double* q;       // constant prior term (subtracted), may be null
    const double* a2;      // per-axis alias sums |a|^2 (ml), |b|^2 (nl), |c|^2 (sl)
    const double* b2;
    const double* c2;
    double cfac, shift;    // filter: cfac / (G2 + shift)
    int Mp;
    const double2 *twM, *twL, *twN, *twZ;
};

// ---- step 1: r2c rows; unit = 32 rows of M complex (P = M / R threads each)
template <int M>
__device__ __forceinline__ void r2c_unit(const LrArgs& A, long long unit, long long rows, double2* sm) {
    using Pl = fftc::Plan<M>;
    constexpr int R = Pl::R, P = Pl::P, TG = LS_THREADS / P, LPAD = M + M / R, XP = M + 2;
    const int tid = threadIdx.x, ls = tid / P, t = tid % P;
    const long long row = unit * TG + ls;
    const bool active = row < rows;
    const double2* z = reinterpret_cast<const double2*>(A.y) + row * M;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = active ? __ldg(z + t + P * r) : make_double2(0.0, 0.0);
    fftc::stockham<M, false>(v, t, sm, [&](int q) { return ls * LPAD + q + q / R; }, A.twM);
    __syncthreads();
    double2* buf = sm + ls * XP;
#pragma unroll
    for (int j = 0; j < R; ++j) buf[Pl::out_q(t, j)] = v[j];
    __syncthreads();
    if (active) {
        double2* out = A.Yh + row * A.Mp;
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int k = t + P * j;
            const double2 a = buf[k], b = buf[(M - k) & (M - 1)];
            const double2 e = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
            const double2 o = make_double2(0.5 * (a.y + b.y), -0.5 * (a.x - b.x));
            out[k] = cadd(e, cmul(__ldg(A.twL + k), o));
        }
        if (t == 0) out[M] = make_double2(buf[0].x - buf[0].y, 0.0);
        for (int k = M + 1 + t; k < A.Mp; k += P) out[k] = make_double2(0.0, 0.0);
    }
    __syncthreads();  // the unit's shared memory is reused by the next unit
}

// ---- steps 2/4: strided axis-2 pass on the half spectrum, in place.
// unit = TG tiles of 8 consecutive columns k at one plane.
template <int NY, bool INV>
__device__ __forceinline__ void col_unit(const LrArgs& A, long long unit, long long tiles, double2* sm) {
    using Pl = fftc::Plan<NY>;
    constexpr int R = Pl::R, P = Pl::P, T = 8, TG = LS_THREADS / (T * P);
    const int tid = threadIdx.x, g = tid / (T * P), rem = tid % (T * P), lt = rem % T, t = rem / T;
    const long long tile = unit * TG + g;
    const bool active = tile < tiles;
    const long long tpp = A.Mp / T;  // tiles per plane
    const long long z = active ? tile / tpp : 0, k0 = active ? (tile % tpp) * T : 0;
    double2* base = A.Yh + z * (long long)A.Mp * NY + k0 + lt;
    auto sidx = [&](int q) { return g * (NY * T) + q * T + lt; };
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = active ? base[(long long)A.Mp * (t + P * r)] : make_double2(0.0, 0.0);
    fftc::stockham<NY, INV>(v, t, sm, sidx, A.twN);
    if (active) {
#pragma unroll
        for (int j = 0; j < R; ++j) base[(long long)A.Mp * Pl::out_q(t, j)] = v[j];
    }
    __syncthreads();
}

// ---- step 3: axis-3 filter sandwich; unit = TG tiles of 8 consecutive
// positions p of the (Mp x NY) plane
template <int NZ>
__device__ __forceinline__ void filter_unit(const LrArgs& A, long long unit, long long tiles, int ny, double2* sm) {
    using Pl = fftc::Plan<NZ>;
    constexpr int R = Pl::R, P = Pl::P, T = 8, TG = LS_THREADS / (T * P) > 0 ? LS_THREADS / (T * P) : 1;
    const int tid = threadIdx.x, g = tid / (T * P), rem = tid % (T * P), lt = rem % T, t = rem / T;
    const long long tile = unit * TG + g;
    const bool active = tile < tiles && g < TG;
    const long long S = (long long)A.Mp * ny;
    const long long p = active ? tile * T + lt : 0;
    auto sidx = [&](int q) { return g * (NZ * T) + q * T + lt; };
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = active ? A.Yh[p + S * (t + P * r)] : make_double2(0.0, 0.0);
    fftc::stockham<NZ, false>(v, t, sm, sidx, A.twZ);
    fftc::to_natural<NZ>(v);
    const int g1 = (int)(p % A.Mp), g2 = (int)(p / A.Mp);
    const double ab2 = __ldg(A.a2 + g1) * __ldg(A.b2 + g2);
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = cscale(v[r], A.cfac / (ab2 * __ldg(A.c2 + t + P * r) + A.shift));
    __syncthreads();
    fftc::stockham<NZ, true>(v, t, sm, sidx, A.twZ);
    if (active) {
#pragma unroll
        for (int j = 0; j < R; ++j) A.Yh[p + S * Pl::out_q(t, j)] = v[j];
    }
    __syncthreads();
}

// ---- step 5: c2r rows minus q
template <int M>
__device__ __forceinline__ void c2r_unit(const LrArgs& A, long long unit, long long rows, double2* sm) {
    using Pl = fftc::Plan<M>;
    constexpr int R = Pl::R, P = Pl::P, TG = LS_THREADS / P, LPAD = M + M / R, XP = M + 2;
    const int tid = threadIdx.x, ls = tid / P, t = tid % P;
    const long long row = unit * TG + ls;
    const bool active = row < rows;
    double2* buf = sm + ls * XP;
    const double2* in = A.Yh + row * A.Mp;
#pragma unroll
    for (int j = 0; j < R; ++j) buf[t + P * j] = active ? in[t + P * j] : make_double2(0.0, 0.0);
    if (t == 0) buf[M] = active ? in[M] : make_double2(0.0, 0.0);
    __syncthreads();
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int k = t + P * r;
        const double2 a = buf[k], b = buf[M - k];
        const double2 s = make_double2(a.x + b.x, a.y - b.y);
        const double2 d = make_double2(a.x - b.x, a.y + b.y);
        const double2 wd = cmulc(__ldg(A.twL + k), d);
        v[r] = make_double2(s.x - wd.y, s.y + wd.x);
    }
    __syncthreads();
    fftc::stockham<M, true>(v, t, sm, [&](int q) { return ls * LPAD + q + q / R; }, A.twM);
    if (active) {
        double2* oz = reinterpret_cast<double2*>(A.u) + row * M;
        const double2* qz = reinterpret_cast<const double2*>(A.q) + row * M;
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int n = Pl::out_q(t, j);
            double2 r = v[j];
            if (A.q) r = csub(r, __ldg(qz + n));
            oz[n] = r;
        }
    }
    __syncthreads();
}

template <int M, int NY, int NZ>
struct LrShape {
    static constexpr int RP = LS_THREADS / fftc::Plan<M>::P;  // rows per row unit
    static constexpr int ROW_SMEM = RP * ((M + M / fftc::Plan<M>::R) > (M + 2) ? (M + M / fftc::Plan<M>::R) : (M + 2));
    static constexpr int COL_SMEM = NY * 8 * (LS_THREADS / (8 * fftc::Plan<NY>::P));
    static constexpr int ZTG = LS_THREADS / (8 * fftc::Plan<NZ>::P) > 0 ? LS_THREADS / (8 * fftc::Plan<NZ>::P) : 1;
    static constexpr int Z_SMEM = NZ * 8 * ZTG;
    static constexpr int SMEM = ROW_SMEM > COL_SMEM ? (ROW_SMEM > Z_SMEM ? ROW_SMEM : Z_SMEM)
                                                    : (COL_SMEM > Z_SMEM ? COL_SMEM : Z_SMEM);
};

template <int M, int NY, int NZ>
__global__ void __launch_bounds__(LS_THREADS, 4) lr_stage_kernel(LrArgs A) {
    using Sh = LrShape<M, NY, NZ>;
    extern __shared__ double2 sm[];
    cg::grid_group grid = cg::this_grid();
    const long long rows = (long long)NY * NZ;
    const long long row_units = (rows + Sh::RP - 1) / Sh::RP;
    const long long col_tiles = (long long)(A.Mp / 8) * NZ;
    const long long col_units = (col_tiles + (LS_THREADS / (8 * fftc::Plan<NY>::P)) - 1) /
                                (LS_THREADS / (8 * fftc::Plan<NY>::P));
    const long long z_tiles = (long long)A.Mp * NY / 8;
    const long long z_units = (z_tiles + Sh::ZTG - 1) / Sh::ZTG;
    for (long long u = blockIdx.x; u < row_units; u += gridDim.x) r2c_unit<M>(A, u, rows, sm);
    grid.sync();
    for (long long u = blockIdx.x; u < col_units; u += gridDim.x) col_unit<NY, false>(A, u, col_tiles, sm);
    grid.sync();
    for (long long u = blockIdx.x; u < z_units; u += gridDim.x) filter_unit<NZ>(A, u, z_tiles, NY, sm);
    grid.sync();
    for (long long u = blockIdx.x; u < col_units; u += gridDim.x) col_unit<NY, true>(A, u, col_tiles, sm);
    grid.sync();
    for (long long u = blockIdx.x; u < row_units; u += gridDim.x) c2r_unit<M>(A, u, rows, sm);
}

template <int M, int NY, int NZ>
void launch_lr_stage(const LrArgs& A0, cudaStream_t st) {
    using Sh = LrShape<M, NY, NZ>;
    static_assert(LS_THREADS % fftc::Plan<M>::P == 0, "row unit shape");
    static_assert(LS_THREADS / (8 * fftc::Plan<NY>::P) >= 1, "column unit shape");
    LrArgs A = A0;
    A.twM = fft_engine().twiddles(M);
    A.twL = fft_engine().twiddles(2 * M);
    A.twN = fft_engine().twiddles(NY);
    A.twZ = fft_engine().twiddles(NZ);
    auto kern = lr_stage_kernel<M, NY, NZ>;
    const size_t smem = (size_t)Sh::SMEM * sizeof(double2);
    VSR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    static int grid = 0;  // per instantiation: co-resident CTAs
    if (!grid) {
        int per_sm = 0, dev = 0, sms = 0;
        VSR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, LS_THREADS, smem));
        VSR_CUDA(cudaGetDevice(&dev));
        VSR_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        grid = std::max(per_sm, 1) * sms;
    }
    void* args[] = {&A};
    VSR_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(LS_THREADS), args, smem, st));
    VSR_LAUNCH_CHECK();
}

#define VSR_LRS_TABLE(X) X(64, 128, 128) X(32, 64, 64) X(16, 32, 32) X(64, 64, 64) X(32, 64, 32) X(16, 32, 16)

}  // namespace

bool lr_stage_ok(const Dims& lr) {
#define VSR_X(MM, NN, ZZ) \
    if (lr.m == 2 * MM && lr.n == NN && lr.s == ZZ) return true;
    VSR_LRS_TABLE(VSR_X)
#undef VSR_X
    return false;
}

void launch_lr_stage(const Dims& lr, const double* y, double2* Yh, double* u, const double* q, const double* a2,
                     const double* b2, const double* c2, double cfac, double shift, cudaStream_t st) {
    LrArgs A{};
    A.y = y, A.Yh = Yh, A.u = u, A.q = q, A.a2 = a2, A.b2 = b2, A.c2 = c2;
    A.cfac = cfac, A.shift = shift, A.Mp = half_pitch(lr.m);
#define VSR_X(MM, NN, ZZ)                             \
    if (lr.m == 2 * MM && lr.n == NN && lr.s == ZZ) { \
        launch_lr_stage<MM, NN, ZZ>(A, st);           \
        return;                                       \
    }
    VSR_LRS_TABLE(VSR_X)
#undef VSR_X
    throw std::logic_error("launch_lr_stage: unsupported LR geometry");
}

}  // namespace vsr
