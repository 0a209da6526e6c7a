// Spatial expansion path of the Tikhonov solve (see spatial.cuh for the
// algebra).  Two kernels: an LR pointwise kernel U(g) and a tiled 3-stage
// separable correlation that writes x in one HBM pass.
#include <algorithm>
#include <cmath>
#include <complex>
#include <type_traits>
#include <vector>

#include "fft.cuh"
#include "fft_core.cuh"
#include "spatial.cuh"

namespace vsr {

// --------------------------------------------------------------- LR kernel
// U(g) = (d yv - Z G1) / (G2 + 2 reg d),  yv = Yl / sqrt(d)
// (x_hat = X̄ + conj(Lambda) U, the stable form of (k - conj(Lambda) w) / (2 reg)).
__global__ void __launch_bounds__(256) spatial_u_kernel(long long ml, long long nl, long long Nl, double dd,
                                                        double inv_sqrt_d, double shift, const double2* __restrict__ Yl,
                                                        const double2* __restrict__ Zl,
                                                        const double2* __restrict__ a1, const double2* __restrict__ b1,
                                                        const double2* __restrict__ c1, const double* __restrict__ a2,
                                                        const double* __restrict__ b2, const double* __restrict__ c2,
                                                        double2* __restrict__ U) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < Nl;
         e += (long long)gridDim.x * blockDim.x) {
        const long long g1 = e % ml, r = e / ml, g2 = r % nl, g3 = r / nl;
        const double2 G1 = cmul(cmul(a1[g1], b1[g2]), c1[g3]);
        const double G2 = (a2[g1] * b2[g2]) * c2[g3];
        const double2 y = cscale(Yl[e], inv_sqrt_d * dd);
        const double2 num = Zl ? csub(y, cmul(Zl[e], G1)) : y;
        U[e] = cscale(num, 1.0 / (G2 + shift));
    }
}

void launch_spatial_v(const Dims& lr, int d, const SpatialPlan& p, const double2* Yl, const double2* Zl,
                      double reg, double2* U, cudaStream_t st) {
    const long long Nl = (long long)lr.count();
    const unsigned blocks = (unsigned)std::min<long long>((Nl + 255) / 256, 148LL * 16);
    spatial_u_kernel<<<blocks, 256, 0, st>>>((long long)lr.m, (long long)lr.n, Nl, (double)d,
                                             1.0 / std::sqrt((double)d), 2.0 * reg * d, Yl, Zl, p.s1[0],
                                             p.s1[1], p.s1[2], p.s2[0], p.s2[1], p.s2[2], U);
    VSR_LAUNCH_CHECK();
}

// --------------------------------------------------- LR axis-3 sandwich
// In place on Y (LR spectrum after the forward axis-1/2 passes, unscaled):
// forward axis-3 FFT, scale fs, U(g) as in spatial_u_kernel, inverse axis-3
// FFT scaled by out_scale.  A CTA owns TG tiles of T consecutive inner
// positions p = g1 + ml g2, each line held by P threads x R registers.
#ifndef VSR_SW_RMAX
#define VSR_SW_RMAX 8
#endif
constexpr int kSwR = VSR_SW_RMAX;  // values per thread of the LR axis-3 sandwich

template <int L>
struct SwShape {
    using Pl = fftc::Plan<L, kSwR>;
    static constexpr int R = Pl::R, P = Pl::P, T = 8;
    static constexpr int TG = (T * P) >= 128 ? 1 : 128 / (T * P);
    static constexpr int THREADS = TG * T * P;
    static constexpr int SMEM = Pl::NEEDS_SMEM ? TG * T * L : 0;  // double2 elements
};

template <int L>
__global__ void __launch_bounds__(SwShape<L>::THREADS, 512 / SwShape<L>::THREADS)
    lr_sandwich_kernel(double2* Y, const double2* __restrict__ Zl, long long S, int pitch, int nl,
                       const double2* __restrict__ a1, const double2* __restrict__ b1,
                       const double2* __restrict__ c1, const double* __restrict__ a2,
                       const double* __restrict__ b2, const double* __restrict__ c2, double cy,
                       double shift, double out_scale, const double2* __restrict__ tw) {
    using Sh = SwShape<L>;
    using Pl = typename Sh::Pl;
    constexpr int R = Sh::R, P = Sh::P, T = Sh::T;
    extern __shared__ double2 smw[];
    const int tid = threadIdx.x;
    const int g = tid / (T * P), rem = tid % (T * P), lt = rem % T, t = rem / T;
    const int ls = g * T + lt;
    const long long tile = (long long)blockIdx.x * Sh::TG + g;
    const bool active = tile * T < S;
    const long long p = active ? tile * T + lt : 0;
    auto sidx = [&](int q) { return (ls / T) * (L * T) + q * T + (ls % T); };

    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = active ? Y[p + S * (t + P * r)] : make_double2(0.0, 0.0);
    if (Zl && active) {  // pull the prior's spectrum toward L2 while the forward transform runs
#pragma unroll
        for (int r = 0; r < R; ++r) asm volatile("prefetch.global.L2 [%0];" ::"l"(Zl + p + S * (t + P * r)));
    }
    // the filter's table reads are issued before the transform (latency hidden under it)
    const int g1 = (int)(p % pitch), g2 = (int)(p / pitch);
    const double ab2 = __ldg(a2 + g1) * __ldg(b2 + g2);
    double cz[R];
#pragma unroll
    for (int r = 0; r < R; ++r) cz[r] = __ldg(c2 + t + P * r);
    fftc::stockham<L, false, decltype(sidx), kSwR>(v, t, smw, sidx, tw);
    fftc::to_natural<L, kSwR>(v);
    // v[r] = F_l(y) at g3 = t + P r (times 1/fs)
    const double2 ab1 = Zl ? cmul(__ldg(a1 + g1), __ldg(b1 + g2)) : make_double2(0.0, 0.0);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int g3 = t + P * r;
        const double2 y = cscale(v[r], cy);
        const double2 num = Zl ? csub(y, cmul(__ldg(Zl + p + S * g3), cmul(ab1, __ldg(c1 + g3)))) : y;
        v[r] = cscale(num, rcp_pos(ab2 * cz[r] + shift));
    }
    __syncthreads();  // the exchange buffer is reused by the inverse transform
    fftc::stockham<L, true, decltype(sidx), kSwR>(v, t, smw, sidx, tw);
    if (active) {
#pragma unroll
        for (int j = 0; j < R; ++j) Y[p + S * Pl::out_q(t, j)] = cscale(v[j], out_scale);
    }
}

template <int L>
static void launch_sandwich_L(const Dims& lr, const SpatialPlan& p, double2* Y, const double2* Zl, double cy,
                              double shift, double out_scale, cudaStream_t st) {
    using Sh = SwShape<L>;
    const long long S = (long long)(lr.m * lr.n);
    const long long tiles = S / Sh::T;
    const unsigned blocks = (unsigned)((tiles + Sh::TG - 1) / Sh::TG);
    const size_t smem = (size_t)Sh::SMEM * sizeof(double2);
    auto kern = lr_sandwich_kernel<L>;
    if (smem > 48 * 1024)
        VSR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<blocks, Sh::THREADS, smem, st>>>(Y, Zl, S, (int)lr.m, (int)lr.n, p.s1[0], p.s1[1], p.s1[2], p.s2[0],
                                            p.s2[1], p.s2[2], cy, shift, out_scale,
                                            fft_engine().twiddles(L));
    VSR_LAUNCH_CHECK();
}

// lr: the grid the sandwich runs on, lr.m = row pitch (ml, or the half-
// spectrum pitch with Zl == nullptr).
bool spatial_sandwich_ok(const Dims& lr) {
    const size_t L = lr.s;
    return L >= 8 && L <= 1024 && is_pow2(L) && (lr.m * lr.n) % 8 == 0 && lr.m * lr.n * L < (1ull << 31);
}

void launch_spatial_sandwich(const Dims& lr, int d, const SpatialPlan& p, double2* Y, const double2* Zl,
                             double reg, double fwd_scale, double out_scale, cudaStream_t st) {
    const double cy = fwd_scale * (double)d / std::sqrt((double)d);
    const double shift = 2.0 * reg * d;
    switch (lr.s) {
        case 8: launch_sandwich_L<8>(lr, p, Y, Zl, cy, shift, out_scale, st); break;
        case 16: launch_sandwich_L<16>(lr, p, Y, Zl, cy, shift, out_scale, st); break;
        case 32: launch_sandwich_L<32>(lr, p, Y, Zl, cy, shift, out_scale, st); break;
        case 64: launch_sandwich_L<64>(lr, p, Y, Zl, cy, shift, out_scale, st); break;
        case 128: launch_sandwich_L<128>(lr, p, Y, Zl, cy, shift, out_scale, st); break;
        case 256: launch_sandwich_L<256>(lr, p, Y, Zl, cy, shift, out_scale, st); break;
        case 512: launch_sandwich_L<512>(lr, p, Y, Zl, cy, shift, out_scale, st); break;
        case 1024: launch_sandwich_L<1024>(lr, p, Y, Zl, cy, shift, out_scale, st); break;
        default: throw std::logic_error("spatial_sandwich: unsupported axis-3 length");
    }
}

// ------------------------------------------------------------ expand kernel
// Polyphase form: a tile is CX x CY x CZ LR cells (origin on the lattice), i.e.
// r1 CX x r2 CY x r3 CZ outputs.  Output n = r (c0 + c) + phi reads LR cells
// c0 + c + delta, delta in [dmin, dmin + DM), with tap k[r delta - phi + h]
// (zero-padded per phase in kp[phi * DM + delta - dmin]).
//   stage A (axis 3): T1[tz][qy][qx], one (qy, qx) column per thread, its LZ
//                     LR inputs loaded from L2 straight into registers
//   stage B (axis 2): T2[tz][ty][qx], one (tz, qx) column per thread
//   stage C (axis 1): x rows; a thread owns XB consecutive LR columns of a row
//                     and all r1 phases (R1 > 0: compile-time, vector stores)
constexpr int SP_THREADS = 128;
constexpr int SP_CX = 16, SP_CY = 4, SP_CZ = 4, SP_XB = 2;
constexpr int SP_MAX_ROWS = 1024;  // TZ * TY bound (rates r2 * r3 <= 64)

struct AxisTaps {
    int r, dmin;
};

struct ExpandArgs {
    int m, n, s, ml, nl, sl;
    AxisTaps ax[3];
    int tiles1, tiles2;
    const double* kp;  // kp1 (r1*DM) | kp2 (r2*DM) | kp3 (r3*DM)
    const double* u;
    const double* z;
    double* x;
    unsigned long long* bad;
};

__device__ __forceinline__ int wrap_idx(int j, int L) {
    j %= L;
    return j < 0 ? j + L : j;
}

template <int DM, int R1>
__global__ void __launch_bounds__(SP_THREADS, (DM <= 8 ? 8 : 6)) spatial_expand_kernel(ExpandArgs A) {
    extern __shared__ double sm[];
    constexpr int LX = SP_CX + DM - 1, LY = SP_CY + DM - 1, LZ = SP_CZ + DM - 1;
    const int r1 = R1 > 0 ? R1 : A.ax[0].r, r2 = A.ax[1].r, r3 = A.ax[2].r;
    const int TY = r2 * SP_CY, TZ = r3 * SP_CZ;
    const int nkp = (r1 + r2 + r3) * DM;
    double* kp1 = sm;
    double* kp2 = kp1 + r1 * DM;
    double* kp3 = kp2 + r2 * DM;
    double* t1 = sm + nkp;                 // TZ * LY * LX
    double* t2 = t1 + TZ * LY * LX;        // TZ * TY * LX
    // stage-C row tables: tz | ty << 8, and the LR index of the row's prior
    // samples (-1 off the lattice)
    double* zt = t2 + TZ * TY * LX;                      // lattice prior tile, CZ x CY x CX
    int* rowinfo = reinterpret_cast<int*>(zt + SP_CZ * SP_CY * SP_CX);
    int* zrow = rowinfo + TZ * TY;                          // offset of the row's prior samples in zt, -1 off lattice
    __shared__ long long zoff[LZ];
    __shared__ int yoff[LY], xoff[LX];

    const int tid = threadIdx.x;
    const int cx0 = blockIdx.x * SP_CX, cy0 = blockIdx.y * SP_CY, cz0 = blockIdx.z * SP_CZ;
    const int rows = TZ * TY;

    for (int i = tid; i < nkp; i += SP_THREADS) kp1[i] = A.kp[i];
    // prior samples of the tile: loaded now into registers, parked in smem after
    // stage A (their latency overlaps stage A), read in stage C
    constexpr int NZT = SP_CZ * SP_CY * SP_CX, ZPER = (NZT + SP_THREADS - 1) / SP_THREADS;
    double zreg[ZPER];
#pragma unroll
    for (int k = 0; k < ZPER; ++k) {
        const int i = tid + k * SP_THREADS;
        const int cx = i % SP_CX, r = i / SP_CX, cy = r % SP_CY, cz = r / SP_CY;
        const bool in = A.z && i < NZT && cx0 + cx < A.ml && cy0 + cy < A.nl && cz0 + cz < A.sl;
        zreg[k] = in ? __ldg(A.z + ((size_t)(cz0 + cz) * A.nl + cy0 + cy) * A.ml + cx0 + cx) : 0.0;
    }
    if (tid < LZ) zoff[tid] = (long long)wrap_idx(cz0 + A.ax[2].dmin + tid, A.sl) * A.nl * A.ml;
    else if (tid >= 32 && tid < 32 + LY) yoff[tid - 32] = wrap_idx(cy0 + A.ax[1].dmin + tid - 32, A.nl) * A.ml;
    else if (tid >= 64 && tid < 64 + LX) xoff[tid - 64] = wrap_idx(cx0 + A.ax[0].dmin + tid - 64, A.ml);
    for (int row = tid; row < rows; row += SP_THREADS) {
        const int tz = row / TY, ty = row - tz * TY;
        const bool lat = A.z != nullptr && (ty % r2) == 0 && (tz % r3) == 0;
        rowinfo[row] = tz | (ty << 8);
        zrow[row] = lat ? ((tz / r3) * SP_CY + ty / r2) * SP_CX : -1;
    }
    __syncthreads();
    // stage A: axis 3
    for (int col = tid; col < LY * LX; col += SP_THREADS) {
        const int qy = col / LX, qx = col - qy * LX;
        const double* src = A.u + yoff[qy] + xoff[qx];
        double in[LZ];
#pragma unroll
        for (int i = 0; i < LZ; ++i) in[i] = __ldg(src + zoff[i]);
        for (int ph = 0; ph < r3; ++ph) {
            double k[DM];
#pragma unroll
            for (int d = 0; d < DM; ++d) k[d] = kp3[ph * DM + d];
#pragma unroll
            for (int c = 0; c < SP_CZ; ++c) {
                double acc = 0.0;
#pragma unroll
                for (int d = 0; d < DM; ++d) acc = fma(k[d], in[c + d], acc);
                t1[((r3 * c + ph) * LY) * LX + col] = acc;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < ZPER; ++k)
        if (tid + k * SP_THREADS < NZT) zt[tid + k * SP_THREADS] = zreg[k];
    __syncthreads();
    // stage B: axis 2
    for (int col = tid; col < TZ * LX; col += SP_THREADS) {
        const int tz = col / LX, qx = col - tz * LX;
        double in[LY];
#pragma unroll
        for (int i = 0; i < LY; ++i) in[i] = t1[(tz * LY + i) * LX + qx];
        for (int ph = 0; ph < r2; ++ph) {
            double k[DM];
#pragma unroll
            for (int d = 0; d < DM; ++d) k[d] = kp2[ph * DM + d];
#pragma unroll
            for (int c = 0; c < SP_CY; ++c) {
                double acc = 0.0;
#pragma unroll
                for (int d = 0; d < DM; ++d) acc = fma(k[d], in[c + d], acc);
                t2[(tz * TY + r2 * c + ph) * LX + qx] = acc;
            }
        }
    }
    __syncthreads();
    // stage C: axis 1 + lattice prior
    constexpr int NXB = SP_CX / SP_XB;
    const int X0 = cx0 * r1, Y0 = cy0 * r2, Z0 = cz0 * r3;
    const int xb = tid % NXB, c0 = xb * SP_XB, n1 = X0 + r1 * c0;
    constexpr bool HOIST = R1 > 0 && R1 * DM <= 16;  // all phases' taps in registers
    double kh[HOIST ? R1 * DM : 1];
    if constexpr (HOIST) {
#pragma unroll
        for (int i = 0; i < R1 * DM; ++i) kh[i] = kp1[i];
    }
    for (int row = tid / NXB; row < rows; row += SP_THREADS / NXB) {
        const int info = rowinfo[row], zr = zrow[row];
        const int tz = info & 0xff, ty = info >> 8;
        const int n2 = Y0 + ty, n3 = Z0 + tz;
        if (n2 >= A.n || n3 >= A.s || n1 >= A.m) continue;
        const bool lat = zr >= 0;
        double zv[SP_XB];
#pragma unroll
        for (int j = 0; j < SP_XB; ++j) zv[j] = lat ? zt[zr + c0 + j] : 0.0;
        double in[DM + SP_XB - 1];
        const double* src = t2 + row * LX + c0;
#pragma unroll
        for (int i = 0; i < DM + SP_XB - 1; ++i) in[i] = src[i];
        double* xp = A.x + ((size_t)n3 * A.n + n2) * A.m + n1;
        bool fin = true;
        if constexpr (R1 > 0) {
            double out[SP_XB * R1];
#pragma unroll
            for (int ph = 0; ph < R1; ++ph) {
                double k[DM];
#pragma unroll
                for (int d = 0; d < DM; ++d) k[d] = HOIST ? kh[(HOIST ? ph * DM + d : 0)] : kp1[ph * DM + d];
#pragma unroll
                for (int j = 0; j < SP_XB; ++j) {
                    double acc = 0.0;
#pragma unroll
                    for (int d = 0; d < DM; ++d) acc = fma(k[d], in[j + d], acc);
                    if (ph == 0) acc += zv[j];
                    out[j * R1 + ph] = acc;
                    fin = fin && isfinite(acc);
                }
            }
            if (n1 + SP_XB * R1 <= A.m && (SP_XB * R1) % 2 == 0 && (A.m & 1) == 0) {
#pragma unroll
                for (int i = 0; i < SP_XB * R1; i += 2)
                    *reinterpret_cast<double2*>(xp + i) = make_double2(out[i], out[i + 1]);
            } else {
#pragma unroll
                for (int i = 0; i < SP_XB * R1; ++i)
                    if (n1 + i < A.m) xp[i] = out[i];
            }
        } else {
            for (int ph = 0; ph < r1; ++ph) {
                const double* k = kp1 + ph * DM;
#pragma unroll
                for (int j = 0; j < SP_XB; ++j) {
                    double acc = 0.0;
#pragma unroll
                    for (int d = 0; d < DM; ++d) acc = fma(k[d], in[j + d], acc);
                    if (ph == 0) acc += zv[j];
                    if (n1 + j * r1 + ph < A.m) xp[j * r1 + ph] = acc;
                    fin = fin && isfinite(acc);
                }
            }
        }
        if (!fin) {
            for (int i = 0; i < SP_XB * r1; ++i)
                if (n1 + i < A.m && !isfinite(xp[i])) {
                    atomicMin(A.bad, (unsigned long long)(xp + i - A.x));
                    break;
                }
        }
    }
}

// ------------------------------------------------ expand kernel, z march
// Same polyphase correlation, reordered so the output-heavy axis runs last
// from registers: a CTA owns a CX x CY LR column (output W x H per plane) and
// marches along z through its chunk of LR planes.  Four stages per LR plane:
//   a. the prefetched LR tile (LY x LX with the x/y halo) is parked in smem and
//      the next plane's tile is fetched into registers;
//   b. stage x: one LR row, two LR cells x R1 phases per item (pair loads);
//   c. stage y: one output column, two LR cells x R2 phases per item;
//   d. stage z: each thread keeps the last DM xy-expanded planes of its
//      column pairs in a register ring (slot = plane mod DM, compile-time via
//      the DM-fold unroll) and writes R3 output planes, 16-B stores.
// The stages are software-pipelined: phase p parks plane p, runs stage x on
// plane p - 1, y on p - 2 and z on p - 3 out of double-buffered tiles, so a
// phase holds four independent pieces of work and ends in ONE barrier.
// No z halo is re-read except the DM - 1 warm-up planes of each chunk; taps
// are kernel parameters (constant-bank operands of the DFMAs).  Finiteness:
// fma(v, 0, chk) turns any inf/nan into a NaN chk; a thread that sees one
// rescans its own outputs for the first bad flat index.
constexpr int MX_CX = 16, MX_CY = 4, MX_THREADS = 128, MX_KMAX = 64;
constexpr int MX_ZCMAX = 64;
constexpr int MX_PD = 3;  // LR plane tiles in flight (cp.async ring depth - 2)  // LR planes per CTA chunk (bounds the prior's smem stage)

struct MarchArgs {
    int m, n, s, ml, nl, sl;
    int dmin1, dmin2, dmin3;
    int zc;  // LR planes per CTA
    double k1[MX_KMAX], k2[MX_KMAX], k3[MX_KMAX];
    float f1[MX_KMAX], f2[MX_KMAX], f3[MX_KMAX];  // the same taps for the fp32 march
    const double* u;
    const double* z;
    void* x;  // double (reference precision) or float (fp32 mode)
    unsigned long long* bad;
};

// ISO: the three axes share one tap set (an isotropic PSF at equal rates, the
// common case): the DFMAs' uniform-register operands then fit without the
// spill / refill traffic three distinct sets cause (~12 % of the instructions)
template <class T, bool ISO>
__device__ __forceinline__ T march_tap(const MarchArgs& A, int axis, int i) {
    if (ISO) axis = 0;
    if constexpr (std::is_same<T, double>::value)
        return axis == 0 ? A.k1[i] : (axis == 1 ? A.k2[i] : A.k3[i]);
    else
        return axis == 0 ? A.f1[i] : (axis == 1 ? A.f2[i] : A.f3[i]);
}

// T = double: the reference precision.  T = float (fp32 mode): the LR tile
// and prior arrive as fp64 and are rounded on use; the three correlation
// stages, the register ring and x run in fp32 (half the HBM bytes of x).
template <int DM, int R1, int R2, int R3, int CY, class T = double, bool ISO = false>
__global__ void __launch_bounds__(MX_THREADS, 4) spatial_march_kernel(const __grid_constant__ MarchArgs A) {
    static_assert(!ISO || (R1 == R2 && R2 == R3), "one tap set needs equal rates");
    using T2 = std::conditional_t<std::is_same<T, double>::value, double2, float2>;
    static_assert(R1 == 2, "stage z pairs (2c, 2c + 1) assume the lattice column is the even one");
    constexpr int CX = MX_CX, NT = MX_THREADS;
    constexpr int LX = CX + DM - 1, LY = CY + DM - 1;
    constexpr int LXP = LX + (LX & 1);  // even pitch: 16-B aligned pair loads
    constexpr int W = R1 * CX, H = R2 * CY;
    constexpr int NLD = (LY * LX + NT - 1) / NT;
    constexpr int NXI = LY * (CX / 2), NYI = W * (CY / 2);
    constexpr int NPAIR = (DM + 2) / 2;  // pair loads covering DM + 1 inputs
    constexpr int CPR = W / 2, RG = NT / CPR, RPT = H / RG;
    static_assert(NT % CPR == 0 && H % RG == 0, "stage-z thread map");
    constexpr int NB = MX_PD + 2, LTB = LY * LXP + 2;  // + pad slot (keeps 16-B alignment)
    __shared__ __align__(16) double lt[NB][LTB];
    constexpr int NZB = MX_PD + 4;  // prior ring: fetched PD phases before plane q lands, read 3 after
    __shared__ __align__(16) double zs[NZB][CY * CX];
    __shared__ __align__(16) T ex[2][LY * W];
    __shared__ __align__(16) T ey[2][H * W];
    __shared__ int xoff[LX], yoff[LY];

    const int tid = threadIdx.x;
    const int cx0 = blockIdx.x * CX, cy0 = blockIdx.y * CY;
    const int c30 = blockIdx.z * A.zc;
    const int nz = min(A.zc, A.sl - c30);
    if (tid < LX)
        xoff[tid] = wrap_idx(cx0 + A.dmin1 + tid, A.ml);
    else if (tid >= 32 && tid < 32 + LY)
        yoff[tid - 32] = wrap_idx(cy0 + A.dmin2 + tid - 32, A.nl) * A.ml;
    __syncthreads();
    // loads past the tile read offset 0 and park in the pad slot (never read),
    // so the prefetch is unconditional: no select keeps a register waiting on it
    int loff[NLD], lsm[NLD];
#pragma unroll
    for (int k = 0; k < NLD; ++k) {
        const int e = tid + NT * k;
        if (e < LY * LX) {
            const int qy = e / LX, qx = e - qy * LX;
            loff[k] = yoff[qy] + xoff[qx];
            lsm[k] = qy * LXP + qx;
        } else {
            loff[k] = 0;
            lsm[k] = LY * LXP;
        }
    }
    const long long plane = (long long)A.ml * A.nl;
    const int jend = nz + DM - 1;  // LR planes the chunk reads
    int zq = wrap_idx(c30 + A.dmin3, A.sl);  // LR z of the next plane to fetch
    const int cp = tid % CPR, rg = tid / CPR;
    const int X0 = cx0 * R1, Y0 = cy0 * R2;
    T2 ring[RPT][DM];
    T chk = 0;
    // LR plane tiles: cp.async ring of NB buffers, MX_PD planes in flight
    // per-element shared addresses of buffer 0 and global pointers of LR z = 0
    // per-element shared addresses of buffer 0; 32-bit in-plane offsets
    // against a running plane pointer (one wide add per element per fetch)
    unsigned lsa[NLD];
#pragma unroll
    for (int k = 0; k < NLD; ++k) lsa[k] = (unsigned)__cvta_generic_to_shared(&lt[0][lsm[k]]);
    const double* uz = A.u + zq * plane;  // LR plane zq
    unsigned bo = 0;                      // byte offset of the next fetch's ring buffer
    int zfs = NZB - (DM - 1) % NZB;  // prior slot of the next fetch: (q - (DM - 1)) mod NZB, q = 0
    if (zfs == NZB) zfs = 0;
    // the prior rows of this thread's (y, 2h) pair in output plane c3 = c30 + oz
    const bool zact = A.z && tid < CY * (CX / 2);
    const double* zp = A.z + ((long long)c30 * A.nl + cy0 + (zact ? tid / (CX / 2) : 0)) * A.ml + cx0 +
                       2 * (zact ? tid % (CX / 2) : 0) - (long long)(DM - 1) * plane;
    const unsigned zsa = (unsigned)__cvta_generic_to_shared(&zs[0][2 * tid]);
    auto fetch = [&](int q) {
        if (q < jend) {
#pragma unroll
            for (int k = 0; k < NLD; ++k)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(lsa[k] + bo), "l"(uz + loff[k])
                             : "memory");
            uz += plane;
            if (++zq == A.sl) zq = 0, uz = A.u;
            bo = bo + LTB * 8u == NB * LTB * 8u ? 0u : bo + LTB * 8u;
        }
        // the lattice prior of output plane c3 (its last LR plane is q): cold in
        // HBM, so it rides in the same group, DM + 2 phases before stage z reads it
        const int oz = q - (DM - 1);
        if (zact && oz >= 0 && oz < nz)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(zsa + zfs * (unsigned)(CY * CX * 8)),
                         "l"(zp + (long long)q * plane) : "memory");
        zfs = zfs + 1 == NZB ? 0 : zfs + 1;
        asm volatile("cp.async.commit_group;" ::: "memory");  // (empty past the chunk: uniform counting)
    };
    for (int q = 0; q < MX_PD; ++q) fetch(q);
    const long long hplane = (long long)A.n * A.m;
    T* const xrow = static_cast<T*>(A.x) + (long long)(Y0 + rg * RPT) * A.m + X0 + 2 * cp;
    // loop-invariant per-thread offsets of the x and y stages (one item each
    // when the stage fits the CTA) and rotating slot counters instead of the
    // runtime modulos: the march is issue-bound
    static_assert(NXI <= NT && NYI <= NT, "one stage-x / stage-y item per thread");
    const bool xact = tid < NXI;
    const int sxq = xact ? tid / (CX / 2) : 0, sxc = xact ? 2 * (tid - sxq * (CX / 2)) : 0;
    const int sx_in = sxq * LXP + sxc, sx_out = sxq * W + R1 * sxc;
    const bool yact = tid < NYI;
    const int syc = yact ? 2 * (tid / W) : 0, syn = yact ? tid % W : 0;
    const int sy_in = syc * W + syn, sy_out = R2 * syc * W + syn;
    const long long xrs = A.m;
    // advanced at the top of each phase p: lslot = (p - 1) mod NB (stage x's
    // LR tile), zslot = (p - 3 - (DM - 1)) mod NZB (stage z's prior plane)
    int lslot = NB - 2;
    int zslot = ((-DM - 3) % NZB + NZB) % NZB;
    T* xz = xrow + (long long)R3 * c30 * hplane;  // output plane R3 * c3 of the next stage-z plane
    for (int pb = 0; pb < jend + 3; pb += DM) {
#pragma unroll
        for (int s = 0; s < DM; ++s) {
            const int p = pb + s;
            if (p >= jend + 3) break;
            // a. fetch plane p + PD; plane p must land before this phase's barrier
            fetch(p + MX_PD);
            // d. stage z on plane p - 3 (issued first: its loads and stores
            //    overlap the smem work of stages x and y below)
            const int jz = p - 3;
            zslot = zslot + 1 == NZB ? 0 : zslot + 1;
            lslot = lslot + 1 == NB ? 0 : lslot + 1;
            if (jz >= 0) {
                const T* eb = ey[jz & 1];
                const int slot = ((s - 3) % DM + DM) % DM;  // compile-time after the unroll
#pragma unroll
                for (int rr = 0; rr < RPT; ++rr)
                    ring[rr][slot] = *reinterpret_cast<const T2*>(eb + (rg * RPT + rr) * W + 2 * cp);
                if (jz >= DM - 1) {
                    T zv[RPT];
#pragma unroll
                    for (int rr = 0; rr < RPT; ++rr) {
                        const int row = rg * RPT + rr;
                        zv[rr] = (A.z && row % R2 == 0) ? (T)zs[zslot][(row / R2) * CX + cp] : (T)0;
                    }
                    T* xp = xz;
#pragma unroll
                    for (int ph = 0; ph < R3; ++ph, xp += hplane) {
#pragma unroll
                        for (int rr = 0; rr < RPT; ++rr) {
                            T ax = 0, ay = 0;
#pragma unroll
                            for (int i = 0; i < DM; ++i) {
                                const T2 v = ring[rr][(slot + 1 + i) % DM];
                                ax = fma(march_tap<T, ISO>(A, 2, ph * DM + i), v.x, ax);
                                ay = fma(march_tap<T, ISO>(A, 2, ph * DM + i), v.y, ay);
                            }
                            if (ph == 0) ax += zv[rr];
                            chk = fma(ax, (T)0, chk);
                            chk = fma(ay, (T)0, chk);
                            T2 o;
                            o.x = ax;
                            o.y = ay;
                            __stcs(reinterpret_cast<T2*>(xp + rr * xrs), o);  // streaming: x must not evict u
                        }
                    }
                    xz += R3 * hplane;
                }
            }
            // b. stage x on plane p - 1
            const int jx = p - 1;
            if (jx >= 0 && jx < jend) {
                const double* lb = lt[lslot];
                T* xb = ex[jx & 1];
                if (xact) {
                    const double* row = lb + sx_in;
                    T in[2 * NPAIR];
#pragma unroll
                    for (int i = 0; i < NPAIR; ++i) {
                        const double2 v = *reinterpret_cast<const double2*>(row + 2 * i);
                        in[2 * i] = (T)v.x;
                        in[2 * i + 1] = (T)v.y;
                    }
                    T o[2 * R1];
#pragma unroll
                    for (int cell = 0; cell < 2; ++cell)
#pragma unroll
                        for (int ph = 0; ph < R1; ++ph) {
                            T acc = 0;
#pragma unroll
                            for (int i = 0; i < DM; ++i) acc = fma(march_tap<T, ISO>(A, 0, ph * DM + i), in[cell + i], acc);
                            o[cell * R1 + ph] = acc;
                        }
                    T* dst = xb + sx_out;
#pragma unroll
                    for (int i = 0; i < 2 * R1; i += 2) {
                        T2 w2;
                        w2.x = o[i];
                        w2.y = o[i + 1];
                        *reinterpret_cast<T2*>(dst + i) = w2;
                    }
                }
            }
            // c. stage y on plane p - 2
            const int jy = p - 2;
            if (jy >= 0 && jy < jend) {
                const T* xb = ex[jy & 1];
                T* yb = ey[jy & 1];
                if (yact) {
                    T in[DM + 1];
#pragma unroll
                    for (int i = 0; i < DM + 1; ++i) in[i] = xb[sy_in + i * W];
#pragma unroll
                    for (int cell = 0; cell < 2; ++cell)
#pragma unroll
                        for (int ph = 0; ph < R2; ++ph) {
                            T acc = 0;
#pragma unroll
                            for (int i = 0; i < DM; ++i) acc = fma(march_tap<T, ISO>(A, 1, ph * DM + i), in[cell + i], acc);
                            yb[sy_out + (R2 * cell + ph) * W] = acc;
                        }
                }
            }
            asm volatile("cp.async.wait_group %0;" ::"n"(MX_PD) : "memory");  // plane p (and the prior) landed
            __syncthreads();
        }
    }
    if (chk != chk) {  // some output is inf/nan: find this thread's first one
        unsigned long long best = ~0ull;
        for (int c3 = c30; c3 < c30 + nz; ++c3)
            for (int ph = 0; ph < R3; ++ph)
                for (int rr = 0; rr < RPT; ++rr)
                    for (int e = 0; e < 2; ++e) {
                        const unsigned long long idx =
                            ((unsigned long long)(R3 * c3 + ph) * A.n + Y0 + rg * RPT + rr) * A.m + X0 + 2 * cp + e;
                        if (!isfinite(static_cast<const T*>(A.x)[idx]) && idx < best) best = idx;
                    }
        atomicMin(A.bad, best);
    }
}

template <int DM, int R3, int CY, class T, bool ISO = false>
static void launch_march_cy(MarchArgs& A, unsigned tx, unsigned ty, cudaStream_t st) {
    auto kern = spatial_march_kernel<DM, 2, 2, R3, CY, T, ISO>;
    int dev = 0, sms = 0;
    VSR_CUDA(cudaGetDevice(&dev));
    VSR_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    // z chunk length: minimise waves x (planes per CTA incl. the DM - 1 warm-up
    // planes and 3 pipeline phases); ties: the longer chunk
    const long long cols = (long long)tx * ty;
    static long long memo_key = -1;  // per instantiation: last (sl, cols, prior) and its choice
    static int memo_zc = 0;
    const long long key = ((long long)A.sl << 33) ^ (cols << 1) ^ (A.z ? 1 : 0);
    int zc = std::min(A.sl, MX_ZCMAX);
    double best = 1e300;
    int occ = 0;
    if (memo_key != key) VSR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, MX_THREADS, 0));
    for (int c = memo_key == key ? 0 : std::min(A.sl, MX_ZCMAX); c >= 4; --c) {
        const long long ctas = cols * ((A.sl + c - 1) / c), slots = (long long)std::max(occ, 1) * sms;
        const double cost = (double)((ctas + slots - 1) / slots) * (c + DM + 2);
        if (cost < best) best = cost, zc = c;
    }
    if (memo_key == key)
        zc = memo_zc;
    else
        memo_key = key, memo_zc = zc;
    if (const char* e = std::getenv("VSR_MARCH_ZC")) zc = std::max(1, std::atoi(e));
    zc = std::min(std::min(zc, A.sl), MX_ZCMAX);
    A.zc = zc;
    const unsigned tz = (unsigned)((A.sl + zc - 1) / zc);
    kern<<<dim3(tx, ty, tz), MX_THREADS, 0, st>>>(A);
    VSR_LAUNCH_CHECK();
}

template <int DM, int R3, class T>
static void launch_march_k(MarchArgs& A, unsigned tx, unsigned ty, bool iso, cudaStream_t st) {
    static const bool cy8 = [] {
        const char* e = std::getenv("VSR_MARCH_CY");  // 8-row column tiles unless VSR_MARCH_CY=4
        return !(e && e[0] == '4');
    }();
    if (cy8 && ty % 2 == 0) {
        if constexpr (R3 == 2)
            if (iso) return launch_march_cy<DM, R3, 8, T, true>(A, tx, ty / 2, st);
        launch_march_cy<DM, R3, 8, T>(A, tx, ty / 2, st);
    } else {
        launch_march_cy<DM, R3, 4, T>(A, tx, ty, st);
    }
}

// The march kernel serves rates (2, 2, 2|4) with a tile-aligned LR grid.
static bool march_ok(const Dims& hr, const int rates[3], int dm) {
    if (rates[0] != 2 || rates[1] != 2 || (rates[2] != 2 && rates[2] != 4)) return false;
    if (dm != 4 && dm != 5 && dm != 7 && dm != 8) return false;
    if (hr.s / rates[2] < 1) return false;
    const char* e = std::getenv("VSR_NO_MARCH");
    if (e && e[0] == '1') return false;
    return (hr.m / 2) % MX_CX == 0 && (hr.n / 2) % MX_CY == 0 && rates[2] * dm <= MX_KMAX;
}

static const int kDms[] = {4, 5, 7, 8, 12, 16};  // 5, 7: the 9- and 13-tap PSFs at rate 2

// DM (padded taps per phase) serving every axis, 0 if the support is too wide.
static int pick_dm(const SpatialPlan& p) {
    int need = 0;
    for (int a = 0; a < 3; ++a) need = std::max(need, p.ndelta[a]);
    for (int dm : kDms)
        if (dm >= need) return dm;
    return 0;
}

static size_t expand_smem(const int rates[3], int dm) {
    const size_t LX = SP_CX + dm - 1, LY = SP_CY + dm - 1;
    const size_t TY = (size_t)rates[1] * SP_CY, TZ = (size_t)rates[2] * SP_CZ;
    const size_t kp = (size_t)(rates[0] + rates[1] + rates[2]) * dm;
    return (kp + TZ * LY * LX + TZ * TY * LX + SP_CZ * SP_CY * SP_CX) * sizeof(double) + 2 * TZ * TY * sizeof(int);
}

int spatial_tile(const SpatialPlan& p, const int rates[3]) {
    const int dm = pick_dm(p);
    if (!dm) return 0;
    return expand_smem(rates, dm) <= 200 * 1024 ? dm : 0;
}

template <int DM, int R1>
static void launch_expand_k(const ExpandArgs& A, size_t smem, dim3 blocks, cudaStream_t st) {
    auto kern = spatial_expand_kernel<DM, R1>;
    // always: the static tables count against the 48 KB default as well
    VSR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<blocks, SP_THREADS, smem, st>>>(A);
    VSR_LAUNCH_CHECK();
}

template <int DM>
static void launch_expand_dm(const ExpandArgs& A, size_t smem, dim3 blocks, cudaStream_t st) {
    switch (A.ax[0].r) {
        case 1: launch_expand_k<DM, 1>(A, smem, blocks, st); break;
        case 2: launch_expand_k<DM, 2>(A, smem, blocks, st); break;
        case 4: launch_expand_k<DM, 4>(A, smem, blocks, st); break;
        default: launch_expand_k<DM, 0>(A, smem, blocks, st); break;
    }
}

bool spatial_march_ok(const Dims& hr, const int rates[3], const SpatialPlan& p) {
    const int dm = spatial_tile(p, rates);
    return dm && dm == p.dm && march_ok(hr, rates, dm) &&
           p.kp_host.size() == (size_t)(rates[0] + rates[1] + rates[2]) * dm;
}

template <class T>
static void march_dispatch(const Dims& hr, const int rates[3], const SpatialPlan& p, const double* u,
                           const double* z, T* x, unsigned long long* bad, cudaStream_t st) {
    const int dm = p.dm;
    MarchArgs M{};
    M.m = (int)hr.m, M.n = (int)hr.n, M.s = (int)hr.s;
    M.ml = M.m / 2, M.nl = M.n / 2, M.sl = M.s / rates[2];
    M.dmin1 = p.dmin[0], M.dmin2 = p.dmin[1], M.dmin3 = p.dmin[2];
    const double* kp = p.kp_host.data();
    for (int i = 0; i < 2 * dm; ++i) M.k1[i] = kp[i], M.f1[i] = (float)kp[i];
    for (int i = 0; i < 2 * dm; ++i) M.k2[i] = kp[2 * dm + i], M.f2[i] = (float)kp[2 * dm + i];
    for (int i = 0; i < rates[2] * dm; ++i) M.k3[i] = kp[4 * dm + i], M.f3[i] = (float)kp[4 * dm + i];
    M.u = u, M.z = z, M.x = x, M.bad = bad;
    const unsigned tx = (unsigned)(M.ml / MX_CX), ty = (unsigned)(M.nl / MX_CY);
    const bool r4 = rates[2] == 4;
    // one tap set for all axes (bitwise equal; VSR_MARCH_ISO=0 forces the general kernel)
    static const bool iso_on = [] {
        const char* e = std::getenv("VSR_MARCH_ISO");
        return !(e && e[0] == '0');
    }();
    // The per-axis factors of an isotropic PSF come out of three different
    // lines of Lambda and differ in the last bits, so "equal" is within
    // 1e-14 of the largest tap (an output error below 1e-14 relative, the
    // same order as the 1e-14 support cut above); the shared set is the mean.
    bool iso = iso_on && !r4;
    double kmax = 0;
    for (int i = 0; i < 2 * dm; ++i) kmax = std::max(kmax, std::fabs(kp[i]));
    for (int i = 0; iso && i < 2 * dm; ++i)
        iso = std::fabs(kp[i] - kp[2 * dm + i]) <= 1e-14 * kmax && std::fabs(kp[i] - kp[4 * dm + i]) <= 1e-14 * kmax;
    if (iso)
        for (int i = 0; i < 2 * dm; ++i) {
            const double k = (kp[i] + kp[2 * dm + i] + kp[4 * dm + i]) / 3.0;
            M.k1[i] = M.k2[i] = M.k3[i] = k;
            M.f1[i] = M.f2[i] = M.f3[i] = (float)k;
        }
    if (const char* e = std::getenv("VSR_MARCH_DEBUG"))
        if (e[0] == '1') std::fprintf(stderr, "vsr: z-march dm=%d r3=%d iso=%d\n", dm, rates[2], (int)iso);
    switch (dm) {
        case 4: r4 ? launch_march_k<4, 4, T>(M, tx, ty, false, st) : launch_march_k<4, 2, T>(M, tx, ty, iso, st); break;
        case 5: r4 ? launch_march_k<5, 4, T>(M, tx, ty, false, st) : launch_march_k<5, 2, T>(M, tx, ty, iso, st); break;
        case 7: r4 ? launch_march_k<7, 4, T>(M, tx, ty, false, st) : launch_march_k<7, 2, T>(M, tx, ty, iso, st); break;
        default: r4 ? launch_march_k<8, 4, T>(M, tx, ty, false, st) : launch_march_k<8, 2, T>(M, tx, ty, iso, st); break;
    }
}

void launch_spatial_expand_f32(const Dims& hr, const int rates[3], const SpatialPlan& p, const double* u,
                               const double* z, float* x, unsigned long long* bad, cudaStream_t st) {
    if (!spatial_march_ok(hr, rates, p)) throw std::logic_error("spatial_expand (fp32): no z-march geometry");
    march_dispatch<float>(hr, rates, p, u, z, x, bad, st);
}

void launch_spatial_expand(const Dims& hr, const int rates[3], const SpatialPlan& p, const double* u,
                           const double* z, double c0, double* x, unsigned long long* bad, cudaStream_t st) {
    (void)c0;  // folded into u's inverse-FFT scale by the caller
    const int dm = spatial_tile(p, rates);
    if (!dm) throw std::logic_error("spatial_expand: support too wide for the tile budget");
    if (dm != p.dm) throw std::logic_error("spatial_expand: plan taps built for another width");
    if (march_ok(hr, rates, dm) && p.kp_host.size() == (size_t)(rates[0] + rates[1] + rates[2]) * dm) {
        march_dispatch<double>(hr, rates, p, u, z, x, bad, st);
        return;
    }
    ExpandArgs A;
    A.m = (int)hr.m, A.n = (int)hr.n, A.s = (int)hr.s;
    A.ml = A.m / rates[0], A.nl = A.n / rates[1], A.sl = A.s / rates[2];
    for (int a = 0; a < 3; ++a) A.ax[a] = AxisTaps{rates[a], p.dmin[a]};
    A.tiles1 = (A.ml + SP_CX - 1) / SP_CX;
    A.tiles2 = (A.nl + SP_CY - 1) / SP_CY;
    const int tiles3 = (A.sl + SP_CZ - 1) / SP_CZ;
    if ((size_t)rates[1] * rates[2] * SP_CY * SP_CZ > SP_MAX_ROWS || (size_t)A.tiles2 > 65535 || tiles3 > 65535)
        throw std::logic_error("spatial_expand: tile grid out of range");
    A.kp = p.kp;
    A.u = u, A.z = z, A.x = x, A.bad = bad;
    if ((size_t)A.ml * A.nl * A.sl >= (1ull << 31) || hr.count() >= (1ull << 40))
        throw std::logic_error("spatial_expand: LR volume exceeds 32-bit indexing");
    const size_t smem = expand_smem(rates, dm);
    const dim3 blocks((unsigned)A.tiles1, (unsigned)A.tiles2, (unsigned)tiles3);
    switch (dm) {
        case 4: launch_expand_dm<4>(A, smem, blocks, st); break;
        case 5: launch_expand_dm<5>(A, smem, blocks, st); break;
        case 7: launch_expand_dm<7>(A, smem, blocks, st); break;
        case 8: launch_expand_dm<8>(A, smem, blocks, st); break;
        case 12: launch_expand_dm<12>(A, smem, blocks, st); break;
        default: launch_expand_dm<16>(A, smem, blocks, st); break;
    }
}

// Phase-padded taps for a padded width dm: kp[phi * dm + i] = k[r (dmin + i) - phi + h]
// when |r (dmin + i) - phi| <= h, else 0; axes concatenated.
void spatial_phase_taps(const int rates[3], const int h[3], const int dmin[3], const std::vector<double>& taps,
                        int dm, std::vector<double>& out) {
    size_t off = 0;
    for (int a = 0; a < 3; ++a) {
        const int r = rates[a];
        for (int ph = 0; ph < r; ++ph)
            for (int i = 0; i < dm; ++i) {
                const int t = r * (dmin[a] + i) - ph;
                out.push_back(t >= -h[a] && t <= h[a] ? taps[off + t + h[a]] : 0.0);
            }
        off += 2 * h[a] + 1;
    }
}

// -------------------------------------------------------------- host plan
// From the separable spectral tables a (m), b (n), c (s): the 1-D spatial
// PSF factors k_a[p] = (1/L) sum_f a[f] e^{+2 pi i f p / L} (long double
// DFT), phase-normalised to real, with their circular half supports, and the
// per-axis alias sums of a and |a|^2.  Returns false (use the FFT path) when
// a factor is not real or not compact.
bool spatial_plan_host(const Dims& hr, const int rates[3], const std::vector<double2>& tabs,
                       std::vector<double>& taps, int h[3], std::vector<double2>& s1, std::vector<double>& s2) {
    using cld = std::complex<long double>;
    const size_t L[3] = {hr.m, hr.n, hr.s};
    const long double two_pi = 6.283185307179586476925286766559005768L;
    std::vector<std::vector<cld>> k(3);
    size_t off = 0;
    for (int a = 0; a < 3; ++a) {
        const size_t n = L[a];
        k[a].assign(n, cld(0, 0));
        std::vector<cld> tw(n);
        for (size_t j = 0; j < n; ++j) {
            const long double ang = two_pi * (long double)j / (long double)n;
            tw[j] = cld(std::cos(ang), std::sin(ang));
        }
        for (size_t p = 0; p < n; ++p) {
            cld acc(0, 0);
            for (size_t f = 0; f < n; ++f) acc += cld(tabs[off + f].x, tabs[off + f].y) * tw[(f * p) % n];
            k[a][p] = acc / (long double)n;
        }
        off += n;
    }
    // phase-normalise each factor by its largest entry; the product's phase goes to axis 3
    cld ph_total(1, 0);
    for (int a = 0; a < 3; ++a) {
        size_t imax = 0;
        for (size_t p = 1; p < L[a]; ++p)
            if (std::abs(k[a][p]) > std::abs(k[a][imax])) imax = p;
        const long double mag = std::abs(k[a][imax]);
        if (mag == 0) return false;
        const cld ph = k[a][imax] / mag;
        for (auto& v : k[a]) v /= ph;
        ph_total *= ph;
    }
    for (auto& v : k[2]) v *= ph_total;
    taps.clear();
    s1.clear();
    s2.clear();
    for (int a = 0; a < 3; ++a) {
        const size_t n = L[a];
        long double mx = 0;
        for (auto& v : k[a]) mx = std::max(mx, std::abs(v));
        const long double thr = 1e-14L * mx;
        for (auto& v : k[a])
            if (std::fabs(v.imag()) > 1e-12L * mx) return false;  // complex PSF factor
        // circular half support around the origin
        int hh = 0;
        for (size_t p = 0; p < n; ++p) {
            if (std::abs(k[a][p]) <= thr) continue;
            const size_t dist = std::min(p, n - p);
            hh = std::max(hh, (int)dist);
        }
        if (2 * (size_t)hh + 1 > n || hh > 64) return false;
        h[a] = hh;
        for (int p = -hh; p <= hh; ++p) {
            const size_t idx = (size_t)((p % (long long)n + (long long)n) % (long long)n);
            taps.push_back((double)k[a][idx].real());
        }
    }
    // alias sums of the tables along each axis (A1, A2 ...)
    off = 0;
    for (int a = 0; a < 3; ++a) {
        const size_t n = L[a], nlr = n / rates[a];
        for (size_t g = 0; g < nlr; ++g) {
            double2 acc1 = make_double2(0, 0);
            double acc2 = 0;
            for (int b = 0; b < rates[a]; ++b) {
                const double2 v = tabs[off + g + b * nlr];
                acc1.x += v.x, acc1.y += v.y;
                acc2 += v.x * v.x + v.y * v.y;
            }
            s1.push_back(acc1);
            s2.push_back(acc2);
        }
        off += n;
    }
    return true;
}

}  // namespace vsr
