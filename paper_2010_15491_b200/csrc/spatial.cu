// Spatial expansion path of the Tikhonov solve (see spatial.cuh for the
// algebra).  Two kernels: an LR pointwise kernel U(g) and a tiled 3-stage
// separable correlation that writes x in one HBM pass.
#include <algorithm>
#include <cmath>
#include <complex>
#include <vector>

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
constexpr int SP_THREADS = 256;
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
__global__ void __launch_bounds__(SP_THREADS, (DM <= 8 ? 4 : 3)) spatial_expand_kernel(ExpandArgs A) {
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
    __shared__ long long zoff[LZ];
    __shared__ int yoff[LY], xoff[LX];
    // stage-C row table: tz | ty << 8 | lattice << 16 (rows <= 256 * 256)
    __shared__ int rowinfo[SP_MAX_ROWS];

    const int tid = threadIdx.x;
    const int cx0 = blockIdx.x * SP_CX, cy0 = blockIdx.y * SP_CY, cz0 = blockIdx.z * SP_CZ;
    const int rows = TZ * TY;

    for (int i = tid; i < nkp; i += SP_THREADS) kp1[i] = A.kp[i];
    if (tid < LZ) zoff[tid] = (long long)wrap_idx(cz0 + A.ax[2].dmin + tid, A.sl) * A.nl * A.ml;
    else if (tid >= 32 && tid < 32 + LY) yoff[tid - 32] = wrap_idx(cy0 + A.ax[1].dmin + tid - 32, A.nl) * A.ml;
    else if (tid >= 64 && tid < 64 + LX) xoff[tid - 64] = wrap_idx(cx0 + A.ax[0].dmin + tid - 64, A.ml);
    for (int row = tid; row < rows; row += SP_THREADS) {
        const int tz = row / TY, ty = row - tz * TY;
        rowinfo[row] = tz | (ty << 8) | (((ty % r2) == 0 && (tz % r3) == 0) ? 1 << 16 : 0);
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
    const size_t zplane = (size_t)A.nl * A.ml;
    const int xb = tid % NXB, c0 = xb * SP_XB, n1 = X0 + r1 * c0;
    for (int row = tid / NXB; row < rows; row += SP_THREADS / NXB) {
        const int info = rowinfo[row];
        const int tz = info & 0xff, ty = (info >> 8) & 0xff;
        const int n2 = Y0 + ty, n3 = Z0 + tz;
        if (n2 >= A.n || n3 >= A.s || n1 >= A.m) continue;
        const bool lat = A.z != nullptr && (info >> 16);
        double zv[SP_XB];
        const double* zp = lat ? A.z + (size_t)(cz0 + tz / r3) * zplane + (size_t)(cy0 + ty / r2) * A.ml + cx0 + c0
                               : nullptr;
#pragma unroll
        for (int j = 0; j < SP_XB; ++j) zv[j] = lat ? __ldg(zp + j) : 0.0;
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
                for (int d = 0; d < DM; ++d) k[d] = kp1[ph * DM + d];
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

static const int kDms[] = {4, 8, 12, 16};

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
    return (kp + TZ * LY * LX + TZ * TY * LX) * sizeof(double);
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

void launch_spatial_expand(const Dims& hr, const int rates[3], const SpatialPlan& p, const double* u,
                           const double* z, double c0, double* x, unsigned long long* bad, cudaStream_t st) {
    (void)c0;  // folded into u's inverse-FFT scale by the caller
    const int dm = spatial_tile(p, rates);
    if (!dm) throw std::logic_error("spatial_expand: support too wide for the tile budget");
    if (dm != p.dm) throw std::logic_error("spatial_expand: plan taps built for another width");
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
    const size_t smem = expand_smem(rates, dm);
    const dim3 blocks((unsigned)A.tiles1, (unsigned)A.tiles2, (unsigned)tiles3);
    switch (dm) {
        case 4: launch_expand_dm<4>(A, smem, blocks, st); break;
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
