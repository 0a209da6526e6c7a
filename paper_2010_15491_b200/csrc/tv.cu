// ADMM-TV spatial kernels (see tv.cuh).
//
// The fused stencil marches a 32 x 8 column of voxels through a chunk of KC
// planes along axis 3 ("2.5D"): two x planes (with a one-voxel periodic halo)
// live in shared memory, rho_x / rho_y of the current plane are exchanged
// through shared memory for the divergence, and rho_z of the previous plane
// stays in a register.  Every HBM byte of x, dual, dual' and theta is touched
// once per iteration (halo re-reads hit L2).
#include <type_traits>

#include "tv.cuh"

namespace vsr {
namespace {

constexpr int TX = 32, TY = 8, STH = TX * TY;

__device__ __forceinline__ int wrapi(long long v, long long len) {
    while (v < 0) v += len;
    while (v >= len) v -= len;
    return (int)v;
}

struct Shrunk {
    double u0, u1, u2, dn0, dn1, dn2, r0, r1, r2;
};

// 1/sqrt(x) for finite x > 0: MUFU.RSQ64H seed (rsqrt.approx, ~2^-22) and two
// Newton steps (~2^-44, then ~1 ulp) - branch-free, unlike the libm rsqrt()
// whose denormal/inf handling costs ~17 % of the stencil's instructions.
__device__ __forceinline__ double fast_rsqrt(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    const double hx = 0.5 * x;
    y = y * fma(-hx * y, y, 1.5);
    y = y * fma(-hx * y, y, 1.5);
    return y;
}

// |v| and 1/|v| (0 for v = 0).  m2 below the normal range (|v| < 1e-154)
// takes the exact path.
__device__ __forceinline__ double norm3(double a, double b, double c, double* inv) {
    const double m2 = a * a + b * b + c * c;
    double r;
    if (m2 > 1e-300 && m2 < 1e300)
        r = fast_rsqrt(m2);
    else
        r = m2 > 0.0 ? rsqrt(m2) : 0.0;
    *inv = r;
    return m2 * r;
}

// fp32 mode (the fast stencil with S = float): the same shrink in fp32
struct ShrunkF {
    float u0, u1, u2, dn0, dn1, dn2, r0, r1, r2;
};
__device__ __forceinline__ float norm3(float a, float b, float c, float* inv) {
    const float m2 = a * a + b * b + c * c;
    float r;
    if (m2 > 1e-30f && m2 < 1e30f) {
        r = rsqrtf(m2);
        r = r * fmaf(-0.5f * m2 * r, r, 1.5f);  // one Newton step: ~1 ulp
    } else {
        r = m2 > 0.0f ? rsqrtf(m2) : 0.0f;
    }
    *inv = r;
    return m2 * r;
}
__device__ __forceinline__ ShrunkF shrink_point(float l0, float l1, float l2, float d0, float d1, float d2,
                                                float thr) {
    ShrunkF o;
    const float n0 = l0 + d0, n1 = l1 + d1, n2 = l2 + d2;
    float inv;
    const float mag = norm3(n0, n1, n2, &inv);
    const float f = mag > thr ? 1.0f - thr * inv : 0.0f;
    o.u0 = f * n0;
    o.u1 = f * n1;
    o.u2 = f * n2;
    o.dn0 = n0 - o.u0;
    o.dn1 = n1 - o.u1;
    o.dn2 = n2 - o.u2;
    o.r0 = o.u0 - o.dn0;
    o.r1 = o.u1 - o.dn1;
    o.r2 = o.u2 - o.dn2;
    return o;
}

// solvers.cpp:286-301 (factor = mag > t ? 1 - t/mag : 0) and :387-390;
// t/mag evaluated as t * rsqrt(mag^2).
__device__ __forceinline__ Shrunk shrink_point(double l0, double l1, double l2, double d0, double d1,
                                               double d2, double thr) {
    Shrunk o;
    const double n0 = l0 + d0, n1 = l1 + d1, n2 = l2 + d2;
    double inv;
    const double mag = norm3(n0, n1, n2, &inv);
    const double f = mag > thr ? 1.0 - thr * inv : 0.0;
    o.u0 = f * n0;
    o.u1 = f * n1;
    o.u2 = f * n2;
    o.dn0 = n0 - o.u0;
    o.dn1 = n1 - o.u1;
    o.dn2 = n2 - o.u2;
    o.r0 = o.u0 - o.dn0;
    o.r1 = o.u1 - o.dn1;
    o.r2 = o.u2 - o.dn2;
    return o;
}

__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

constexpr int XW = TX + 2, XH = TY + 2;  // x plane with halo [-1, TX] x [-1, TY]
constexpr int DW = TX + 1, DH = TY + 1;  // dual plane with low halo [-1, TX) x [-1, TY)
constexpr int NSLOT = 4;                  // plane ring: compute k, k+1; in flight k+2, k+3

__host__ __device__ constexpr size_t stencil_smem_doubles(bool init) {
    return (size_t)NSLOT * XH * XW + (init ? 0 : (size_t)NSLOT * 3 * DH * DW) + TY * (TX + 1) +
           (TY + 1) * TX;
}

// cp.async-pipelined march along axis 3: the x plane (with halo) and the three
// dual planes (with low halo) of z = k+3 are requested while plane k is
// computed, so one kernel keeps ~3 planes of loads in flight per CTA.
template <bool INIT, bool RELCHG>
__global__ void __launch_bounds__(STH)
    tv_stencil_kernel(int m, int n, int s, int KC, const double* __restrict__ x,
                      const double* __restrict__ dual_in, double* __restrict__ dual_out,
                      double* __restrict__ theta, double thr, const double* __restrict__ xprev,
                      double* __restrict__ partials) {
    extern __shared__ double sm[];
    double* xs = sm;                                            // [NSLOT][XH][XW]
    double* ds = xs + NSLOT * XH * XW;                          // [NSLOT][3][DH][DW]
    double* rx = ds + (INIT ? 0 : NSLOT * 3 * DH * DW);         // [TY][TX+1]
    double* ry = rx + TY * (TX + 1);                            // [TY+1][TX]
    __shared__ double red[32 * 4];

    const int tid = threadIdx.x;
    const int tx = tid % TX, ty = tid / TX;
    const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
    const int k0 = blockIdx.z * KC;
    const int k1 = min(k0 + KC, s);
    const long long plane = (long long)m * n;
    const long long N = plane * s;
    const int gi = i0 + tx, gj = j0 + ty;
    const bool valid = gi < m && gj < n;
    const long long col = valid ? (long long)gi + (long long)m * gj : 0;

    // per-thread load assignments (independent of z): 2 x elements, 2 dual elements
    long long xo[2], dof[2];
    bool xa[2], da[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int e = tid + q * STH;
        xa[q] = e < XH * XW;
        const int jj = (xa[q] ? e : 0) / XW - 1, ii = (xa[q] ? e : 0) % XW - 1;
        xo[q] = (long long)wrapi((long long)i0 + ii, m) + (long long)m * wrapi((long long)j0 + jj, n);
        da[q] = e < DH * DW;
        const int dj = (da[q] ? e : 0) / DW - 1, di = (da[q] ? e : 0) % DW - 1;
        dof[q] = (long long)wrapi((long long)i0 + di, m) + (long long)m * wrapi((long long)j0 + dj, n);
    }
    auto issue = [&](int z) {
        const int slot = (z - (k0 - 1)) & (NSLOT - 1);
        const long long zoff = plane * wrapi(z, s);
        double* xsl = xs + slot * XH * XW;
#pragma unroll
        for (int q = 0; q < 2; ++q)
            if (xa[q]) cp_async8(xsl + tid + q * STH, x + xo[q] + zoff);
        if (!INIT && z < k1) {
            double* dsl = ds + slot * 3 * DH * DW;
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int q = 0; q < 2; ++q)
                    if (da[q]) cp_async8(dsl + c * DH * DW + tid + q * STH, dual_in + c * N + dof[q] + zoff);
        }
        cp_async_commit();
    };

    double acc_res = 0.0, acc_tv = 0.0, acc_dx = 0.0, acc_xp = 0.0;
    double rz_prev = 0.0;

    issue(k0 - 1);
    issue(k0);
    issue(k0 + 1);
    for (int k = k0 - 1; k < k1; ++k) {
        if (k + 3 <= k1)
            issue(k + 3);
        else
            cp_async_commit();
        cp_async_wait<2>();
        __syncthreads();
        const bool warm = k < k0;
        const int sc = (k - (k0 - 1)) & (NSLOT - 1), sn = (sc + 1) & (NSLOT - 1);
        const double* X0 = xs + sc * XH * XW;
        const double* X1 = xs + sn * XH * XW;
        const double* D0 = ds + sc * 3 * DH * DW;
        const long long zoff = plane * wrapi(k, s);

        // ---- interior point (tx, ty)
        const double xc = X0[(ty + 1) * XW + tx + 1];
        const double l0 = X0[(ty + 1) * XW + tx + 2] - xc;
        const double l1 = X0[(ty + 2) * XW + tx + 1] - xc;
        const double l2 = X1[(ty + 1) * XW + tx + 1] - xc;
        double r0, r1, r2;
        if constexpr (INIT) {
            r0 = l0;
            r1 = l1;
            r2 = l2;
            if (!warm && valid) {
                const long long idx = col + zoff;
                dual_out[idx] = 0.0;
                dual_out[N + idx] = 0.0;
                dual_out[2 * N + idx] = 0.0;
                acc_tv += sqrt(l0 * l0 + l1 * l1 + l2 * l2);
            }
        } else {
            const int di = (ty + 1) * DW + tx + 1;
            const Shrunk o = shrink_point(l0, l1, l2, D0[di], D0[DH * DW + di], D0[2 * DH * DW + di], thr);
            r0 = o.r0;
            r1 = o.r1;
            r2 = o.r2;
            if (!warm && valid) {
                const long long idx = col + zoff;
                dual_out[idx] = o.dn0;
                dual_out[N + idx] = o.dn1;
                dual_out[2 * N + idx] = o.dn2;
                const double e0 = l0 - o.u0, e1 = l1 - o.u1, e2 = l2 - o.u2;
                acc_res += e0 * e0 + e1 * e1 + e2 * e2;
                acc_tv += sqrt(l0 * l0 + l1 * l1 + l2 * l2);
            }
        }
        if constexpr (RELCHG) {
            if (!warm && valid) {
                const double xp = __ldg(xprev + col + zoff);
                const double dd = xc - xp;
                acc_dx += dd * dd;
                acc_xp += xp * xp;
            }
        }
        if (!warm) {
            rx[ty * (TX + 1) + tx + 1] = r0;
            ry[(ty + 1) * TX + tx] = r1;
            // halo: rho_x at ii = -1 (jj = tid < TY), rho_y at jj = -1 (ii = tid - TY)
            if (tid < TY + TX) {
                const int ii = tid < TY ? -1 : tid - TY;
                const int jj = tid < TY ? tid : -1;
                const double hc = X0[(jj + 1) * XW + ii + 1];
                const double h0 = X0[(jj + 1) * XW + ii + 2] - hc;
                const double h1 = X0[(jj + 2) * XW + ii + 1] - hc;
                const double h2 = X1[(jj + 1) * XW + ii + 1] - hc;
                double q0, q1;
                if constexpr (INIT) {
                    q0 = h0;
                    q1 = h1;
                } else {
                    const int hi = (jj + 1) * DW + ii + 1;
                    const Shrunk o =
                        shrink_point(h0, h1, h2, D0[hi], D0[DH * DW + hi], D0[2 * DH * DW + hi], thr);
                    q0 = o.r0;
                    q1 = o.r1;
                }
                if (tid < TY)
                    rx[jj * (TX + 1)] = q0;
                else
                    ry[ii] = q1;
            }
        }
        __syncthreads();
        if (!warm && valid) {
            // diff_adjoint sum in axis order (solvers.cpp:367-373): ((adj_x) + adj_y) + adj_z
            const double ax = rx[ty * (TX + 1) + tx] - rx[ty * (TX + 1) + tx + 1];
            const double ay = ry[ty * TX + tx] - ry[(ty + 1) * TX + tx];
            const double az = rz_prev - r2;
            theta[col + zoff] = (ax + ay) + az;
        }
        rz_prev = r2;
    }
    cp_async_wait<0>();

    double v[4] = {acc_res, acc_tv, acc_dx, acc_xp};
    block_reduce_sum<4>(v, red);
    if (tid == 0) {
        const size_t b = blockIdx.x + (size_t)gridDim.x * (blockIdx.y + (size_t)gridDim.y * blockIdx.z);
#pragma unroll
        for (int q = 0; q < 4; ++q) partials[b * 4 + q] = v[q];
    }
}

// ---------------------------------------------------------------- fast path
// Same march, for even m: planes move as aligned 16-byte pairs staged through
// registers one step ahead (x plane k+2 and dual plane k+1 are in flight while
// plane k is computed), all per-thread load offsets are computed once, and
// the plane pointer advances incrementally.  ~4x fewer issued instructions
// than the element-wise cp.async variant above.
constexpr int FXW = TX + 4;                 // x row in smem: columns i0-2 .. i0+33
constexpr int FDW = TX + 2;                 // dual row: columns i0-2 .. i0+31
constexpr int FXH = TY + 2, FDH = TY + 1;   // x rows j0-1 .. j0+TY; dual rows j0-1 .. j0+TY-1
constexpr int FXP = FXH * (FXW / 2);        // 180 x pairs per plane
constexpr int FDP = FDH * (FDW / 2);        // 153 dual pairs per component
constexpr int FXS = FXH * FXW, FDS = 3 * FDH * FDW;

constexpr int FRS = TY * (TX + 1) + (TY + 1) * TX;  // one rho_x + rho_y exchange set
__host__ __device__ constexpr size_t fast_smem_doubles() {
    return (size_t)3 * FXS + 2 * FDS + 2 * FRS;  // two exchange sets, alternating by step
}


// S = double: the reference precision.  S = float (fp32 mode): x, dual,
// dual' and theta are stored in fp32 (half the HBM bytes); the stencil
// arithmetic, the shared-memory planes and the reductions stay fp64.
template <bool INIT, bool RELCHG, class S = double>
__global__ void __launch_bounds__(STH)
    tv_stencil_fast_kernel(int m, int n, int s, int KC, const S* __restrict__ x,
                           const S* __restrict__ dual_in, S* __restrict__ dual_out,
                           S* __restrict__ theta, double thr, const S* __restrict__ xprev,
                           double* __restrict__ partials, int halo, long long dsi, long long dso,
                           const S* __restrict__ ylo_x = nullptr, const S* __restrict__ yhi_x = nullptr,
                           const S* __restrict__ ylo_d = nullptr) {
    using S2 = std::conditional_t<std::is_same<S, double>::value, double2, float2>;
    extern __shared__ double sm_raw[];
    S* sm = reinterpret_cast<S*>(sm_raw);
    S* const rxy = sm + 3 * FXS + 2 * FDS;  // two sets of rx [TY][TX+1], ry [TY+1][TX]
    __shared__ double red[32 * 4];

    const int tid = threadIdx.x;
    const int tx = tid % TX, ty = tid / TX;
    const int i0 = blockIdx.x * TX, j0 = blockIdx.y * TY;
    const int k0 = blockIdx.z * KC;
    const int k1 = min(k0 + KC, s);
    const long long plane = (long long)m * n;
    const bool valid = (i0 + tx) < m && (j0 + ty) < n;
    const int col = valid ? (i0 + tx) + m * (j0 + ty) : 0;

    auto wrap = [](int v, int len) {
        v %= len;
        return v < 0 ? v + len : v;
    };
    // y-slab mode (slab.cu: ylo_x set): axis 2 is not periodic here; the halo
    // rows -1 and n come from the neighbouring ranks' x (and dual) slabs, read
    // in place over NVLink peer memory (row n-1 of the lower one, row 0 of the
    // upper one; same plane stride)
    const bool yslab = ylo_x != nullptr;
    auto yrow = [&](int jr, const S*& base, const S* lo, const S* hi) {
        if (!yslab) return wrap(jr, n);
        if (jr < 0) {
            base = lo;
            return n - 1;
        }
        if (jr >= n) {
            // (no upper neighbour for the dual: rows past the slab are only reached
            // when the slab is shorter than a tile, and never used; read row n - 1)
            if (!hi) return n - 1;
            base = hi;
            return 0;
        }
        return jr;
    };
    // load assignments: one x pair (tid < FXP), up to two dual pairs
    const bool xa = tid < FXP;
    int xoff = 0, xsm = 0;
    const S* xsrc = x;
    if (xa) {
        const int row = tid / (FXW / 2), pc = tid % (FXW / 2);
        xoff = wrap(i0 - 2 + 2 * pc, m) + m * yrow(j0 - 1 + row, xsrc, ylo_x, yhi_x);
        xsm = row * FXW + 2 * pc;
    }
    bool da[2];
    long long doff[2];
    int dsm[2];
    const S* dsrc[2] = {dual_in, dual_in};
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int e = tid + q * STH;
        da[q] = !INIT && e < 3 * FDP;
        const int c = da[q] ? e / FDP : 0, rem = da[q] ? e % FDP : 0;
        const int row = rem / (FDW / 2), pc = rem % (FDW / 2);
        doff[q] = (long long)c * dsi + wrap(i0 - 2 + 2 * pc, m) +
                  (long long)m * yrow(j0 - 1 + row, dsrc[q], ylo_d, nullptr);
        dsm[q] = c * FDH * FDW + row * FDW + 2 * pc;
    }
    // plane pointers advance by one plane per step; in periodic mode they wrap
    // only where z leaves [0, s) (z = -1 at the chunk start, z = s at its end)
    auto zp = [&](int z) -> long long {
        return plane * (long long)(halo ? z : (z < 0 ? z + s : (z >= s ? z - s : z)));
    };
    // smem ring: x slots rotate through three buffers, dual through two
    S* xsl[3] = {sm, sm + FXS, sm + 2 * FXS};
    S* dsl[2] = {sm + 3 * FXS, sm + 3 * FXS + FDS};
    auto ld_pair = [](const S* p) { return __ldg(reinterpret_cast<const S2*>(p)); };

    S2 rxv{}, rdv[2] = {S2{}, S2{}};
    // prologue: x(k0-1), x(k0), dual(k0-1) resident; x(k0+1), dual(k0) in registers
    if (xa) *reinterpret_cast<S2*>(xsl[0] + xsm) = ld_pair(xsrc + zp(k0 - 1) + xoff);
    if (!INIT) {
        const long long zo = zp(k0 - 1);
#pragma unroll
        for (int q = 0; q < 2; ++q)
            if (da[q]) *reinterpret_cast<S2*>(dsl[0] + dsm[q]) = ld_pair(dsrc[q] + zo + doff[q]);
    }
    if (xa) *reinterpret_cast<S2*>(xsl[1] + xsm) = ld_pair(xsrc + zp(k0) + xoff);
    const S* xnext = xsrc + xoff;    // advanced below; holds plane k+3 at step k
    const S* dnext[2] = {dsrc[0] + doff[0], dsrc[1] + doff[1]};  // plane k+2 at step k
    long long zx = zp(k0 + 1), zd = zp(k0);
    if (xa && k0 + 1 <= k1) rxv = ld_pair(xnext + zx);
    if (!INIT && k0 < k1) {
#pragma unroll
        for (int q = 0; q < 2; ++q)
            if (da[q]) rdv[q] = ld_pair(dnext[q] + zd);
    }
    // halo points (rho_x at ii = -1 for TY rows, rho_y at jj = -1 for TX columns)
    // packed into whole warps: warp 0 takes the TX row points, warp 1 the TY
    // column points, so the other warps skip the halo shrink entirely
    const int lane = tid & 31, warp = tid >> 5;
    const int hslot = warp == 0 ? TY + lane : (warp == 1 && lane < TY ? lane : -1);
    const bool hwork = hslot >= 0 && hslot < TY + TX;
    const int hii = hslot < TY ? -1 : hslot - TY;
    const int hjj = hslot < TY ? hslot : -1;
    const int hx = (hjj + 1) * FXW + hii + 2;
    const int hd = (hjj + 1) * FDW + hii + 2;
    const int xi = (ty + 1) * FXW + tx + 2;
    const int di = (ty + 1) * FDW + tx + 2;

    double acc_res = 0.0, acc_tv = 0.0, acc_dx = 0.0, acc_xp = 0.0;
    S rz_prev = 0;
    const S thr_s = (S)thr;
    long long zo = zp(k0 - 1);
    // The march is unrolled by 6 (lcm of the x ring of 3 slots and the dual ring
    // of 2), so every slot is a compile-time offset of the shared-memory base.
    // steady steps (k0 <= k, k + 4 <= k1: planes k-1 .. k+3 inside [0, s), no
    // warm-up, every look-ahead load due) drop the per-plane bounds and wrap tests
    // ONE barrier per step.  Plane k + 2 (x) / k + 1 (dual) goes into the slot
    // nobody reads during step k, and is first read in step k + 1, after this
    // step's barrier; the slot's previous plane was last read before the previous
    // step's barrier.  The rho exchange set alternates by step parity, so step
    // k + 1's writes cannot overtake step k's reads after the barrier.
    auto step = [&](int k, auto x0, auto x1, auto x2, auto d0, auto d1, auto par, auto steady) {
        constexpr bool ST = decltype(steady)::value;
        S* const rx = rxy + decltype(par)::value * FRS;
        S* const ry = rx + TY * (TX + 1);
        S* const XS0 = sm + decltype(x0)::value * FXS;
        S* const XS1 = sm + decltype(x1)::value * FXS;
        S* const XS2 = sm + decltype(x2)::value * FXS;
        S* const DS0 = sm + 3 * FXS + decltype(d0)::value * FDS;
        S* const DS1 = sm + 3 * FXS + decltype(d1)::value * FDS;
        // registers -> smem for step k+1, then request x(k+3), dual(k+2)
        if ((ST || k + 2 <= k1) && xa) *reinterpret_cast<S2*>(XS2 + xsm) = rxv;
        if (!INIT && (ST || k + 1 <= k1 - 1)) {
#pragma unroll
            for (int q = 0; q < 2; ++q)
                if (da[q]) *reinterpret_cast<S2*>(DS1 + dsm[q]) = rdv[q];
        }
        if (ST || k + 3 <= k1) {
            zx += plane;
            if (!ST && !halo && zx >= plane * s) zx -= plane * s;
            if (xa) rxv = ld_pair(xnext + zx);
        }
        if (!INIT && (ST || k + 2 <= k1 - 1)) {
            zd += plane;
            if (!ST && !halo && zd >= plane * s) zd -= plane * s;
#pragma unroll
            for (int q = 0; q < 2; ++q)
                if (da[q]) rdv[q] = ld_pair(dnext[q] + zd);
        }
        const bool warm = !ST && k < k0;
        const S* X0 = XS0;
        const S* X1 = XS1;
        [[maybe_unused]] const S* D0 = DS0;

        const S xc = X0[xi];
        const S l0 = X0[xi + 1] - xc;
        const S l1 = X0[xi + FXW] - xc;
        const S l2 = X1[xi] - xc;
        S r0, r1, r2;
        if constexpr (INIT) {
            r0 = l0;
            r1 = l1;
            r2 = l2;
            if (!warm && valid) {
                const long long idx = col + zo;
                dual_out[idx] = (S)0;
                dual_out[dso + idx] = (S)0;
                dual_out[2 * dso + idx] = (S)0;
                {
                    S inv_;
                    acc_tv += (double)norm3(l0, l1, l2, &inv_);
                }
            }
        } else {
            const auto o = shrink_point(l0, l1, l2, D0[di], D0[FDH * FDW + di], D0[2 * FDH * FDW + di], thr_s);
            r0 = o.r0;
            r1 = o.r1;
            r2 = o.r2;
            if (!warm && valid) {
                const long long idx = col + zo;
                dual_out[idx] = o.dn0;
                dual_out[dso + idx] = o.dn1;
                dual_out[2 * dso + idx] = o.dn2;
                const double e0 = l0 - o.u0, e1 = l1 - o.u1, e2 = l2 - o.u2;
                acc_res += e0 * e0 + e1 * e1 + e2 * e2;
                {
                    S inv_;
                    acc_tv += (double)norm3(l0, l1, l2, &inv_);
                }
            }
        }
        if constexpr (RELCHG) {
            if (!warm && valid) {
                const double xp = (double)__ldg(xprev + col + zo);
                const double dd = xc - xp;
                acc_dx += dd * dd;
                acc_xp += xp * xp;
            }
        }
        if (!warm) {
            rx[ty * (TX + 1) + tx + 1] = r0;
            ry[(ty + 1) * TX + tx] = r1;
            if (hwork) {  // halo: rho_x at ii = -1, rho_y at jj = -1
                const S hc = X0[hx];
                const S h0 = X0[hx + 1] - hc;
                const S h1 = X0[hx + FXW] - hc;
                [[maybe_unused]] const S h2 = X1[hx] - hc;
                S q0, q1;
                if constexpr (INIT) {
                    q0 = h0;
                    q1 = h1;
                } else {
                    const auto o =
                        shrink_point(h0, h1, h2, D0[hd], D0[FDH * FDW + hd], D0[2 * FDH * FDW + hd], thr_s);
                    q0 = o.r0;
                    q1 = o.r1;
                }
                if (hslot < TY)
                    rx[hjj * (TX + 1)] = q0;
                else
                    ry[hii] = q1;
            }
        }
        __syncthreads();
        if (!warm && valid) {
            // diff_adjoint sum in axis order (solvers.cpp:367-373): ((adj_x) + adj_y) + adj_z
            const S ax = rx[ty * (TX + 1) + tx] - rx[ty * (TX + 1) + tx + 1];
            const S ay = ry[ty * TX + tx] - ry[(ty + 1) * TX + tx];
            const S az = rz_prev - r2;
            theta[col + zo] = (ax + ay) + az;
        }
        rz_prev = r2;
        // rotate the rings: x slots (k, k+1, k+2) -> (k+1, k+2, k+3); dual (k, k+1) -> (k+1, k+2)
        zo += plane;
        if (!ST && !halo && zo >= plane * s) zo -= plane * s;
    };
    using I0 = std::integral_constant<int, 0>;
    using I1 = std::integral_constant<int, 1>;
    using I2 = std::integral_constant<int, 2>;
    // (fp32 only: at fp64 the second step body costs spills at the 64-register
    // allocation, 229 vs 219 us; fp32 160 -> 154 us)
    constexpr bool kSteady = std::is_same<S, float>::value;
    auto any_step = [&](int k, auto x0, auto x1, auto x2, auto d0, auto d1, auto par) {
        if (kSteady && k >= k0 && k + 4 <= k1)
            step(k, x0, x1, x2, d0, d1, par, std::true_type{});
        else if (k < k1)
            step(k, x0, x1, x2, d0, d1, par, std::false_type{});
    };
    __syncthreads();  // the prologue's planes
    for (int k = k0 - 1; k < k1; k += 6) {
        any_step(k, I0{}, I1{}, I2{}, I0{}, I1{}, I0{});
        any_step(k + 1, I1{}, I2{}, I0{}, I1{}, I0{}, I1{});
        any_step(k + 2, I2{}, I0{}, I1{}, I0{}, I1{}, I0{});
        any_step(k + 3, I0{}, I1{}, I2{}, I1{}, I0{}, I1{});
        any_step(k + 4, I1{}, I2{}, I0{}, I0{}, I1{}, I0{});
        any_step(k + 5, I2{}, I0{}, I1{}, I1{}, I0{}, I1{});
    }

    double v[4] = {acc_res, acc_tv, acc_dx, acc_xp};
    block_reduce_sum<4>(v, red);
    if (tid == 0) {
        const size_t b = blockIdx.x + (size_t)gridDim.x * (blockIdx.y + (size_t)gridDim.y * blockIdx.z);
#pragma unroll
        for (int q = 0; q < 4; ++q) partials[b * 4 + q] = v[q];
    }
}

// Sum `nvals` interleaved per-block partials in a fixed order.
__device__ void fixed_sum(const double* p, int stride, int nvals, long long nblocks, double* out,
                          double* red) {
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (long long i = threadIdx.x; i < nblocks; i += blockDim.x)
        for (int k = 0; k < nvals; ++k) v[k] += p[i * stride + k];
    block_reduce_sum<4>(v, red);
    __syncthreads();
    if (threadIdx.x == 0)
        for (int k = 0; k < nvals; ++k) out[k] = v[k];
    __syncthreads();
}

__global__ void __launch_bounds__(1024)
    tv_finalize_kernel(int iter, const double* fitp, long long fitn, const double* stp,
                       long long stn, const double* resp, long long resn, double tv_weight,
                       double max_rel_imag, TvIterScalars sc, double* init_obj) {
    __shared__ double red[32 * 4];
    __shared__ double vals[12];
    fixed_sum(fitp, 1, 1, fitn, vals + 0, red);
    fixed_sum(stp, 4, 4, stn, vals + 4, red);
    if (resp) fixed_sum(resp, 2, 2, resn, vals + 8, red);
    if (threadIdx.x == 0) {
        const double fit = vals[0];
        const double resid = vals[4], tv = vals[5], dx2 = vals[6], xp2 = vals[7];
        const double obj = 0.5 * fit + tv_weight * tv;  // solvers.cpp:401, :318
        if (init_obj) {
            *init_obj = obj;
        } else {
            if (sc.iter_dev) iter = (*sc.iter_dev)++;
            sc.objective[iter] = obj;
            sc.primal_residual[iter] = sqrt(resid);
            sc.rel_change[iter] = sqrt(dx2) / fmax(sqrt(xp2), 1e-300);
            if (resp) {
                const double im2 = vals[8], tot2 = vals[9];
                const double ratio = tot2 > 0.0 ? sqrt(im2 / tot2) : 0.0;
                sc.status[2] = ratio;
                if (tot2 > 0.0 && ratio > max_rel_imag && sc.status[0] < 0.0) {
                    sc.status[0] = (double)iter;
                    sc.status[1] = ratio;
                }
            }
        }
    }
}

// ---------------------------------------------------------------- elementwise
__global__ void decimate_kernel(long long m, long long n, int dr, int dc, int ds, long long ml,
                                long long nl, long long Nl, const double* __restrict__ x,
                                double* __restrict__ y) {
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= Nl) return;
    const long long i = g % ml, j = (g / ml) % nl, k = g / (ml * nl);
    y[g] = x[i * dr + m * (j * dc + n * (k * ds))];
}

__global__ void decimate_adjoint_kernel(long long m, long long n, int dr, int dc, int ds,
                                        long long N, double scale, const double* __restrict__ y,
                                        long long ml, long long nl, double* __restrict__ x) {
    const long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= N) return;
    const long long i = f % m, j = (f / m) % n, k = f / (m * n);
    double v = 0.0;
    if (i % dr == 0 && j % dc == 0 && k % ds == 0) v = y[i / dr + ml * (j / dc + nl * (k / ds))] * scale;
    x[f] = v;
}

__global__ void nn_upsample_kernel(long long m, long long n, int dr, int dc, int ds, long long N,
                                   const double* __restrict__ y, long long ml, long long nl,
                                   double* __restrict__ x) {
    const long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (f >= N) return;
    const long long i = f % m, j = (f / m) % n, k = f / (m * n);
    x[f] = y[i / dr + ml * (j / dc + nl * (k / ds))];
}

__global__ void diff_kernel(long long m, long long n, long long s, int axis, bool adjoint,
                            const double* __restrict__ x, double* __restrict__ out) {
    const long long N = m * n * s;
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= N) return;
    const long long i = p % m, j = (p / m) % n, k = p / (m * n);
    const long long pos = axis == 0 ? i : (axis == 1 ? j : k);
    const long long len = axis == 0 ? m : (axis == 1 ? n : s);
    const long long stride = axis == 0 ? 1 : (axis == 1 ? m : m * n);
    long long q;
    if (!adjoint)
        q = (pos + 1 == len) ? p - (len - 1) * stride : p + stride;  // operators.cpp:201-203
    else
        q = (pos == 0) ? p + (len - 1) * stride : p - stride;  // operators.cpp:218-220
    out[p] = x[q] - x[p];
}

__global__ void shrink_kernel(long long count, const double* __restrict__ a,
                              const double* __restrict__ b, const double* __restrict__ c,
                              double thr, double* __restrict__ o1, double* __restrict__ o2,
                              double* __restrict__ o3) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= count) return;
    const double n0 = a[p], n1 = b[p], n2 = c[p];
    const double mag = sqrt(n0 * n0 + n1 * n1 + n2 * n2);
    const double f = mag > thr ? 1.0 - thr / mag : 0.0;
    o1[p] = f * n0;
    o2[p] = f * n1;
    o3[p] = f * n2;
}

__global__ void gamma_kernel(long long m, long long n, long long N, const double* __restrict__ nr,
                             const double* __restrict__ nc, const double* __restrict__ ns,
                             double tau, double* __restrict__ g) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= N) return;
    const long long i = p % m, j = (p / m) % n, k = p / (m * n);
    g[p] = 1.0 / (((nr[i] + nc[j]) + ns[k]) + tau);  // solvers.cpp:196-202
}

__global__ void tv_norm_kernel(long long m, long long n, long long s, const double* __restrict__ x,
                               double* __restrict__ partials) {
    __shared__ double red[32];
    const long long N = m * n * s;
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double acc = 0.0;
    if (p < N) {
        const long long i = p % m, j = (p / m) % n, k = p / (m * n);
        const double xc = x[p];
        const double g0 = x[(i + 1 == m) ? p - (m - 1) : p + 1] - xc;
        const double g1 = x[(j + 1 == n) ? p - (n - 1) * m : p + m] - xc;
        const double g2 = x[(k + 1 == s) ? p - (s - 1) * m * n : p + m * n] - xc;
        acc = sqrt(g0 * g0 + g1 * g1 + g2 * g2);
    }
    double v[1] = {acc};
    block_reduce_sum<1>(v, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = v[0];
}

unsigned blocks256(long long n) { return (unsigned)((n + 255) / 256); }

}  // namespace

StencilGeom stencil_geom(const Dims& d) {
    StencilGeom g;
    const unsigned gx = (unsigned)((d.m + TX - 1) / TX), gy = (unsigned)((d.n + TY - 1) / TY);
    // chunk so that the grid has >= ~16 waves of 148 SMs when possible
    const long long tiles = (long long)gx * gy;
    int kc = 16;
    while (kc > 4 && tiles * (((long long)d.s + kc - 1) / kc) < 148 * 16) kc >>= 1;
    g.kc = kc;
    g.grid = dim3(gx, gy, (unsigned)((d.s + kc - 1) / kc));
    return g;
}

void launch_tv_stencil(const Dims& d, bool init, const double* x, const double* dual_in,
                       double* dual_out, double* theta, double thr, const double* xprev,
                       double* partials, cudaStream_t st) {
    const StencilGeom g = stencil_geom(d);
    const int m = (int)d.m, n = (int)d.n, s = (int)d.s;
    if (m % 2 == 0) {
        const size_t smem = fast_smem_doubles() * sizeof(double);
        const long long N = (long long)d.count();
#define VSR_FAST(I, R)                                                                               \
    tv_stencil_fast_kernel<I, R><<<g.grid, STH, smem, st>>>(m, n, s, g.kc, x, dual_in, dual_out, theta, \
                                                            thr, xprev, partials, 0, N, N)
        if (init)
            VSR_FAST(true, false);
        else if (xprev)
            VSR_FAST(false, true);
        else
            VSR_FAST(false, false);
#undef VSR_FAST
        VSR_LAUNCH_CHECK();
        return;
    }
    const size_t smem = stencil_smem_doubles(init) * sizeof(double);
    if (init) {
        tv_stencil_kernel<true, false><<<g.grid, STH, smem, st>>>(m, n, s, g.kc, x, dual_in, dual_out,
                                                                  theta, thr, xprev, partials);
    } else if (xprev) {
        tv_stencil_kernel<false, true><<<g.grid, STH, smem, st>>>(m, n, s, g.kc, x, dual_in, dual_out,
                                                                  theta, thr, xprev, partials);
    } else {
        tv_stencil_kernel<false, false><<<g.grid, STH, smem, st>>>(m, n, s, g.kc, x, dual_in, dual_out,
                                                                   theta, thr, xprev, partials);
    }
    VSR_LAUNCH_CHECK();
}

void launch_tv_stencil_f32(const Dims& d, bool init, const float* x, const float* dual_in, float* dual_out,
                           float* theta, double thr, const float* xprev, double* partials, cudaStream_t st) {
    const StencilGeom g = stencil_geom(d);
    const int m = (int)d.m, n = (int)d.n, s = (int)d.s;
    if (m % 2) throw std::logic_error("tv stencil (fp32 mode): axis 1 must be even");
    const size_t smem = fast_smem_doubles() * sizeof(float);
    const long long N = (long long)d.count();
#define VSR_FAST(I, R)                                                                                      \
    tv_stencil_fast_kernel<I, R, float><<<g.grid, STH, smem, st>>>(m, n, s, g.kc, x, dual_in, dual_out, theta, \
                                                                   thr, xprev, partials, 0, N, N)
    if (init)
        VSR_FAST(true, false);
    else if (xprev)
        VSR_FAST(false, true);
    else
        VSR_FAST(false, false);
#undef VSR_FAST
    VSR_LAUNCH_CHECK();
}

void launch_tv_finalize(int iter, const double* fit_partials, size_t fit_blocks,
                        const double* st_partials, size_t st_blocks, const double* res_partials,
                        size_t res_blocks, double tv_weight, double max_rel_imag,
                        TvIterScalars sc, double* init_objective_out, cudaStream_t st) {
    tv_finalize_kernel<<<1, 1024, 0, st>>>(iter, fit_partials, (long long)fit_blocks, st_partials,
                                           (long long)st_blocks, res_partials,
                                           (long long)res_blocks, tv_weight, max_rel_imag, sc,
                                           init_objective_out);
    VSR_LAUNCH_CHECK();
}

void launch_decimate(const Dims& hr, const int rates[3], const double* x, double* y,
                     cudaStream_t st) {
    const long long ml = hr.m / rates[0], nl = hr.n / rates[1], sl = hr.s / rates[2];
    const long long Nl = ml * nl * sl;
    decimate_kernel<<<blocks256(Nl), 256, 0, st>>>((long long)hr.m, (long long)hr.n, rates[0],
                                                   rates[1], rates[2], ml, nl, Nl, x, y);
    VSR_LAUNCH_CHECK();
}

void launch_decimate_adjoint(const Dims& hr, const int rates[3], const double* y, double* x,
                             double scale, cudaStream_t st) {
    const long long N = (long long)hr.count();
    decimate_adjoint_kernel<<<blocks256(N), 256, 0, st>>>(
        (long long)hr.m, (long long)hr.n, rates[0], rates[1], rates[2], N, scale, y,
        (long long)(hr.m / rates[0]), (long long)(hr.n / rates[1]), x);
    VSR_LAUNCH_CHECK();
}

void launch_nn_upsample(const Dims& hr, const int rates[3], const double* y, double* x,
                        cudaStream_t st) {
    const long long N = (long long)hr.count();
    nn_upsample_kernel<<<blocks256(N), 256, 0, st>>>((long long)hr.m, (long long)hr.n, rates[0],
                                                     rates[1], rates[2], N, y,
                                                     (long long)(hr.m / rates[0]),
                                                     (long long)(hr.n / rates[1]), x);
    VSR_LAUNCH_CHECK();
}

void launch_diff(const Dims& d, int axis, bool adjoint, const double* x, double* out,
                 cudaStream_t st) {
    diff_kernel<<<blocks256((long long)d.count()), 256, 0, st>>>(
        (long long)d.m, (long long)d.n, (long long)d.s, axis, adjoint, x, out);
    VSR_LAUNCH_CHECK();
}

void launch_shrink(size_t count, const double* nu1, const double* nu2, const double* nu3,
                   double thr, double* o1, double* o2, double* o3, cudaStream_t st) {
    shrink_kernel<<<blocks256((long long)count), 256, 0, st>>>((long long)count, nu1, nu2, nu3, thr,
                                                              o1, o2, o3);
    VSR_LAUNCH_CHECK();
}

void launch_gamma(const Dims& d, const double* nr, const double* nc, const double* ns, double tau,
                  double* gamma, cudaStream_t st) {
    const long long N = (long long)d.count();
    gamma_kernel<<<blocks256(N), 256, 0, st>>>((long long)d.m, (long long)d.n, N, nr, nc, ns, tau,
                                               gamma);
    VSR_LAUNCH_CHECK();
}

size_t tv_norm_blocks(const Dims& d) { return blocks256((long long)d.count()); }

void launch_tv_norm(const Dims& d, const double* x, double* partials, cudaStream_t st) {
    tv_norm_kernel<<<blocks256((long long)d.count()), 256, 0, st>>>(
        (long long)d.m, (long long)d.n, (long long)d.s, x, partials);
    VSR_LAUNCH_CHECK();
}

void launch_tv_stencil_yslab(const Dims& loc, bool init, const double* x, const double* dual_in, double* dual_out,
                             double* theta, double thr, const double* xprev, double* partials, const double* ylo_x,
                             const double* yhi_x, const double* ylo_d, cudaStream_t st) {
    if (loc.m % 2 != 0) throw std::invalid_argument("slab stencil: axis 1 must be even");
    const StencilGeom g = stencil_geom(loc);
    const int m = (int)loc.m, n = (int)loc.n, s = (int)loc.s;
    const long long N = (long long)loc.count();
    const size_t smem = fast_smem_doubles() * sizeof(double);
#define VSR_FAST(I, R)                                                                                          \
    tv_stencil_fast_kernel<I, R><<<g.grid, STH, smem, st>>>(m, n, s, g.kc, x, dual_in, dual_out, theta, thr, xprev, \
                                                            partials, 0, N, N, ylo_x, yhi_x, ylo_d)
    if (init)
        VSR_FAST(true, false);
    else if (xprev)
        VSR_FAST(false, true);
    else
        VSR_FAST(false, false);
#undef VSR_FAST
    VSR_LAUNCH_CHECK();
}

}  // namespace vsr
