// Pipelined ADMM-TV x-update "sandwich" on the Hermitian half spectrum
// (forward axis-1 FFT -> Gamma-weighted fold -> inverse axis-1 FFT), the
// dominant spectral kernel of an ADMM-TV iteration.  Same arithmetic as the
// Gw branch of fold_axis1_tile (fused.cu), reference solvers.cpp:219-233
// (tv_x_core) with k = conj(Lambda) F D^H y + mu theta_hat (:342-344, :375)
// and spectral.cpp:101-113 (apply_adjoint_weighted).
//
// Why a second kernel: the one-tile-per-CTA version holds 16 values per
// thread (128 registers), so an SM runs 2 CTAs and a CTA's HBM reads, its FFT
// arithmetic and its HBM writes run one after another; DRAM idles whenever
// both CTAs compute.  Here a persistent CTA of two 256-thread groups keeps
// three tile buffers in shared memory: while the two groups transform and
// fold two tiles, the third buffer is being filled by the bulk-copy engine
// (cp.async.bulk rows -> smem, completion on an mbarrier).  A group that
// finishes its last shared-memory exchange hands its buffer straight to the
// bulk engine for the tile three ahead, then writes its results from
// registers (full 32-byte sectors).  Lambda comes from the separable tables
// (a[f1] from shared memory, b[f2] c[f3] per line), Gamma from the per-axis
// tables, Gw(g) and the LR spectrum of y from L2: no per-element tables in
// shared memory and no register-staged loads.
#include "fft.cuh"
#include "fft_core.cuh"
#include "fused.cuh"

#include <algorithm>
#include <type_traits>
#include <cstdlib>
#include <vector>

namespace vsr {
namespace {

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared bulk copy, completion counted on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// named barrier over one thread group (id 0 is __syncthreads)
template <int NT>
struct GroupSync {
    int id;
    __device__ __forceinline__ void operator()() const { asm volatile("bar.sync %0, %1;" ::"r"(id), "n"(NT) : "memory"); }
};

template <int L, int A, int RM, class C = double2>
struct SwShape {
    static constexpr int R = L < RM ? L : RM;
    static constexpr int P = L / R;          // threads per line
    static constexpr int GT = A * P;         // threads per group
    static constexpr int NG = 2;             // groups per CTA
    static constexpr int THREADS = NG * GT;
    // row pitch in elements: bank-conflict free row <-> line-interleaved, and
    // every row start 16-B aligned for the bulk copies (float2: L + 2)
    static constexpr int PITCH = sizeof(C) == 16 ? L + 1 : L + 2;
    // tile buffers: 3 fit at fp64 (64 KB tiles); the fp32 mode's 33 KB tiles
    // allow 4, so each group's next tile is issued a whole tile-time ahead
    static constexpr int NBUF = sizeof(C) == 16 ? 3 : 4;
    static constexpr size_t BUF = (size_t)A * PITCH * sizeof(C);
    // the per-position tables a[f1], |e^{2 pi i f1/m} - 1|^2 stay in shared
    // memory unless the three buffers leave no room
    // (L = 1024: the fp32 mode's smaller buffers leave room for both tables; at fp64
    // the 8 KB Gamma row table still fits beside the three buffers, a[f1] does not)
    static constexpr bool TAB_SMEM = L <= 512 || sizeof(C) == 8;
    static constexpr bool NR_SMEM = TAB_SMEM || (L == 1024 && sizeof(C) == 16);
    static constexpr size_t TAB = (TAB_SMEM ? (size_t)L * sizeof(double2) : 0) + (NR_SMEM ? (size_t)L * sizeof(double) : 0);
    // per group: the tile's LR row of Y and of Gw (ml = L / dr entries, dr >= 2)
    static constexpr size_t ROWS = (size_t)(L / 2) * (sizeof(double2) + sizeof(double));
    static constexpr size_t META = (size_t)NBUF * A * 80;  // LineMeta per line of each buffer
    // the twiddle table too, where it fits (L <= 256; measured neutral at 512)
    static constexpr bool TW_SMEM = L <= 256;
    static constexpr size_t TWB = TW_SMEM ? (size_t)L * sizeof(C) : 0;
    static constexpr size_t STASH = (size_t)NG * A * 24;  // per group: each line's store rows (LineStore)
    static constexpr size_t SMEM = 64 + NBUF * BUF + META + TAB + TWB + NG * ROWS + NG * 32 * sizeof(double) + STASH;
    static_assert(SMEM <= 232448, "shared memory budget");
    static_assert(2 * NBUF * 8 <= 64, "mbarrier header");
};

// per-line placement of a tile's alias row (the half-spectrum mirror rules of
// fold_axis1_tile, T = 1) and its separable Lambda / Gamma factors.  Written
// by the warp that issues the tile's loads (the factors by cp.async, tracked
// by the buffer's mbarrier), read by the group that processes the tile.
struct __align__(16) LineMeta {
    double2 b;       // Lambda factor b[f2]
    double2 c;       // Lambda factor c[f3]
    double nc, ns;   // Gamma row terms |e^{2 pi i f2/n} - 1|^2, |e^{2 pi i f3/s} - 1|^2
    long long rd;    // row read (and, for mirrored lines of role 1, written conjugated)
    long long wr;    // direct store row; -1 for a mirrored line that is not stored
    long long sec;   // extra conjugated copy, -1 if none
    int mir;         // read as a conjugate mirror
    int pad;
};
static_assert(sizeof(LineMeta) == 80, "LineMeta layout");

// per-line placement of a tile's alias row (the half-spectrum mirror rules of
// fold_axis1_tile, T = 1)
struct LineInfo {
    long long rd;   // row read (and, for mirrored lines of role 1, written conjugated)
    long long wr;   // direct store row (valid when !mir)
    long long sec;  // extra conjugated copy, -1 if none
    bool mir;
};

__device__ __forceinline__ int tile_role(const FoldGeom& G, int bx2, int bx3) {
    const int mg2 = bx2 == 0 ? 0 : (int)G.nl - bx2, mg3 = bx3 == 0 ? 0 : (int)G.sl - bx3;
    if (mg2 == bx2 && mg3 == bx3) return 0;
    if (bx3 < mg3 || (bx3 == mg3 && bx2 < mg2)) return 1;
    return 2;
}

__device__ __forceinline__ LineInfo line_info(const FoldGeom& G, const int* __restrict__ wplane, int bx2, int bx3,
                                              int a, int role) {
    const int bc = a % G.dc, bs = a / G.dc;
    const long long f2 = bx2 + bc * G.nl, f3 = bx3 + bs * G.sl;
    auto wpl = [&](long long z) -> long long { return wplane ? (long long)__ldg(wplane + z) : z; };
    LineInfo li;
    li.mir = 2 * f3 > G.s;
    const long long nf2 = f2 == 0 ? 0 : G.n - f2;
    li.wr = li.mir ? 0 : G.m * (f2 + G.n * wpl(f3));
    li.rd = li.mir ? G.m * (nf2 + G.n * wpl(G.s - f3)) : li.wr;
    const long long mrow = G.m * (nf2 + G.n * wpl(f3));
    li.sec = (role == 1 && !li.mir && (f3 == 0 || 2 * f3 == G.s) && mrow != li.wr) ? mrow : -1;
    return li;
}

// a line's store rows, copied out of its LineMeta before the inverse
// transform (the issue after it re-arms the metadata) so they need not stay
// in registers across the transform
struct LineStore {
    long long wr, sec;
    int flip, pad;
};
static_assert(sizeof(LineStore) == 24, "LineStore layout");

__device__ __forceinline__ double2 lds_d2(unsigned a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ double lds_d(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

#ifndef VSR_RCP_FREE
#define VSR_RCP_FREE 4
#endif
constexpr int kRcpFree = VSR_RCP_FREE;

struct SwArgs {
    FoldGeom G;
    const double2* Yl;
    SepTables sep;
    const void* W;  // C rows (double2, or float2 in fp32 mode)
    void* out;
    GammaTables tabs;
    double cA, shift, inv_scale, invsqrtd, fwd_scale;
    const void* tw;  // C twiddles
    double* fit;
};

template <int NT, int NWARP>
__device__ __forceinline__ double group_sum(double v, double* red, int gt, int bar) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_down_sync(0xffffffffu, v, off);
    const int lane = gt & 31, warp = gt >> 5;
    if (lane == 0) red[warp] = v;
    asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(NT) : "memory");
    double t = 0.0;
    if (warp == 0) {
        t = lane < NWARP ? red[lane] : 0.0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) t += __shfl_down_sync(0xffffffffu, t, off);
    }
    return t;
}

// C = double2: the reference precision.  C = float2 (fp32 mode): rows and
// the axis-1 transforms in fp32, the fold in fp64 (see the fold below).
template <int L, int A, int DR, int RM, bool FIT, class C>
__global__ void __launch_bounds__(SwShape<L, A, RM, C>::THREADS, 1) tv_sandwich_pipe_kernel(SwArgs args) {
    using Sh = SwShape<L, A, RM, C>;
    using RT = typename CplxT<C>::real;
    using Pl = fftc::Plan<L, RM>;
    constexpr int R = Pl::R, P = Pl::P, GT = Sh::GT, NLN = A;
    constexpr int RD = R / DR;  // r = rr + RD * br: alias br of g1 = t + P rr
    constexpr int ML = L / DR;
    static_assert(R % DR == 0, "dr must divide the radix");
    static_assert(GT % 32 == 0, "a group is whole warps");
    static_assert(A <= 32, "one row per lane of the issuing warp");
    constexpr unsigned ROWB = (unsigned)(L * sizeof(C));
    const C* __restrict__ Wc = static_cast<const C*>(args.W);
    C* __restrict__ outc = static_cast<C*>(args.out);
    const FoldGeom& G = args.G;
    const GammaTables& tb = args.tabs;

    extern __shared__ __align__(128) unsigned char smraw[];
    // full[b]: buffer b's rows and line factors landed (tx count + cp.async arrivals);
    // issued[b]: buffer b's next load was armed (a parity wait is only sound
    // within one phase, and the consumer of tile k + 3 may get there before
    // tile k's rows have even landed)
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smraw);
    unsigned long long* issued = full + Sh::NBUF;  // 2 NBUF <= 8 mbarriers in the 64-byte header
    C* bufs = reinterpret_cast<C*>(smraw + 64);
    unsigned char* tail = smraw + 64 + Sh::NBUF * Sh::BUF;
    LineMeta* meta = reinterpret_cast<LineMeta*>(tail);
    tail += Sh::META;
    double2* sa_s = reinterpret_cast<double2*>(tail);
    double* nr_s = reinterpret_cast<double*>(sa_s + (Sh::TAB_SMEM ? L : 0));
    tail += Sh::TAB;
    C* tw_s = reinterpret_cast<C*>(tail);
    tail += Sh::TWB;
    double* red_s = reinterpret_cast<double*>(tail);
    tail += Sh::NG * 32 * sizeof(double);
    LineStore* stash = reinterpret_cast<LineStore*>(tail + Sh::NG * Sh::ROWS) + (threadIdx.x / Sh::GT) * A;
    // this group's LR rows of Y and Gw, by 32-bit shared address (a generic
    // pointer here costs two registers across the whole tile loop)
    const unsigned yrow_a = smem_u32(tail) + (threadIdx.x / Sh::GT) * (unsigned)Sh::ROWS;
    const unsigned gwrow_a = yrow_a + ML * (unsigned)sizeof(double2);
    const double2* __restrict__ sa_t = Sh::TAB_SMEM ? sa_s : args.sep.a;
    const double* __restrict__ nr_t = Sh::NR_SMEM ? nr_s : tb.nr;

    const int tid = threadIdx.x;
    const int g = tid / GT, gt = tid % GT;
    const int ln = gt % NLN, t = gt / NLN;
    const int ntiles = tb.ntiles;
    const int2* __restrict__ tiles = tb.tiles;

    // One warp arms buffer b for tile `tile`: lane j < A writes line j's
    // placement, cp.asyncs its factors (tracked by full[b]) and bulk-loads its
    // row; lane 0 sets the byte count, arrives, and marks the buffer issued.
    auto issue = [&](int tile, int b, int lane) {
        const int2 tt = __ldg(tiles + tile);
        const int role = tile_role(G, tt.x, tt.y);
        if (role != 2 && lane < A) {
            const int bc = lane % G.dc, bs = lane / G.dc;
            const long long f2 = tt.x + bc * G.nl, f3 = tt.y + bs * G.sl;
            const LineInfo li = line_info(G, tb.wplane, tt.x, tt.y, lane, role);
            LineMeta* mt = meta + b * A + lane;
            mt->rd = li.rd;
            mt->wr = !li.mir ? li.wr : (role == 1 ? li.rd : -1);
            mt->sec = li.sec;
            mt->mir = li.mir;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&mt->b)), "l"(args.sep.b + f2)
                         : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&mt->c)), "l"(args.sep.c + f3)
                         : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(&mt->nc)), "l"(tb.nc + f2)
                         : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(&mt->ns)), "l"(tb.ns + f3)
                         : "memory");
            // pending count + 1 now, - 1 when this lane's cp.asyncs complete
            asm volatile("cp.async.mbarrier.arrive.shared::cta.b64 [%0];" ::"r"(smem_u32(full + b)) : "memory");
        }
        __syncwarp();
        if (lane == 0)
            asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(full + b)),
                         "r"(role == 2 ? 0u : ROWB * A)
                         : "memory");
        __syncwarp();
        if (role != 2 && lane < A)
            bulk_g2s(bufs + ((size_t)b * A + lane) * Sh::PITCH, Wc + meta[b * A + lane].rd, ROWB, full + b);
        if (lane == 0) {
            mbar_arrive(full + b);
            mbar_arrive(issued + b);
        }
    };

    if (tid == 0) {
        for (int b = 0; b < Sh::NBUF; ++b) {
            mbar_init(full + b, 1);
            mbar_init(issued + b, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if constexpr (Sh::TAB_SMEM)
        for (int i = tid; i < L; i += Sh::THREADS) sa_s[i] = __ldg(args.sep.a + i);
    if constexpr (Sh::NR_SMEM)
        for (int i = tid; i < L; i += Sh::THREADS) nr_s[i] = __ldg(tb.nr + i);
    if constexpr (Sh::TW_SMEM)
        for (int i = tid; i < L; i += Sh::THREADS) tw_s[i] = __ldg(static_cast<const C*>(args.tw) + i);
    using TwT = std::conditional_t<Sh::TW_SMEM, fftc::TwShared<C>, const C*>;
    TwT twp;
    if constexpr (Sh::TW_SMEM)
        twp = fftc::TwShared<C>{tw_s};
    else
        twp = static_cast<const C*>(args.tw);
    __syncthreads();
    if (tid < 32)
        for (int k = 0; k < Sh::NBUF; ++k) {
            const int tile = blockIdx.x + k * gridDim.x;
            if (tile < ntiles) issue(tile, k, tid);
        }

    const GroupSync<GT> gsync{1 + g};
    auto sidx = [&](int q) { return q * NLN + ln; };
    double fit = 0.0;  // this thread's data-fit terms over all its tiles (fixed order)
    const double cAs = args.cA * args.fwd_scale;  // theta_hat enters only as mu * fwd_scale * FFT(...)

    // this group's tiles k = g, g + NG, ... (one loop-carried register)
    for (int k = (int)(threadIdx.x / GT);; k += Sh::NG) {
        const int tile = blockIdx.x + k * gridDim.x;
        if (tile >= ntiles) break;
        const int b = k % Sh::NBUF;
        C* sm = bufs + (size_t)b * A * Sh::PITCH;
        const LineMeta* mt = meta + b * A + ln;
        const int2 tt = __ldg(tiles + tile);
        const int role = tile_role(G, tt.x, tt.y);
        if (role != 2) {  // the tile's LR rows of Y and Gw -> this group's staging (cp.async)
            const long long lr = G.ml * (tt.x + G.nl * (long long)tt.y);
            for (int i = gt; i < ML; i += GT)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(yrow_a + 16u * i),
                             "l"(args.Yl + lr + i) : "memory");
            for (int i = gt; i < ML / 2; i += GT)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(gwrow_a + 16u * i),
                             "l"(tb.gw + lr + 2 * i) : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        mbar_wait(issued + b, (unsigned)((k / Sh::NBUF) & 1));
        mbar_wait(full + b, (unsigned)((k / Sh::NBUF) & 1));
        C v[R];
        double tfit = 0.0;
        if (role != 2) {
            const bool mir = mt->mir;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                v[r] = sm[ln * Sh::PITCH + t + P * r];
                if (mir) v[r].y = -v[r].y;
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
            gsync();  // rows read before the exchange overwrites the buffer; LR rows landed
            fftc::stockham<L, false, decltype(sidx), RM, GroupSync<GT>, TwT>(v, t, sm, sidx, twp, gsync);
            fftc::to_natural<L, RM>(v);
            // fold (reference form): S = sum_b Lambda_b g_b, g_b = Gamma_b k_b; w = S / (Gw + mu d);
            // x̂_b = (g_b - Gamma_b conj(Lambda_b) w) / mu; data fit from S and w.
            // fold_rr below evaluates it for one LR position group rr of this thread, in fp64.
            const double2 bc_ = cmul(mt->b, mt->c);
            const double base_g = mt->nc + mt->ns;
            // DR = 4: branch-free reciprocals interleave (115 vs 121 us at config 2).
            // DR = 2 (8 position groups per thread): the freer schedule spills
            // 200-750 B at the 128-register cap, so the branch stays as a fence.
            auto rcp_fold = [](double x) { return DR >= kRcpFree ? rcp_pos_normal(x) : rcp_pos(x); };
            // With t_b = Gamma_b Lambda_b and Gw = sum_b Gamma_b |Lambda_b|^2 (the gw
            // table), S = Gw y + mu' sum_b t_b theta_b, and
            //   x̂_b = (conj(t_b) (y - w) + Gamma_b mu' theta_b) / mu,
            //   y - w = (mu d y - mu' sum_b t_b theta_b) / (Gw + mu d):
            // the same map as g_b - Gamma_b conj(Lambda_b) w with 13 fewer fp64
            // operations per element, fewer values live across the alias sum, and
            // y - w formed without cancelling two O(Gw y) terms.
            const double gcs = cAs * args.inv_scale;
            auto fold_rr = [&](const int rr) {
                const double2 yraw = lds_d2(yrow_a + 16u * (t + P * rr));
                const double gwv = lds_d(gwrow_a + 8u * (t + P * rr));
                const double2 yv = cscale(yraw, args.invsqrtd);
                // (early: with the branching reciprocal it would otherwise sit behind the shuffles)
                const double us = rcp_fold(gwv + args.shift) * args.inv_scale;  // >= shift >= DBL_MIN (host check)
                double2 tb_[DR], pv[DR];  // t_b and Gamma_b mu' theta_b / mu (v[r] itself dies in the first loop)
                double Sx = 0, Sy = 0;
#pragma unroll
                for (int br = 0; br < DR; ++br) {
                    const int r = rr + RD * br;
                    const int q = t + P * r;
                    const double2 Lr = cmul(sa_t[q], bc_);
                    const double gg = rcp_fold((nr_t[q] + base_g) + tb.tau);  // >= tau >= DBL_MIN (host check)
                    tb_[br] = cscale(Lr, gg);
                    const double2 vr = to_d2(v[r]);
                    pv[br] = cscale(vr, gg * gcs);
                    Sx = fma(tb_[br].x, vr.x, Sx);
                    Sx = fma(-tb_[br].y, vr.y, Sx);
                    Sy = fma(tb_[br].x, vr.y, Sy);
                    Sy = fma(tb_[br].y, vr.x, Sy);
                }
#pragma unroll
                for (int o = 1; o < A; o <<= 1) {
                    Sx += __shfl_xor_sync(0xffffffffu, Sx, o);
                    Sy += __shfl_xor_sync(0xffffffffu, Sy, o);
                }
                // (y - w) / mu
                const double2 u = cmake<double2>(fma(args.shift, yv.x, -cAs * Sx) * us, fma(args.shift, yv.y, -cAs * Sy) * us);
#pragma unroll
                for (int br = 0; br < DR; ++br) {
                    const int r = rr + RD * br;
                    double ox = fma(tb_[br].x, u.x, pv[br].x), oy = fma(tb_[br].x, u.y, pv[br].y);
                    ox = fma(tb_[br].y, u.y, ox);
                    oy = fma(-tb_[br].y, u.x, oy);
                    v[r] = from_d2<C>(cmake<double2>(ox, oy));
                }
                if constexpr (FIT) {
                    if (ln == 0) {
                        // A x̂ folded: (S - Gw w) / mu with S = Gw y + mu' sum, w = S / (Gw + mu d)
                        const double Stx = fma(gwv, yv.x, cAs * Sx), Sty = fma(gwv, yv.y, cAs * Sy);
                        const double ax = Stx * args.inv_scale - gwv * (Stx * us),
                                     ay = Sty * args.inv_scale - gwv * (Sty * us);
                        const double rx = yraw.x - args.invsqrtd * ax, ry = yraw.y - args.invsqrtd * ay;
                        tfit += rx * rx + ry * ry;
                    }
                }
            };
            // fp32 mode too folds in fp64: the Woodbury form cancels at low
            // frequencies and amplifies rounding by ~Gamma_b |Lambda_b|^2 / (mu d)
            // -- 1/tau at DC, hundreds at the lowest non-zero frequencies -- while
            // the map itself is well conditioned in its inputs (fp32 spectra are fine)
#pragma unroll
            for (int rr = 0; rr < RD; ++rr) fold_rr(rr);
            // this line's store rows, read before the inverse transform's barriers
            // (after them, the issue below re-arms buffer b's metadata)
            if (t == 0) stash[ln] = LineStore{mt->wr, mt->sec, mir ? (int)0x80000000 : 0, 0};
            fftc::stockham<L, true, decltype(sidx), RM, GroupSync<GT>, TwT>(v, t, sm, sidx, twp, gsync);
        } else {
            gsync();  // every thread of the group has seen this phase before it is re-armed
        }
        // the buffer is free (the last exchange ended with a group barrier):
        // hand it to the bulk engine for the tile three ahead
        if (gt < 32) {
            const int nt = blockIdx.x + (k + Sh::NBUF) * gridDim.x;
            if (nt < ntiles) issue(nt, b, gt);
        }
        if (role != 2) {
            // direct rows as computed; mirrored rows (role 1) conjugated into their mirror position
            const long long wr = stash[ln].wr, sec = stash[ln].sec;
            const int flip = stash[ln].flip;
            if (wr >= 0) {
                C* dst = outc + wr;
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const C val = v[j];
                    RT y;
                    if constexpr (std::is_same<C, double2>::value)
                        y = __hiloint2double(__double2hiint(val.y) ^ flip, __double2loint(val.y));
                    else
                        y = __int_as_float(__float_as_int(val.y) ^ flip);
                    dst[Pl::out_q(t, j)] = cmake<C>(val.x, y);
                }
            }
            if (sec >= 0) {  // planes 0 and s/2 only
                C* dst = outc + sec;
#pragma unroll
                for (int j = 0; j < R; ++j) dst[Pl::out_q(t, j)] = cmake<C>(v[j].x, -v[j].y);
            }
            if constexpr (FIT) fit += role == 1 ? 2.0 * tfit : tfit;  // the skipped mirror set: same |residual|^2
        }
    }
    if constexpr (FIT) {
        // one partial per (CTA, group); slots past 2 * grid (fewer CTAs than
        // tiles) are zero so the fixed-order finalize can read ntiles of them
        const double tot = group_sum<GT, GT / 32>(fit, red_s + 32 * g, gt, 1 + g);
        const int slot = 2 * blockIdx.x + g;
        if (gt == 0 && slot < ntiles) args.fit[slot] = tot;
        for (int i = 2 * gridDim.x + blockIdx.x + tid * gridDim.x; i < ntiles; i += Sh::THREADS * gridDim.x)
            args.fit[i] = 0.0;
    }
}

int sm_count() {
    static int n = [] {
        int dev = 0, v = 0;
        VSR_CUDA(cudaGetDevice(&dev));
        VSR_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
        return v;
    }();
    return n;
}

template <int L, int A, int DR, int RM, class C>
void launch_pipe(const SwArgs& a, cudaStream_t st) {
    using Sh = SwShape<L, A, RM, C>;
    auto kern = a.fit ? tv_sandwich_pipe_kernel<L, A, DR, RM, true, C> : tv_sandwich_pipe_kernel<L, A, DR, RM, false, C>;
    VSR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sh::SMEM));
    // two groups per CTA: at most ntiles / 2 CTAs, so every (CTA, group) partial slot is < ntiles
    const int grid = std::max(1, std::min(a.tabs.ntiles / 2, sm_count()));
    kern<<<grid, Sh::THREADS, Sh::SMEM, st>>>(a);
    VSR_LAUNCH_CHECK();
}

// (L = m, A = dc*ds, DR = dr): the TV geometries of the BASELINE configs
// (first three) and their neighbours; a group is A * L / 16 threads, whole
// warps, at most 256
#define VSR_PIPE_TABLE(X)                                                          \
    X(256, 16, 4) X(512, 8, 2) X(1024, 4, 2) X(64, 16, 4) X(128, 16, 4)               \
    X(64, 8, 2) X(128, 8, 2) X(256, 8, 2) X(128, 4, 2) X(256, 4, 2) X(512, 4, 2)

template <class C>
bool sandwich_pipe_t(const FoldGeom& G, const double2* Yl, const SepTables& sep, const void* W, void* out,
                            const GammaTables& tabs, double cA, double shift, double inv_scale, double fwd_scale,
                            double* fit_partials, cudaStream_t st) {
    if (!sep.a || !tabs.gw || !tabs.half3 || tabs.fit_only || !tabs.tiles || tabs.ntiles <= 0 || !out || out == W)
        return false;
    if (tv_sandwich1_tile_g2(G) != 1) return false;
    // the fold's reciprocals skip the subnormal-denominator branch: both
    // denominators are bounded below by these two (Gamma's tau, mu d)
    if (!(tabs.tau >= 2.2250738585072014e-308) || !(shift >= 2.2250738585072014e-308)) return false;
    const int A = G.dc * G.ds;
    SwArgs a{G, Yl, sep, W, out, tabs, cA, shift, inv_scale, 1.0 / std::sqrt((double)G.d), fwd_scale,
             nullptr, fit_partials};
#define VSR_X(LL, AA, DD)                                                      \
    if (G.m == LL && A == AA && G.dr == DD) {                                  \
        if constexpr (std::is_same<C, double2>::value)                         \
            a.tw = fft_engine().twiddles((size_t)LL);                          \
        else                                                                   \
            a.tw = fft_engine().twiddles_f((size_t)LL);                        \
        launch_pipe<LL, AA, DD, 16, C>(a, st);                                 \
        return true;                                                           \
    }
    VSR_PIPE_TABLE(VSR_X)
#undef VSR_X
    return false;
}

}  // namespace

bool tv_sandwich_pipe_ok(const FoldGeom& G) {
    if (tv_sandwich1_tile_g2(G) != 1) return false;
    const int A = G.dc * G.ds;
#define VSR_X(LL, AA, DD) \
    if (G.m == LL && A == AA && G.dr == DD) return true;
    VSR_PIPE_TABLE(VSR_X)
#undef VSR_X
    return false;
}

bool tv_sandwich_pipe(const FoldGeom& G, const double2* Yl, const SepTables& sep, const double2* W, double2* out,
                      const GammaTables& tabs, double cA, double shift, double inv_scale, double fwd_scale,
                      double* fit_partials, cudaStream_t st) {
    return sandwich_pipe_t<double2>(G, Yl, sep, W, out, tabs, cA, shift, inv_scale, fwd_scale, fit_partials, st);
}

bool tv_sandwich_pipe_f32(const FoldGeom& G, const double2* Yl, const SepTables& sep, const float2* W, float2* out,
                          const GammaTables& tabs, double cA, double shift, double inv_scale, double fwd_scale,
                          double* fit_partials, cudaStream_t st) {
    return sandwich_pipe_t<float2>(G, Yl, sep, W, out, tabs, cA, shift, inv_scale, fwd_scale, fit_partials, st);
}

std::vector<int2> tv_sandwich1_active_tiles(const FoldGeom& G) {
    // half spectrum, one LR (g2, g3) per tile: the sets whose mirror is not run
    // elsewhere (role 0 or 1 of fold_axis1_tile), g3-major
    std::vector<int2> v;
    for (long long g3 = 0; g3 < G.sl; ++g3)
        for (long long g2 = 0; g2 < G.nl; ++g2) {
            const long long mg2 = g2 == 0 ? 0 : G.nl - g2, mg3 = g3 == 0 ? 0 : G.sl - g3;
            const bool self = mg2 == g2 && mg3 == g3;
            if (self || g3 < mg3 || (g3 == mg3 && g2 < mg2)) v.push_back(make_int2((int)g2, (int)g3));
        }
    return v;
}

}  // namespace vsr
