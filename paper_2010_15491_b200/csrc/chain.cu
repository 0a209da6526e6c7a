// Chained in-plane FFT passes through an L2-resident ring (see chain.cuh).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "chain.cuh"
#include "fft_core.cuh"

namespace vsr {
namespace {

template <int LM, int LN>
struct CShape {
    using P1 = fftc::Plan<LM>;  // axis 1: contiguous rows of length LM
    using P2 = fftc::Plan<LN>;  // axis 2: strided columns of length LN
    static constexpr int T2 = 8;
    static constexpr int TH0 = T2 * P2::P > 128 ? T2 * P2::P : 128;
    static constexpr int TH = TH0 > P1::P ? TH0 : P1::P;
    static constexpr int TG2 = TH / (T2 * P2::P);  // column groups per strided tile
    static constexpr int COLS = TG2 * T2;          // columns per strided tile
    static constexpr int NX = TH / P1::P;          // rows per contiguous tile
    static constexpr int LPAD1 = LM + LM / P1::R;
    static constexpr int S1 = P1::NEEDS_SMEM ? NX * LPAD1 : 0;
    static constexpr int S2 = P2::NEEDS_SMEM ? TG2 * T2 * LN : 0;
    static constexpr int SMEM = S1 > S2 ? S1 : S2;  // double2 elements
};

__device__ __forceinline__ void wait_count(int* p, int target) {
    if (threadIdx.x == 0) {
        while (atomicAdd(p, 0) < target) __nanosleep(128);
        __threadfence();
    }
    __syncthreads();
}

// Barrier, then one thread publishes with a gpu-scope fence + atomic (the
// grid-sync pattern: bar.sync orders the CTA's stores before thread 0's fence).
__device__ __forceinline__ void signal_done(int* p) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(p, 1);
    }
}

// axis-2 tile: columns [i0, i0 + COLS) of one plane.  src/dst point at the plane.
template <int LM, int LN, bool INV, bool SRC_RING>
__device__ __forceinline__ void strided_tile(const double2* src, double2* dst, int i0, double2* sm,
                                             const double2* __restrict__ tw) {
    using Sh = CShape<LM, LN>;
    constexpr int P = Sh::P2::P, R = Sh::P2::R, T2 = Sh::T2;
    const int tid = threadIdx.x;
    const int g = tid / (T2 * P), rem = tid % (T2 * P), lt = rem % T2, t = rem / T2;
    const int i = i0 + g * T2 + lt;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const double2* a = src + i + (long long)LM * (t + P * r);
        v[r] = SRC_RING ? __ldcg(a) : *a;
    }
    fftc::stockham<LN, INV>(v, t, sm, [&](int q) { return g * (T2 * LN) + q * T2 + lt; }, tw);
#pragma unroll
    for (int j = 0; j < R; ++j) dst[i + (long long)LM * Sh::P2::out_q(t, j)] = v[j];
}

// axis-1 tile: rows [j0, j0 + NX) of one plane.
template <int LM, int LN, bool INV, bool REAL_IN, bool REAL_OUT>
__device__ __forceinline__ void contig_tile(const void* src, void* dst, int j0, double2* sm,
                                            const double2* __restrict__ tw, double scale,
                                            long long dst_plane_base, double& acc_im,
                                            double& acc_tot, unsigned long long* bad) {
    using Sh = CShape<LM, LN>;
    constexpr int P = Sh::P1::P, R = Sh::P1::R;
    const int tid = threadIdx.x;
    const int line = tid / P, t = tid % P;
    const long long row = (long long)LM * (j0 + line);
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int q = t + P * r;
        if constexpr (REAL_IN)
            v[r] = make_double2(reinterpret_cast<const double*>(src)[row + q], 0.0);
        else
            v[r] = __ldcg(reinterpret_cast<const double2*>(src) + row + q);
    }
    fftc::stockham<LM, INV>(v, t, sm, [&](int q) { return line * Sh::LPAD1 + q + q / R; }, tw);
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const long long o = row + Sh::P1::out_q(t, j);
        if constexpr (REAL_OUT) {
            const double2 z = cscale(v[j], scale);
            acc_im += z.y * z.y;
            acc_tot += z.x * z.x + z.y * z.y;
            reinterpret_cast<double*>(dst)[o] = z.x;
            if (!isfinite(z.x)) atomicMin(bad, (unsigned long long)(dst_plane_base + o));
        } else {
            reinterpret_cast<double2*>(dst)[o] = v[j];
        }
    }
}

template <int LM, int LN, bool FWD>
__global__ void __launch_bounds__(CShape<LM, LN>::TH, 640 / CShape<LM, LN>::TH)
    chain_kernel(int G, int C, int RING, int LA, const void* in, void* out, double2* ring, int* ctr,
                 const double2* __restrict__ tw1, const double2* __restrict__ tw2, double scale,
                 double* __restrict__ partials, unsigned long long* __restrict__ bad) {
    using Sh = CShape<LM, LN>;
    extern __shared__ double2 sm[];
    __shared__ double red[64];
    constexpr long long PL = (long long)LM * LN;
    const int sPer = LM / Sh::COLS, cPer = LN / Sh::NX;  // tiles per plane
    // A = first pass, B = second pass
    const int nA = (FWD ? cPer : sPer) * G, nB = (FWD ? sPer : cPer) * G;
    const long long total = (long long)C * (nA + nB);
    int* doneA = ctr + 1;
    int* doneB = ctr + 1 + C;
    // queue order: A(0..LA-1), then pairs [B(c), A(c+LA)] for c < C-LA, then B(C-LA..C-1)
    const long long headA = (long long)LA * nA;
    const long long pairs = (long long)(C - LA) * (nA + nB);
    __shared__ int item_sh;
    for (;;) {
        if (threadIdx.x == 0) item_sh = atomicAdd(ctr, 1);
        __syncthreads();
        const long long item = item_sh;
        __syncthreads();
        if (item >= total) break;
        bool isA;
        int c, tile;
        if (item < headA) {
            isA = true, c = (int)(item / nA), tile = (int)(item % nA);
        } else if (item < headA + pairs) {
            const long long j = item - headA;
            const int p = (int)(j / (nA + nB)), r = (int)(j % (nA + nB));
            if (r < nB)
                isA = false, c = p, tile = r;
            else
                isA = true, c = p + LA, tile = r - nB;
        } else {
            const long long j = item - headA - pairs;
            isA = false, c = C - LA + (int)(j / nB), tile = (int)(j % nB);
        }
        double2* slot = ring + (long long)(c % RING) * G * PL;
        if (isA) {
            if (c >= RING) wait_count(doneB + (c - RING), nB);
            if constexpr (!FWD) {  // axis-2 inverse: W -> ring
                const int zl = tile / sPer, cb = tile % sPer;
                const double2* src = reinterpret_cast<const double2*>(in) + (long long)(c * G + zl) * PL;
                strided_tile<LM, LN, true, false>(src, slot + zl * PL, cb * Sh::COLS, sm, tw2);
            } else {  // axis-1 r2c: theta -> ring
                const int zl = tile / cPer, rb = tile % cPer;
                const double* src = reinterpret_cast<const double*>(in) + (long long)(c * G + zl) * PL;
                double a0 = 0, a1 = 0;
                contig_tile<LM, LN, false, true, false>(src, slot + zl * PL, rb * Sh::NX, sm, tw1, 1.0, 0,
                                                        a0, a1, nullptr);
            }
            signal_done(doneA + c);
        } else {
            wait_count(doneA + c, nA);
            if constexpr (!FWD) {  // axis-1 inverse c2r: ring -> x
                const int zl = tile / cPer, rb = tile % cPer;
                const long long pb = (long long)(c * G + zl) * PL;
                double acc_im = 0.0, acc_tot = 0.0;
                contig_tile<LM, LN, true, false, true>(slot + zl * PL, reinterpret_cast<double*>(out) + pb,
                                                       rb * Sh::NX, sm, tw1, scale, pb, acc_im, acc_tot, bad);
                double vals[2] = {acc_im, acc_tot};
                block_reduce_sum<2>(vals, red);
                if (threadIdx.x == 0) {
                    const long long b = (long long)c * nB + tile;
                    partials[2 * b] = vals[0];
                    partials[2 * b + 1] = vals[1];
                }
            } else {  // axis-2 forward: ring -> W
                const int zl = tile / sPer, cb = tile % sPer;
                double2* dst = reinterpret_cast<double2*>(out) + (long long)(c * G + zl) * PL;
                strided_tile<LM, LN, false, true>(slot + zl * PL, dst, cb * Sh::COLS, sm, tw2);
            }
            signal_done(doneB + c);
        }
    }
}

template <int LM, int LN>
bool tiles_fit() {
    using Sh = CShape<LM, LN>;
    return LM % Sh::COLS == 0 && LN % Sh::NX == 0;
}

struct Sizes {
    int th, smem, sper, cper;
};

template <int LM, int LN>
Sizes sizes() {
    using Sh = CShape<LM, LN>;
    return {Sh::TH, Sh::SMEM * (int)sizeof(double2), LM / Sh::COLS, LN / Sh::NX};
}

bool sizes_for(const Dims& d, Sizes& out) {
    if (d.m != d.n) return false;
    switch (d.m) {
#define VSR_C(L)                          \
    case L:                               \
        if (!tiles_fit<L, L>()) return false; \
        out = sizes<L, L>();              \
        return true;
        VSR_C(32)
        VSR_C(64)
        VSR_C(128)
        VSR_C(256)
        VSR_C(512)
        VSR_C(1024)
#undef VSR_C
        default:
            return false;
    }
}

template <bool FWD>
void launch(const Dims& d, const ChainPlan& p, const ChainWork& w, const void* in, void* out,
            double scale, double* partials, unsigned long long* bad, cudaStream_t st) {
    const double2* tw = fft_engine().twiddles(d.m);
    VSR_CUDA(cudaMemsetAsync(w.counters, 0, sizeof(int) * (1 + 2 * p.chunks), st));
    switch (d.m) {
#define VSR_C(L)                                                                                   \
    case L: {                                                                                      \
        auto k = chain_kernel<L, L, FWD>;                                                          \
        const int smem = CShape<L, L>::SMEM * (int)sizeof(double2);                                \
        if (smem > 48 * 1024)                                                                      \
            VSR_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
        k<<<(unsigned)p.blocks, CShape<L, L>::TH, smem, st>>>(p.g, p.chunks, p.ring, p.lookahead, in,   \
                                                             out, w.ring, \
                                                             w.counters, tw, tw, scale, partials,  \
                                                             bad);                                 \
        break;                                                                                     \
    }
        VSR_C(32)
        VSR_C(64)
        VSR_C(128)
        VSR_C(256)
        VSR_C(512)
        VSR_C(1024)
#undef VSR_C
        default:
            throw std::logic_error("chain: unsupported plane size");
    }
    VSR_LAUNCH_CHECK();
}

template <int L>
int occupancy(bool fwd) {
    int nb = 0;
    const int smem = CShape<L, L>::SMEM * (int)sizeof(double2);
    if (fwd) {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(chain_kernel<L, L, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, chain_kernel<L, L, true>, CShape<L, L>::TH, smem);
    } else {
        if (smem > 48 * 1024)
            cudaFuncSetAttribute(chain_kernel<L, L, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, chain_kernel<L, L, false>, CShape<L, L>::TH, smem);
    }
    return std::max(nb, 1);
}

}  // namespace

ChainPlan chain_plan(const Dims& d) {
    ChainPlan p;
    Sizes sz;
    if (!sizes_for(d, sz) || d.s < 2) return p;
    const size_t plane_bytes = d.m * d.n * sizeof(double2);
    // chunk ~4 MB of planes (G divides s), ring of 3 chunks
    size_t g = std::max<size_t>(1, (1u << 20) / plane_bytes);
    while (g > 1 && d.s % g) --g;
    p.g = (int)g;
    p.chunks = (int)(d.s / g);
    p.a_tiles = (size_t)sz.sper * g;  // per chunk (inverse: strided first)
    p.b_tiles = (size_t)sz.cper * g;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int occ = 1;
    switch (d.m) {
        case 32: occ = occupancy<32>(false); break;
        case 64: occ = occupancy<64>(false); break;
        case 128: occ = occupancy<128>(false); break;
        case 256: occ = occupancy<256>(false); break;
        case 512: occ = occupancy<512>(false); break;
        case 1024: occ = occupancy<1024>(false); break;
    }
    p.blocks = (size_t)sms * occ;
    // lookahead: A tiles run ~2 resident waves ahead of the B tiles that consume them
    double mult = 1.5;
    if (const char* e = std::getenv("VSR_CHAIN_LA")) mult = std::atof(e);
    const size_t la = (size_t)std::ceil(mult * (double)p.blocks / (double)p.a_tiles);
    p.lookahead = (int)std::min<size_t>(std::max<size_t>(la, 1), (size_t)p.chunks);
    p.ring = std::min(p.lookahead + 1, p.chunks);
    p.scratch_elems = (size_t)p.ring * g * d.m * d.n;
    p.ok = true;
    return p;
}

void launch_chain_inverse(const Dims& d, const ChainPlan& p, const ChainWork& w, const double2* W,
                          double* out, double scale, const PassReduce& red, cudaStream_t st) {
    launch<false>(d, p, w, W, out, scale, red.partials, red.bad_index, st);
}

void launch_chain_forward(const Dims& d, const ChainPlan& p, const ChainWork& w, const double* theta,
                          double2* W, cudaStream_t st) {
    launch<true>(d, p, w, theta, W, 1.0, nullptr, nullptr, st);
}

}  // namespace vsr
