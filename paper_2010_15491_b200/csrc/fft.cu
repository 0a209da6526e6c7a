// fp64 3D FFT engine, sm_100a.  See fft.cuh for the design summary.
//
// Reference semantics reproduced (proj/src/fft.cpp):
//   * forward = sign -1 (FFTW_FORWARD), inverse = sign +1 (:57,67,76);
//   * axis 1 (m) is the fastest-varying (FFTW's last dimension, :32-38);
//   * unitary scaling 1/sqrt(N) applied after the transform (:68-69,77-78);
//   * ifft3_real reduces sum(imag^2) and sum(|z|^2) for the residue check (:84-93).
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <type_traits>

#include "fft.cuh"
#include "fft_core.cuh"

namespace vsr {
namespace {

using fftc::ilog2;

// ------------------------------------------------------------ pass kernel
// Kernel shape: a CTA owns NL = TG * T lines of length L.  Each line is served
// by P = L / R threads, each holding R elements in registers.
//   CONTIG = true : axis 1; lines are contiguous, lanes run along a line.
//   CONTIG = false: strided axis; a tile is T consecutive inner indices, lanes
//                   run across the tile so HBM rows are T * 16 B.
// Stockham stages: k = log_R(L) radix-R stages, then an optional final radix
// RL < R stage (each thread then does R / RL butterflies).
template <int L, int R, int T, int TG, bool CONTIG>
struct PassShape {
    static constexpr int P = L / R;
    static constexpr int NL = TG * T;
    static constexpr int THREADS = NL * P;
    static constexpr int LOGL = ilog2(L), LOGR = ilog2(R);
    static constexpr int K = LOGL / LOGR;                // full radix-R stages
    static constexpr int RL = 1 << (LOGL - K * LOGR);   // final small radix (1 = none)
    static constexpr int NSTAGE = K + (RL > 1 ? 1 : 0);
    static constexpr int LPAD = CONTIG ? (L + L / R) : L;  // smem line pitch (contig)
    static constexpr int SMEM_ELEMS = NSTAGE > 1 ? NL * LPAD : 0;
    __device__ static __forceinline__ int sidx(int ls, int q) {
        if constexpr (CONTIG)
            return ls * LPAD + q + q / R;
        else
            return (ls / T) * (L * T) + q * T + (ls % T);
    }
};

template <int L, int R, int T, int TG, bool CONTIG, bool INV, int IK, int OK, class C = double2>
__global__ void __launch_bounds__(PassShape<L, R, T, TG, CONTIG>::THREADS)
    fft_pass_kernel(const void* in_, void* out_, long long S,
                    long long nlines_or_tiles, const C* __restrict__ tw, double scale,
                    double* __restrict__ partials, unsigned long long* __restrict__ bad_index) {
    using Sh = PassShape<L, R, T, TG, CONTIG>;
    using RT = typename CplxT<C>::real;
    constexpr int P = Sh::P;
    extern __shared__ double2 sm_raw[];
    C* sm = reinterpret_cast<C*>(sm_raw);

    const int tid = threadIdx.x;
    int ls, t;  // line slot in CTA, thread index within its line
    long long base;
    long long estride;
    bool active;
    if constexpr (CONTIG) {
        ls = tid / P;
        t = tid % P;
        const long long line = (long long)blockIdx.x * Sh::NL + ls;
        active = line < nlines_or_tiles;
        base = line * L;
        estride = 1;
    } else {
        const int g = tid / (T * P);
        const int rem = tid % (T * P);
        const int lt = rem % T;
        t = rem / T;
        ls = g * T + lt;
        const long long tile = (long long)blockIdx.x * TG + g;
        active = tile < nlines_or_tiles;
        const long long tiles_per_o = S / T;
        const long long o = active ? tile / tiles_per_o : 0;
        const long long p0 = active ? (tile % tiles_per_o) * T : 0;
        base = p0 + lt + S * (long long)L * o;
        estride = S;
    }

    C v[R];
    // ---- load: first stage (radix R, Ns = 1) reads q = t + P * r
    if (active) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const long long off = base + estride * (long long)(t + P * r);
            if constexpr (IK == IN_REAL) {
                v[r] = cmake<C>(reinterpret_cast<const RT*>(in_)[off], (RT)0);
            } else if constexpr (IK == IN_HALF) {
                const int q = t + P * r;
                if (q <= L / 2) {
                    v[r] = reinterpret_cast<const C*>(in_)[off];
                } else {
                    const C h = reinterpret_cast<const C*>(in_)[base + estride * (long long)(L - q)];
                    v[r] = cmake<C>(h.x, -h.y);
                }
            } else {
                v[r] = reinterpret_cast<const C*>(in_)[off];
            }
        }
    } else {
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = cmake<C>((RT)0, (RT)0);
    }

    fftc::stockham<L, INV>(v, t, sm, [&](int q) { return Sh::sidx(ls, q); }, tw);

    // ---- store (output order: slot j holds line position Plan<L>::out_q(t, j))
    double acc_im = 0.0, acc_tot = 0.0;
    if (active) {
#pragma unroll
        for (int j = 0; j < R; ++j) {
            const int q = fftc::Plan<L>::out_q(t, j);
            const long long off = base + estride * (long long)q;
            const C z = cscale(v[j], (RT)scale);
            if constexpr (OK == OUT_REAL) {
                acc_im += (double)z.y * z.y;
                acc_tot += (double)z.x * z.x + (double)z.y * z.y;
                reinterpret_cast<RT*>(out_)[off] = z.x;
                if (!isfinite(z.x)) atomicMin(bad_index, (unsigned long long)off);
            } else if constexpr (OK == OUT_HALF) {
                if (q <= L / 2) reinterpret_cast<C*>(out_)[off] = z;
            } else {
                reinterpret_cast<C*>(out_)[off] = z;
            }
        }
    }
    if constexpr (OK == OUT_REAL) {
        __shared__ double red[64];
        double vals[2] = {acc_im, acc_tot};
        block_reduce_sum<2>(vals, red);
        if (tid == 0) {
            partials[2 * blockIdx.x] = vals[0];
            partials[2 * blockIdx.x + 1] = vals[1];
        }
    }
}

// ------------------------------------------------- paired real lines (axis 3)
// Two adjacent real columns (c, c + 1) of a strided axis form one complex line
// z = x_c + i x_{c+1}: one complex FFT serves both (a double2 load is the pair).
//   forward: X_c[k] = (Z[k] + conj Z[L-k]) / 2, X_{c+1}[k] = (Z[k] - conj Z[L-k]) / 2i,
//            stored for k <= L/2 (Hermitian half spectrum along the axis)
//   inverse: Z[k] = X_c[k] + i X_{c+1}[k] (k > L/2 from conj X[L-k]); the real and
//            imaginary parts of IDFT(Z) are the two real columns.
// A CTA owns one tile of T = 8 columns (4 pairs), full lines.
// real columns per tile of the paired passes, every L (1024: 128 KB of smem,
// one CTA per SM); half3_blocks() sizes the residue partials from it too
constexpr int kRPairCols = 16;

template <int L>
struct RPairShape {
    using Pl = fftc::Plan<L>;
    // 16 real columns per tile: 128-byte row segments in the real domain
    static constexpr int R = Pl::R, P = Pl::P, T = kRPairCols, TP = T / 2;
    static constexpr int TG = (TP * P) >= 128 ? 1 : 128 / (TP * P);  // tiles per CTA
    static constexpr int THREADS = TG * TP * P;
    // per tile: the exchange (TP lines of L) or, in the inverse, the staged
    // half-spectrum planes 0..L/2 (2 complex per pair each)
    static constexpr int GREG = TP * (L + 2);
    static constexpr int SMEM = TG * GREG;
};

template <int L, class C = double2>
__global__ void __launch_bounds__(RPairShape<L>::THREADS)
    rpair_fwd_kernel(const typename CplxT<C>::real* __restrict__ in, C* __restrict__ out, long long S,
                     long long tiles, const C* __restrict__ tw, RemotePlanes rp) {
    using Sh = RPairShape<L>;
    using RT = typename CplxT<C>::real;
    constexpr int R = Sh::R, P = Sh::P, T = Sh::T, TP = Sh::TP;
    extern __shared__ double2 sm_raw[];
    C* sm = reinterpret_cast<C*>(sm_raw);
    const int tid = threadIdx.x, g = tid / (TP * P), rem = tid % (TP * P), lp = rem % TP, t = rem / TP;
    const long long tile = (long long)blockIdx.x * Sh::TG + g;
    const bool active = tile < tiles;
    const long long tpo = S / T, o = active ? tile / tpo : 0, c = active ? (tile % tpo) * T + 2 * lp : 0;
    auto sidx = [&](int q) { return g * Sh::GREG + q * TP + lp; };
    const C* src = reinterpret_cast<const C*>(in + c + S * (long long)L * o);
    const long long S2 = S / 2;
    C v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = active ? __ldg(src + S2 * (t + P * r)) : cmake<C>((RT)0, (RT)0);
    fftc::stockham<L, false>(v, t, sm, sidx, tw);  // (its last exchange ends with a barrier)
    // Hermitian split: position k <= L/2 needs Z[k], which this thread holds,
    // and Z[L - k], a position above L/2 (or k itself at k = 0, L/2): only the
    // upper half goes through shared memory
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int q = fftc::Plan<L>::out_q(t, j);
        if (q > L / 2) sm[sidx(q)] = v[j];
    }
    __syncthreads();
    C* dst = out + c + S * (long long)(L / 2 + 1) * o;
    const RT half = (RT)0.5;
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int k = fftc::Plan<L>::out_q(t, j);
        if (k > L / 2 || !active) continue;
        const C a = v[j];
        const C b = (k == 0 || k == L / 2) ? a : sm[sidx(L - k)];
        const C xa = cmake<C>(half * (a.x + b.x), half * (a.y - b.y));
        const C xb = cmake<C>(half * (a.y + b.y), -half * (a.x - b.x));
        // slab-sharded: plane k goes straight to its owner's spectral buffer
        // (peer memory over NVLink), rows of this rank's y range (fp64 only)
        C* d = dst + S * k;
        if constexpr (std::is_same<C, double2>::value)
            if (rp.peer) d = rp.peer[rp.owner[k]] + rp.off[k] + c;
        d[0] = xa;
        d[1] = xb;
    }
    if (rp.peer) __threadfence_system();
}

template <int L, class C = double2>
__global__ void __launch_bounds__(RPairShape<L>::THREADS)
    rpair_inv_kernel(const C* __restrict__ in, typename CplxT<C>::real* __restrict__ out, long long S,
                     long long tiles, const C* __restrict__ tw, double scale, double* __restrict__ partials,
                     unsigned long long* __restrict__ bad_index, RemotePlanes rp) {
    using Sh = RPairShape<L>;
    using RT = typename CplxT<C>::real;
    constexpr int R = Sh::R, P = Sh::P, T = Sh::T, TP = Sh::TP;
    extern __shared__ double2 sm_raw[];
    C* sm = reinterpret_cast<C*>(sm_raw);
    const int tid = threadIdx.x, g = tid / (TP * P), rem = tid % (TP * P), lp = rem % TP, t = rem / TP;
    const long long tile = (long long)blockIdx.x * Sh::TG + g;
    const bool active = tile < tiles;
    const long long tpo = S / T, o = active ? tile / tpo : 0, c = active ? (tile % tpo) * T + 2 * lp : 0;
    auto sidx = [&](int q) { return g * Sh::GREG + q * TP + lp; };
    const C* src = in + c + S * (long long)(L / 2 + 1) * o;
    // each half-spectrum plane q <= L/2 is loaded ONCE (by the thread holding
    // position q), which also stages the combined value its conjugate mirror
    // position L - q needs; positions q > L/2 read that back from shared memory
    // (fp64; the fp32 mode keeps the direct mirror loads, measured faster there)
    C* stg = sm + g * Sh::GREG;
    C v[R];
    if constexpr (!std::is_same<C, double2>::value) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int q = t + P * r;
            const bool lo = q <= L / 2;
            const C* p = src + S * (lo ? q : L - q);
            C A = active ? __ldg(p) : cmake<C>((RT)0, (RT)0), B = active ? __ldg(p + 1) : cmake<C>((RT)0, (RT)0);
            if (!lo) A.y = -A.y, B.y = -B.y;
            v[r] = cmake<C>(A.x - B.y, A.y + B.x);
        }
    } else {
    // q = t + P r with 0 <= t < P: slots r < R/2 hold planes below L/2, slot
    // R/2 holds plane L/2 only on t = 0, the rest are mirrors.  All the plane
    // loads are issued before the first use (one HBM latency per tile, not one
    // per plane); the slab path's per-plane peer addresses are resolved first.
    constexpr int RH = R / 2;
    const C* pl[RH + 1];
#pragma unroll
    for (int r = 0; r <= RH; ++r) {
        const int q = min(t + P * r, L / 2);
        pl[r] = src + S * q;
        if constexpr (std::is_same<C, double2>::value)
            if (rp.peer) pl[r] = rp.peer[rp.owner[q]] + rp.off[q] + c;
    }
    const bool mid = t == 0;  // slot RH is plane L/2
    C A[RH + 1], B[RH + 1];
#pragma unroll
    for (int r = 0; r <= RH; ++r) {
        const bool ld = active && (r < RH || mid);
        A[r] = ld ? __ldg(pl[r]) : cmake<C>((RT)0, (RT)0);
        B[r] = ld ? __ldg(pl[r] + 1) : cmake<C>((RT)0, (RT)0);
    }
#pragma unroll
    for (int r = 0; r <= RH; ++r) {
        if (r == RH && !mid) break;
        const int q = t + P * r;
        // what the mirror position L - q needs is conj(A) + i conj(B): one value per plane
        stg[q * TP + lp] = cmake<C>(A[r].x + B[r].y, B[r].x - A[r].y);
        v[r] = cmake<C>(A[r].x - B[r].y, A[r].y + B[r].x);  // A + i B
    }
    __syncthreads();
#pragma unroll
    for (int r = RH; r < R; ++r) {
        const int q = t + P * r;
        if (q > L / 2) v[r] = stg[(L - q) * TP + lp];
    }
    __syncthreads();  // the staging area becomes the exchange buffer
    }
    fftc::stockham<L, true>(v, t, sm, sidx, tw);
    C* dst = reinterpret_cast<C*>(out + c + S * (long long)L * o);
    const long long S2 = S / 2;
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < R; ++j) {
        const int q = fftc::Plan<L>::out_q(t, j);
        const C z = cscale(v[j], (RT)scale);
        if (!active) continue;
        acc += (double)z.x * z.x + (double)z.y * z.y;
        dst[S2 * q] = z;
        if (!isfinite(z.x) || !isfinite(z.y)) {
            const unsigned long long e = (unsigned long long)(c + S * (long long)L * o + S * (long long)q);
            atomicMin(bad_index, isfinite(z.x) ? e + 1 : e);
        }
    }
    if (partials) {
        __shared__ double red[64];
        double vals[2] = {0.0, acc};  // the pair is real by construction: no imaginary residue
        block_reduce_sum<2>(vals, red);
        if (tid == 0) {
            partials[2 * blockIdx.x] = vals[0];
            partials[2 * blockIdx.x + 1] = vals[1];
        }
    }
}

// ---------------------------------------- wide persistent passes (long lines)
// At L >= 1024 a whole line per tile column leaves the kernels above either
// 64-byte HBM rows (4 columns, 2 CTAs per SM) or one 512-thread CTA per SM whose
// loads, transform and stores run one after another.  These kernels keep 8
// complex columns (128-byte rows) AND overlap: a persistent CTA per SM
// prefetches its next tile with cp.async into a per-thread staging area (each
// thread fetches exactly the elements it will hold, so no barrier guards the
// stage) while the current tile is transformed out of registers; the exchanges
// run split (fftc::stockham_split) through a buffer of reals, which is what
// makes room for the stage: 128 KB stage + 64 KB exchange.  Config 4 (1024^3):
// axis-2 half passes 4.1 -> 3.7 ms, forward paired pass 5.1 -> 4.9 ms.
enum { WIDE_PASS = 0, WIDE_RFWD = 1 };

template <int L>
struct WideShape {
    using Pl = fftc::Plan<L>;
    static constexpr int R = Pl::R, P = Pl::P;
    static constexpr int T = 8;  // complex columns (or real column pairs) per tile
    static constexpr int THREADS = T * P;
    static constexpr size_t XCH = (size_t)T * L * sizeof(double);
    static constexpr size_t STAGE = (size_t)THREADS * R * sizeof(double2);  // [R][THREADS]
    static constexpr size_t TWS = (size_t)L * sizeof(double2);  // the twiddle table, staged once per CTA
    static constexpr size_t SMEM = XCH + STAGE + TWS;
    static_assert(SMEM <= 232448, "shared memory budget");
    // exchange slot of line position q, column lt: rows of T reals; the row
    // index is swizzled by its bit 4 so the four t of a warp (rows 16 apart in
    // the first exchange) do not land on the same 16 banks
    __device__ static __forceinline__ int xidx(int q, int lt) { return (q ^ ((q >> 4) & 1)) * T + lt; }
};

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(smem_dst)),
                 "l"(gsrc)
                 : "memory");
}

// MODE = WIDE_PASS: complex -> complex along a strided axis (in place allowed).
// MODE = WIDE_RFWD: the paired real forward axis-3 transform (rpair_fwd_kernel).  The
// inverse (rpair_inv_kernel) stays on its one-tile-per-CTA kernel: staged by
// plane for the conjugate mirrors it measured 5.9 ms against 4.5 ms at config 4.
template <int L, int MODE, bool INV>
__global__ void __launch_bounds__(WideShape<L>::THREADS, 1)
    fft_wide_kernel(const void* in_, void* out_, long long S, long long tiles, const double2* __restrict__ tw,
                    double scale, RemotePlanes rp) {
    using Sh = WideShape<L>;
    constexpr int R = Sh::R, P = Sh::P, T = Sh::T, NT = Sh::THREADS;
    extern __shared__ double2 sm_raw[];
    double* xch = reinterpret_cast<double*>(sm_raw);
    double2* stage = reinterpret_cast<double2*>(xch + (size_t)T * L);
    double2* tw_s = stage + (size_t)NT * R;
    const int tid = threadIdx.x, lt = tid % T, t = tid / T;
    for (int i = tid; i < L; i += NT) tw_s[i] = __ldg(tw + i);
    __syncthreads();
    const fftc::TwShared<double2> twp{tw_s};
    const long long tpo = S / (MODE == WIDE_PASS ? T : 2 * T);
    auto sidx = [&](int q) { return Sh::xidx(q, lt); };

    // element (row) strides in double2 units and the tile's first element
    const long long in_rs = MODE == WIDE_PASS ? S : S / 2;
    auto in_base = [&](long long tile) -> const double2* {
        const long long o = tile / tpo, c0 = (tile % tpo) * T;
        if (MODE == WIDE_PASS) return static_cast<const double2*>(in_) + c0 + lt + S * (long long)L * o;
        return static_cast<const double2*>(in_) + c0 + lt + (S / 2) * (long long)L * o;
    };
    auto prefetch = [&](long long tile) {
        const double2* src = in_base(tile);
#pragma unroll
        for (int r = 0; r < R; ++r) cp_async16(stage + (size_t)r * NT + tid, src + in_rs * (t + P * r));
        asm volatile("cp.async.commit_group;" ::: "memory");
    };

    long long tile = blockIdx.x;
    if (tile < tiles) prefetch(tile);
    for (; tile < tiles; tile += gridDim.x) {
        double2 v[R];
        asm volatile("cp.async.wait_all;" ::: "memory");
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = stage[(size_t)r * NT + tid];
        const long long next = tile + gridDim.x;
        if (next < tiles) prefetch(next);  // lands while this tile is transformed and stored

        fftc::stockham_split<L, INV, decltype(sidx), 16, fftc::CtaSync, fftc::TwShared<double2>>(v, t, xch, sidx, twp);

        const long long o = tile / tpo, c0 = (tile % tpo) * T;
        if constexpr (MODE == WIDE_PASS) {
            double2* dst = static_cast<double2*>(out_) + c0 + lt + S * (long long)L * o;
#pragma unroll
            for (int j = 0; j < R; ++j) dst[S * (long long)fftc::Plan<L>::out_q(t, j)] = cscale(v[j], scale);
        } else {
            // Hermitian split X_c[k] = (Z[k] + conj Z[L-k]) / 2, X_{c+1}[k] = (Z[k] - conj Z[L-k]) / 2i,
            // k <= L/2: Z[k] is in this thread's registers, Z[L-k] (a position above
            // L/2, or k itself at k = 0, L/2) comes through the real exchange buffer,
            // real parts first, then imaginary parts
            double bx[R];
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const int q = fftc::Plan<L>::out_q(t, j);
                if (q > L / 2) xch[sidx(q)] = v[j].x;
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const int k = fftc::Plan<L>::out_q(t, j);
                if (k <= L / 2) bx[j] = (k == 0 || k == L / 2) ? v[j].x : xch[sidx(L - k)];
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const int q = fftc::Plan<L>::out_q(t, j);
                if (q > L / 2) xch[sidx(q)] = v[j].y;
            }
            __syncthreads();
            double2* dst = static_cast<double2*>(out_) + 2 * (c0 + lt) + S * (long long)(L / 2 + 1) * o;
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const int k = fftc::Plan<L>::out_q(t, j);
                if (k <= L / 2) {
                    const double2 a = v[j];
                    const double by = (k == 0 || k == L / 2) ? a.y : xch[sidx(L - k)];
                    // slab-sharded: plane k goes straight to its owner's spectral buffer
                    // (peer memory over NVLink), as in rpair_fwd_kernel
                    double2* d = rp.peer ? rp.peer[rp.owner[k]] + rp.off[k] + 2 * (c0 + lt) : dst + S * (long long)k;
                    d[0] = make_double2(0.5 * (a.x + bx[j]), 0.5 * (a.y - by));
                    d[1] = make_double2(0.5 * (a.y + by), -0.5 * (a.x - bx[j]));
                }
            }
            __syncthreads();  // the buffer is read out before the next tile's first exchange
        }
    }
    if (MODE == WIDE_RFWD && rp.peer) __threadfence_system();
}

static int wide_sm_count() {
    static int n = [] {
        int dev = 0, v = 0;
        VSR_CUDA(cudaGetDevice(&dev));
        VSR_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
        return v;
    }();
    return n;
}
static bool wide_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("VSR_NO_WIDE");
        return !(e && e[0] == '1');
    }();
    return on;
}

template <int L, int MODE, bool INV>
void launch_wide(const void* in, void* out, long long S, long long tiles, const double2* tw, double scale,
                 cudaStream_t st, const RemotePlanes& rp = RemotePlanes{}) {
    using Sh = WideShape<L>;
    auto kern = fft_wide_kernel<L, MODE, INV>;
    const size_t smem = Sh::SMEM;
    VSR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const unsigned grid = (unsigned)std::min<long long>(tiles, wide_sm_count());
    kern<<<grid, Sh::THREADS, smem, st>>>(in, out, S, tiles, tw, scale, rp);
    VSR_LAUNCH_CHECK();
}

template <int L, class C>
bool launch_rpair(bool fwd, const void* in, void* out, long long S, long long total, const C* tw,
                  double scale, const PassReduce* red, cudaStream_t st, const RemotePlanes& rp) {
    using Sh = RPairShape<L>;
    using RT = typename CplxT<C>::real;
    const long long tiles = total / ((long long)Sh::T * L);
    const unsigned blocks = (unsigned)((tiles + Sh::TG - 1) / Sh::TG);
    const size_t smem = (size_t)Sh::SMEM * sizeof(C);
    if constexpr (L == 1024 && std::is_same<C, double2>::value) {
        static_assert(Sh::T == 2 * WideShape<L>::T && Sh::TG == 1, "wide tiles match the rpair tiles");
        if (fwd && wide_enabled()) {
            launch_wide<L, WIDE_RFWD, false>(in, out, S, tiles, tw, 1.0, st, rp);
            return true;
        }
    }
    if (fwd) {
        auto kern = rpair_fwd_kernel<L, C>;
        if (smem > 48 * 1024) VSR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<blocks, Sh::THREADS, smem, st>>>(static_cast<const RT*>(in), static_cast<C*>(out), S, tiles, tw, rp);
    } else {
        auto kern = rpair_inv_kernel<L, C>;
        if (smem > 48 * 1024) VSR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        kern<<<blocks, Sh::THREADS, smem, st>>>(static_cast<const C*>(in), static_cast<RT*>(out), S, tiles, tw,
                                                scale, red ? red->partials : nullptr,
                                                red ? red->bad_index : nullptr, rp);
    }
    VSR_LAUNCH_CHECK();
    return true;
}

template <class C>
bool dispatch_rpair(bool fwd, size_t L, const void* in, void* out, long long S, long long total, const C* tw,
                    double scale, const PassReduce* red, cudaStream_t st, const RemotePlanes& rp = RemotePlanes{}) {
    switch (L) {
        case 8: return launch_rpair<8, C>(fwd, in, out, S, total, tw, scale, red, st, rp);
        case 16: return launch_rpair<16, C>(fwd, in, out, S, total, tw, scale, red, st, rp);
        case 32: return launch_rpair<32, C>(fwd, in, out, S, total, tw, scale, red, st, rp);
        case 64: return launch_rpair<64, C>(fwd, in, out, S, total, tw, scale, red, st, rp);
        case 128: return launch_rpair<128, C>(fwd, in, out, S, total, tw, scale, red, st, rp);
        case 256: return launch_rpair<256, C>(fwd, in, out, S, total, tw, scale, red, st, rp);
        case 512: return launch_rpair<512, C>(fwd, in, out, S, total, tw, scale, red, st, rp);
        case 1024: return launch_rpair<1024, C>(fwd, in, out, S, total, tw, scale, red, st, rp);
        default: return false;
    }
}

// ------------------------------------------------------------ generic DFT
// Direct O(L) per output DFT along one axis for any L (non powers of two,
// L = 1, and strided shapes the tiled kernel cannot cover).  One thread per
// output element.
template <bool INV, int IK, int OK>
__global__ void __launch_bounds__(256)
    dft_direct_kernel(const void* __restrict__ in_, void* __restrict__ out_, long long S,
                      long long L, long long total, const double2* __restrict__ tw,
                      double scale, double* __restrict__ partials,
                      unsigned long long* __restrict__ bad_index) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    double acc_im = 0.0, acc_tot = 0.0;
    if (e < total) {
        const long long p = e % S;
        const long long q = (e / S) % L;
        const long long o = e / (S * L);
        const long long base = p + S * L * o;
        double2 acc = make_double2(0.0, 0.0);
        long long idx = 0;  // (j * q) mod L
        for (long long j = 0; j < L; ++j) {
            double2 x;
            if constexpr (IK == IN_REAL)
                x = make_double2(reinterpret_cast<const double*>(in_)[base + S * j], 0.0);
            else
                x = reinterpret_cast<const double2*>(in_)[base + S * j];
            const double2 w = tw[idx];
            const double2 prod = INV ? cmulc(w, x) : cmul(w, x);
            acc = cadd(acc, prod);
            idx += q;
            if (idx >= L) idx -= L;
        }
        acc = cscale(acc, scale);
        if constexpr (OK == OUT_REAL) {
            acc_im = acc.y * acc.y;
            acc_tot = acc.x * acc.x + acc.y * acc.y;
            reinterpret_cast<double*>(out_)[e] = acc.x;
            if (!isfinite(acc.x)) atomicMin(bad_index, (unsigned long long)e);
        } else {
            reinterpret_cast<double2*>(out_)[e] = acc;
        }
    }
    if constexpr (OK == OUT_REAL) {
        __shared__ double red[64];
        double vals[2] = {acc_im, acc_tot};
        block_reduce_sum<2>(vals, red);
        if (threadIdx.x == 0) {
            partials[2 * blockIdx.x] = vals[0];
            partials[2 * blockIdx.x + 1] = vals[1];
        }
    }
}

// ------------------------------------------------------------ dispatch
// lines per tile of a strided pass (8: 128-B rows; whole lines sit in smem, so
// lines of 1024+ points take 4 -- 8 at L = 1024 measured slower, 128 KB of
// smem per CTA): the ONE definition the kernels, the block counts and the
// geometry checks all use
constexpr long long strided_cols(long long L) { return L >= 1024 ? 4 : 8; }

template <int L>
struct LCfg {
    static constexpr int R = L < 16 ? L : 16;
    static constexpr int P = L / R;
    // strided tile width and tiles per CTA (>= 128 threads per CTA)
    static constexpr int TS = strided_cols(L);
    static constexpr int TGS = (TS * P) >= 128 ? 1 : (128 / (TS * P));
    // contiguous: lines per CTA
    static constexpr int TGC = P >= 128 ? 1 : (128 / P);
};

struct Launch {
    dim3 grid, block;
    size_t smem;
};

template <int L, bool CONTIG, class CT = double2>
Launch pass_geometry(long long S, long long lines_or_tiles) {
    using C = LCfg<L>;
    constexpr int T = CONTIG ? 1 : C::TS;
    constexpr int TG = CONTIG ? C::TGC : C::TGS;
    using Sh = PassShape<L, C::R, T, TG, CONTIG>;
    Launch g;
    g.block = dim3(Sh::THREADS);
    g.grid = dim3((unsigned)((lines_or_tiles + TG - 1) / TG));
    g.smem = (size_t)Sh::SMEM_ELEMS * sizeof(CT);
    return g;
}

template <int L, bool CONTIG, bool INV, int IK, int OK, class CT = double2>
void launch_pass(long long S, long long units, const void* in, void* out, const CT* tw,
                 double scale, const PassReduce* red, cudaStream_t st) {
    using C = LCfg<L>;
    constexpr int T = CONTIG ? 1 : C::TS;
    constexpr int TG = CONTIG ? C::TGC : C::TGS;
    if constexpr (L == 1024 && !CONTIG && IK == IN_COMPLEX && OK == OUT_COMPLEX && std::is_same<CT, double2>::value) {
        // units are tiles of T = 4 columns; the wide kernel takes 8
        if (wide_enabled() && S % WideShape<L>::T == 0) {
            launch_wide<L, WIDE_PASS, INV>(in, out, S, units * T / WideShape<L>::T, tw, scale, st);
            return;
        }
    }
    auto kern = fft_pass_kernel<L, C::R, T, TG, CONTIG, INV, IK, OK, CT>;
    Launch g = pass_geometry<L, CONTIG, CT>(S, units);
    if (g.smem > 48 * 1024) {
        VSR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)g.smem));
    }
    kern<<<g.grid, g.block, g.smem, st>>>(in, out, S, units, tw, scale,
                                          red ? red->partials : nullptr,
                                          red ? red->bad_index : nullptr);
    VSR_LAUNCH_CHECK();
}

template <bool CONTIG, bool INV, int IK, int OK, class CT = double2>
bool dispatch_L(size_t L, long long S, long long units, const void* in, void* out,
                const CT* tw, double scale, const PassReduce* red, cudaStream_t st) {
    switch (L) {
#define VSR_CASE(LL)                                                                       \
    case LL:                                                                               \
        launch_pass<LL, CONTIG, INV, IK, OK, CT>(S, units, in, out, tw, scale, red, st);   \
        return true;
        VSR_CASE(2)
        VSR_CASE(4)
        VSR_CASE(8)
        VSR_CASE(16)
        VSR_CASE(32)
        VSR_CASE(64)
        VSR_CASE(128)
        VSR_CASE(256)
        VSR_CASE(512)
        VSR_CASE(1024)
        VSR_CASE(2048)
#undef VSR_CASE
        default:
            return false;
    }
}

template <bool CONTIG>
long long pass_units(size_t L, long long S, long long total) {
    if (CONTIG) return total / (long long)L;
    const size_t TS = (size_t)strided_cols((long long)L);
    return total / ((long long)TS * (long long)L);  // tiles of TS whole lines
}

size_t blocks_for(size_t L, bool contig, long long units) {
    size_t P = L < 16 ? 1 : L / 16;
    size_t TS = (size_t)strided_cols((long long)L);
    size_t tg;
    if (contig)
        tg = P >= 128 ? 1 : 128 / P;
    else
        tg = (TS * P) >= 128 ? 1 : 128 / (TS * P);
    return (size_t)((units + (long long)tg - 1) / (long long)tg);
}

bool tiled_ok(size_t L, int axis, long long S) {
    if (L < 2 || L > 2048 || !is_pow2(L)) return false;
    if (axis == 0) return true;
    const long long TS = strided_cols((long long)L);
    return S % TS == 0;
}

}  // namespace

FftEngine& fft_engine() {
    static FftEngine eng;
    return eng;
}

const double2* FftEngine::twiddles(size_t L) {
    int dev = 0;
    VSR_CUDA(cudaGetDevice(&dev));
    const size_t key = ((size_t)dev << 40) | L;
    std::lock_guard<std::mutex> lock(mu_);
    auto it = tw_.find(key);
    if (it != tw_.end()) return it->second;
    std::vector<double2> h(L);
    for (size_t j = 0; j < L; ++j) {
        // long double argument reduction keeps every entry correctly rounded
        // for the table sizes used here.
        const long double ang = 2.0L * 3.141592653589793238462643383279502884L *
                                (long double)j / (long double)L;
        h[j] = make_double2((double)cosl(ang), (double)-sinl(ang));
    }
    double2* d = nullptr;
    VSR_CUDA(cudaMalloc(&d, L * sizeof(double2)));
    VSR_CUDA(cudaMemcpy(d, h.data(), L * sizeof(double2), cudaMemcpyHostToDevice));
    tw_[key] = d;
    return d;
}

const float2* FftEngine::twiddles_f(size_t L) {
    int dev = 0;
    VSR_CUDA(cudaGetDevice(&dev));
    const size_t key = ((size_t)dev << 40) | L;
    std::lock_guard<std::mutex> lock(mu_);
    auto it = twf_.find(key);
    if (it != twf_.end()) return it->second;
    std::vector<float2> h(L);
    for (size_t j = 0; j < L; ++j) {
        const long double ang = 2.0L * 3.141592653589793238462643383279502884L *
                                (long double)j / (long double)L;
        h[j] = make_float2((float)cosl(ang), (float)-sinl(ang));
    }
    float2* d = nullptr;
    VSR_CUDA(cudaMalloc(&d, L * sizeof(float2)));
    VSR_CUDA(cudaMemcpy(d, h.data(), L * sizeof(float2), cudaMemcpyHostToDevice));
    twf_[key] = d;
    return d;
}

static void axis_geometry(const Dims& d, int axis, long long& S, long long& L, long long& total) {
    total = (long long)d.count();
    L = (long long)d.len(axis);
    S = axis == 0 ? 1 : (axis == 1 ? (long long)d.m : (long long)(d.m * d.n));
}

size_t FftEngine::pass_blocks(const Dims& d, int axis) const {
    long long S, L, total;
    axis_geometry(d, axis, S, L, total);
    if (tiled_ok((size_t)L, axis, S)) {
        const long long units = axis == 0 ? pass_units<true>(L, S, total)
                                          : pass_units<false>(L, S, total);
        return blocks_for((size_t)L, axis == 0, units);
    }
    return (size_t)((total + 255) / 256);
}

void FftEngine::axis_pass(const Dims& d, int axis, bool inverse, const void* in, InKind ik,
                          void* out, OutKind ok, double scale, const PassReduce* red,
                          cudaStream_t st) {
    long long S, L, total;
    axis_geometry(d, axis, S, L, total);
    if (total == 0) return;
    const double2* tw = twiddles((size_t)L);
    if (tiled_ok((size_t)L, axis, S)) {
        bool done = false;
        if (axis == 0) {
            const long long units = pass_units<true>(L, S, total);
            if (!inverse) {
                if (ik == IN_REAL && ok == OUT_COMPLEX)
                    done = dispatch_L<true, false, IN_REAL, OUT_COMPLEX>(L, S, units, in, out, tw, scale, red, st);
                else if (ik == IN_COMPLEX && ok == OUT_COMPLEX)
                    done = dispatch_L<true, false, IN_COMPLEX, OUT_COMPLEX>(L, S, units, in, out, tw, scale, red, st);
            } else {
                if (ik == IN_COMPLEX && ok == OUT_REAL)
                    done = dispatch_L<true, true, IN_COMPLEX, OUT_REAL>(L, S, units, in, out, tw, scale, red, st);
                else if (ik == IN_COMPLEX && ok == OUT_COMPLEX)
                    done = dispatch_L<true, true, IN_COMPLEX, OUT_COMPLEX>(L, S, units, in, out, tw, scale, red, st);
            }
        } else {
            const long long units = pass_units<false>(L, S, total);
            if (!inverse) {
                if (ik == IN_COMPLEX && ok == OUT_COMPLEX)
                    done = dispatch_L<false, false, IN_COMPLEX, OUT_COMPLEX>(L, S, units, in, out, tw, scale, red, st);
                else if (ik == IN_REAL && ok == OUT_COMPLEX)
                    done = dispatch_L<false, false, IN_REAL, OUT_COMPLEX>(L, S, units, in, out, tw, scale, red, st);
            } else {
                if (ik == IN_COMPLEX && ok == OUT_COMPLEX)
                    done = dispatch_L<false, true, IN_COMPLEX, OUT_COMPLEX>(L, S, units, in, out, tw, scale, red, st);
                else if (ik == IN_COMPLEX && ok == OUT_REAL)
                    done = dispatch_L<false, true, IN_COMPLEX, OUT_REAL>(L, S, units, in, out, tw, scale, red, st);
            }
        }
        if (done) return;
    }
    // Generic direct DFT.  Out-of-place only: stage through a temporary when
    // the caller asked for an in-place pass.
    void* dst = out;
    void* tmp = nullptr;
    const size_t out_bytes = (size_t)total * (ok == OUT_REAL ? sizeof(double) : sizeof(double2));
    if (in == out) {
        VSR_CUDA(cudaMallocAsync(&tmp, out_bytes, st));
        dst = tmp;
    }
    const unsigned blocks = (unsigned)((total + 255) / 256);
    double* part = red ? red->partials : nullptr;
    unsigned long long* bad = red ? red->bad_index : nullptr;
#define VSR_DIRECT(INV, IK, OK) \
    dft_direct_kernel<INV, IK, OK><<<blocks, 256, 0, st>>>(in, dst, S, L, total, tw, scale, part, bad)
    if (!inverse) {
        if (ik == IN_REAL && ok == OUT_COMPLEX) VSR_DIRECT(false, IN_REAL, OUT_COMPLEX);
        else if (ik == IN_COMPLEX && ok == OUT_COMPLEX) VSR_DIRECT(false, IN_COMPLEX, OUT_COMPLEX);
        else throw std::logic_error("fft: unsupported forward pass kinds");
    } else {
        if (ik == IN_COMPLEX && ok == OUT_REAL) VSR_DIRECT(true, IN_COMPLEX, OUT_REAL);
        else if (ik == IN_COMPLEX && ok == OUT_COMPLEX) VSR_DIRECT(true, IN_COMPLEX, OUT_COMPLEX);
        else throw std::logic_error("fft: unsupported inverse pass kinds");
    }
#undef VSR_DIRECT
    VSR_LAUNCH_CHECK();
    if (tmp) {
        VSR_CUDA(cudaMemcpyAsync(out, tmp, out_bytes, cudaMemcpyDeviceToDevice, st));
        VSR_CUDA(cudaFreeAsync(tmp, st));
    }
}

bool FftEngine::half3_ok(const Dims& d) const {
    return d.s >= 8 && d.s <= 1024 && is_pow2(d.s) && (d.m * d.n) % 16 == 0;
}

size_t FftEngine::half3_blocks(const Dims& d) const {
    const size_t T = kRPairCols;
    const size_t P = d.s < 16 ? 1 : d.s / 16, tp = (T / 2) * P;
    const size_t tg = tp >= 128 ? 1 : 128 / tp;
    return (d.count() / (T * d.s) + tg - 1) / tg;
}

void FftEngine::r2c_axis3_half(const Dims& d, const double* in, double2* out, cudaStream_t st) {
    long long S, L, total;
    axis_geometry(d, 2, S, L, total);
    if (!half3_ok(d)) throw std::logic_error("r2c_axis3_half: unsupported geometry");
    if (!dispatch_rpair(true, (size_t)L, in, out, S, total, twiddles((size_t)L), 1.0, nullptr, st))
        throw std::logic_error("r2c_axis3_half: unsupported length");
}

void FftEngine::r2c_axis3_half_remote(const Dims& d, const double* in, const RemotePlanes& rp, cudaStream_t st) {
    long long S, L, total;
    axis_geometry(d, 2, S, L, total);
    if (!half3_ok(d)) throw std::logic_error("r2c_axis3_half: unsupported geometry");
    if (!dispatch_rpair(true, (size_t)L, in, nullptr, S, total, twiddles((size_t)L), 1.0, nullptr, st, rp))
        throw std::logic_error("r2c_axis3_half: unsupported length");
}

void FftEngine::c2r_axis3_half_remote(const Dims& d, const RemotePlanes& rp, double* out, double scale,
                                      const PassReduce* red, cudaStream_t st) {
    long long S, L, total;
    axis_geometry(d, 2, S, L, total);
    if (!half3_ok(d)) throw std::logic_error("c2r_axis3_half: unsupported geometry");
    if (!dispatch_rpair(false, (size_t)L, nullptr, out, S, total, twiddles((size_t)L), scale, red, st, rp))
        throw std::logic_error("c2r_axis3_half: unsupported length");
}

void FftEngine::c2r_axis3_half(const Dims& d, const double2* in, double* out, double scale, const PassReduce* red,
                               cudaStream_t st) {
    long long S, L, total;
    axis_geometry(d, 2, S, L, total);
    if (!half3_ok(d)) throw std::logic_error("c2r_axis3_half: unsupported geometry");
    if (!dispatch_rpair(false, (size_t)L, in, out, S, total, twiddles((size_t)L), scale, red, st))
        throw std::logic_error("c2r_axis3_half: unsupported length");
}

// ---- fp32 mode (float2 spectra, fp32 arithmetic): the half-spectrum passes of
// the ADMM-TV iteration
void FftEngine::axis_pass_cf(const Dims& d, int axis, bool inverse, float2* inout, cudaStream_t st) {
    long long S, L, total;
    axis_geometry(d, axis, S, L, total);
    if (total == 0) return;
    if (axis == 0 || !tiled_ok((size_t)L, axis, S)) throw std::logic_error("fp32 axis pass: unsupported geometry");
    const long long units = pass_units<false>(L, S, total);
    const float2* tw = twiddles_f((size_t)L);
    const bool done =
        inverse ? dispatch_L<false, true, IN_COMPLEX, OUT_COMPLEX, float2>(L, S, units, inout, inout, tw, 1.0,
                                                                          nullptr, st)
                : dispatch_L<false, false, IN_COMPLEX, OUT_COMPLEX, float2>(L, S, units, inout, inout, tw, 1.0,
                                                                           nullptr, st);
    if (!done) throw std::logic_error("fp32 axis pass: unsupported length");
}

void FftEngine::r2c_axis3_half_f(const Dims& d, const float* in, float2* out, cudaStream_t st) {
    long long S, L, total;
    axis_geometry(d, 2, S, L, total);
    if (!half3_ok(d)) throw std::logic_error("r2c_axis3_half: unsupported geometry");
    if (!dispatch_rpair<float2>(true, (size_t)L, in, out, S, total, twiddles_f((size_t)L), 1.0, nullptr, st))
        throw std::logic_error("r2c_axis3_half: unsupported length");
}

void FftEngine::c2r_axis3_half_f(const Dims& d, const float2* in, float* out, double scale, const PassReduce* red,
                                 cudaStream_t st) {
    long long S, L, total;
    axis_geometry(d, 2, S, L, total);
    if (!half3_ok(d)) throw std::logic_error("c2r_axis3_half: unsupported geometry");
    if (!dispatch_rpair<float2>(false, (size_t)L, in, out, S, total, twiddles_f((size_t)L), scale, red, st))
        throw std::logic_error("c2r_axis3_half: unsupported length");
}

void FftEngine::forward3(const Dims& d, const void* in, InKind ik, double2* out, double scale,
                         cudaStream_t st, Profiler* prof) {
    {
        ProfScope ps(prof, ik == IN_REAL ? "fft_fwd_axis1_r2c" : "fft_fwd_axis1", st);
        axis_pass(d, 0, false, in, ik, out, OUT_COMPLEX, 1.0, nullptr, st);
    }
    {
        ProfScope ps(prof, "fft_fwd_axis2", st);
        axis_pass(d, 1, false, out, IN_COMPLEX, out, OUT_COMPLEX, 1.0, nullptr, st);
    }
    {
        ProfScope ps(prof, "fft_fwd_axis3", st);
        axis_pass(d, 2, false, out, IN_COMPLEX, out, OUT_COMPLEX, scale, nullptr, st);
    }
}

void FftEngine::inverse3(const Dims& d, double2* in, void* out, OutKind ok, double scale,
                         const PassReduce* red, cudaStream_t st, Profiler* prof) {
    {
        ProfScope ps(prof, "fft_inv_axis3", st);
        axis_pass(d, 2, true, in, IN_COMPLEX, in, OUT_COMPLEX, 1.0, nullptr, st);
    }
    {
        ProfScope ps(prof, "fft_inv_axis2", st);
        axis_pass(d, 1, true, in, IN_COMPLEX, in, OUT_COMPLEX, 1.0, nullptr, st);
    }
    {
        ProfScope ps(prof, ok == OUT_REAL ? "fft_inv_axis1_c2r" : "fft_inv_axis1", st);
        axis_pass(d, 0, true, in, IN_COMPLEX, out, ok, scale, red, st);
    }
}

void FftEngine::inverse21(const Dims& d, double2* in, void* out, OutKind ok, double scale,
                          const PassReduce* red, cudaStream_t st, Profiler* prof) {
    {
        ProfScope ps(prof, "fft_inv_axis2", st);
        axis_pass(d, 1, true, in, IN_COMPLEX, in, OUT_COMPLEX, 1.0, nullptr, st);
    }
    {
        ProfScope ps(prof, ok == OUT_REAL ? "fft_inv_axis1_c2r" : "fft_inv_axis1", st);
        axis_pass(d, 0, true, in, IN_COMPLEX, out, ok, scale, red, st);
    }
}

void FftEngine::forward12(const Dims& d, const void* in, InKind ik, double2* out, cudaStream_t st,
                          Profiler* prof) {
    {
        ProfScope ps(prof, ik == IN_REAL ? "fft_fwd_axis1_r2c" : "fft_fwd_axis1", st);
        axis_pass(d, 0, false, in, ik, out, OUT_COMPLEX, 1.0, nullptr, st);
    }
    {
        ProfScope ps(prof, "fft_fwd_axis2", st);
        axis_pass(d, 1, false, out, IN_COMPLEX, out, OUT_COMPLEX, 1.0, nullptr, st);
    }
}

}  // namespace vsr
