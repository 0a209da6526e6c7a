// Per-rank stages of the slab-decomposed (axis 3) distributed path
// (SURVEY §8(e)).  A rank holds z-slab p of every spatial volume (sz = s/P
// planes) and, in the spectral domain, the rows f2 of its alias-closed row
// set R(p) = { g2 + bc*nl : g2 in [p*nl/P, (p+1)*nl/P), bc < dc } for every
// (f1, f3): local spectral layout [f3][jl][f1] with jl = bc*(nl/P) + g2_local,
// i.e. a "local decimation geometry" (m, n/P, s) with rates (dr, dc, ds) and
// nl_local = nl/P, on which the fused fold kernels run unchanged.
//
// The exchange steps (all-to-all, halos, scalar gathers) are done by the
// host orchestrator (paper_2010_15491_b200/dist.py) with NCCL through
// torch.distributed; these functions are the device work between them, all
// enqueued on the context stream.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <functional>
#include <list>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/vsr.h"
#include "fft.cuh"
#include "fold.cuh"
#include "fused.cuh"
#include "tv.cuh"

namespace vsr {
namespace {

struct Slab {
    long long m, n, s, P, sz, nP, ml, nl, sl, nlP;
    int rates[3];
};

Slab make_slab(const size_t hr[3], const size_t rates[3], int P) {
    if (P < 1) throw std::invalid_argument("slab: P must be >= 1");
    Slab g;
    g.m = (long long)hr[0];
    g.n = (long long)hr[1];
    g.s = (long long)hr[2];
    g.P = P;
    for (int a = 0; a < 3; ++a) {
        if (rates[a] == 0 || hr[a] % rates[a]) throw shape_error("slab: rates must divide the HR dims");
        g.rates[a] = (int)rates[a];
    }
    g.ml = g.m / g.rates[0];
    g.nl = g.n / g.rates[1];
    g.sl = g.s / g.rates[2];
    if (g.s % P) throw shape_error("slab: P must divide axis 3 (" + std::to_string(g.s) + ")");
    if (g.nl % P) throw shape_error("slab: P must divide the LR axis 2 (" + std::to_string(g.nl) + ")");
    g.sz = g.s / P;
    g.nP = g.n / P;
    g.nlP = g.nl / P;
    return g;
}

// global row f2 of local spectral row jl on rank p
__host__ __device__ inline long long row_of(long long jl, long long p, long long nlP, long long nl) {
    return (p * nlP + jl % nlP) + (jl / nlP) * nl;
}

// send[q][z][jl][f1] = work[z][row_of(jl, q)][f1]
__global__ void pack_kernel(Slab g, const double2* __restrict__ work, double2* __restrict__ send) {
    const long long total = g.m * g.n * g.sz;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= total) return;
    const long long f1 = e % g.m;
    long long r = e / g.m;
    const long long jl = r % g.nP;
    r /= g.nP;
    const long long z = r % g.sz;
    const long long q = r / g.sz;
    send[e] = work[f1 + g.m * (row_of(jl, q, g.nlP, g.nl) + g.n * z)];
}

// work[z][row_of(jl, q)][f1] = recv[q][z][jl][f1]
__global__ void unpack_kernel(Slab g, const double2* __restrict__ recv, double2* __restrict__ work) {
    const long long total = g.m * g.n * g.sz;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= total) return;
    const long long f1 = e % g.m;
    long long r = e / g.m;
    const long long jl = r % g.nP;
    r /= g.nP;
    const long long z = r % g.sz;
    const long long q = r / g.sz;
    work[f1 + g.m * (row_of(jl, q, g.nlP, g.nl) + g.n * z)] = recv[e];
}

// Yl_loc[g3][g2l][g1] = Yl[g3][p*nlP + g2l][g1]
__global__ void lr_slice_kernel(Slab g, long long p, const double2* __restrict__ Yl, double2* __restrict__ out) {
    const long long total = g.ml * g.nlP * g.sl;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= total) return;
    const long long g1 = e % g.ml;
    const long long g2l = (e / g.ml) % g.nlP;
    const long long g3 = e / (g.ml * g.nlP);
    out[e] = Yl[g1 + g.ml * ((p * g.nlP + g2l) + g.nl * g3)];
}

unsigned blocks(long long n) { return (unsigned)((n + 255) / 256); }

FoldGeom local_geom(const Slab& g) {
    FoldGeom G;
    G.m = g.m;
    G.n = g.nP;
    G.s = g.s;
    G.dr = g.rates[0];
    G.dc = g.rates[1];
    G.ds = g.rates[2];
    G.ml = g.ml;
    G.nl = g.nlP;
    G.sl = g.sl;
    G.d = G.dr * G.dc * G.ds;
    return G;
}

std::vector<double> diff_norm_table(long long len) {
    std::vector<double> t((size_t)len);
    const double two_pi = 2.0 * 3.14159265358979323846;
    for (long long f = 0; f < len; ++f) {
        if (f == 0) {
            t[(size_t)f] = 0.0;
            continue;
        }
        const double ang = two_pi * (double)f / (double)len;
        const double re = std::cos(ang) - 1.0, im = std::sin(ang);
        t[(size_t)f] = re * re + im * im;
    }
    return t;
}

__global__ void sum_partials_kernel(const double* __restrict__ p, int stride, int nvals, long long nb,
                                    double* __restrict__ out) {
    __shared__ double red[32 * 4];
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (long long i = threadIdx.x; i < nb; i += blockDim.x)
        for (int k = 0; k < nvals; ++k) v[k] += p[i * stride + k];
    block_reduce_sum<4>(v, red);
    if (threadIdx.x == 0)
        for (int k = 0; k < nvals; ++k) out[k] = v[k];
}

}  // namespace
}  // namespace vsr

using namespace vsr;

// ---------------------------------------------------------------- C ABI
// Declared in include/vsr.h.  Error handling and the context come from capi.cu.
namespace vsr_capi {
cudaStream_t stream_of(vsr_ctx* ctx);
int device_of(vsr_ctx* ctx);
int guard_call(const std::function<void()>& f);
}  // namespace vsr_capi

namespace {
struct DevGuard {
    int prev = 0, want;
    explicit DevGuard(int dev) : want(dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DevGuard() {
        if (prev != want) cudaSetDevice(prev);
    }
};
}  // namespace

namespace {
// Per-rank constant state of the TV fold, built on the first call for a given
// (context, Lambda slice, geometry, rank) and reused by every iteration: the
// Gamma tables (global rows/slices, local columns), the fit partials, and -
// when this rank's Lambda slice is separable, Lambda = a[f1] b[jl] c[f3] -
// the local 1-D factors, so the fused fold rebuilds Lambda instead of
// streaming 16 N / P bytes per iteration.  lam_loc must stay constant while
// it is used (the slab ADMM-TV program computes it once).
struct TvFoldState {
    const void* ctx = nullptr;
    const double* lam = nullptr;
    long long m = 0, nP = 0, s = 0, rank = -1, P = 0;
    int rates[3] = {0, 0, 0};
    double* nr = nullptr;
    double* nc = nullptr;
    double* ns = nullptr;
    double* fitp = nullptr;
    double2* sep = nullptr;  // a (m) | b (nP) | c (s), or nullptr
    size_t nb = 0;
};

void free_state(TvFoldState& e) {
    cudaFree(e.nr), cudaFree(e.nc), cudaFree(e.ns), cudaFree(e.fitp);
    if (e.sep) cudaFree(e.sep);
}

std::list<TvFoldState>& state_cache() {
    static std::list<TvFoldState> cache;  // references stay valid as entries come and go
    return cache;
}
std::mutex& state_mutex() {
    static std::mutex mu;  // several host threads may drive ranks of one process
    return mu;
}

// rebuild = true (vsr_slab_tv_prepare_d): the Lambda slice behind lam_loc is new
TvFoldState& tv_fold_state(vsr_ctx* ctx, const Slab& g, int rank, const double* lam_loc, const FoldGeom& G,
                           cudaStream_t st, bool rebuild = false) {
    auto& cache = state_cache();
    std::lock_guard<std::mutex> lock(state_mutex());
    for (auto it = cache.begin(); it != cache.end(); ++it) {
        auto& e = *it;
        if (e.ctx == ctx && e.lam == lam_loc && e.m == g.m && e.nP == g.nP && e.s == g.s && e.rank == rank &&
            e.P == g.P && e.rates[0] == g.rates[0] && e.rates[1] == g.rates[1] && e.rates[2] == g.rates[2]) {
            if (!rebuild) return e;
            VSR_CUDA(cudaStreamSynchronize(st));  // no queued fold still reads these tables
            free_state(e);
            cache.erase(it);
            break;
        }
    }
    TvFoldState e;
    e.ctx = ctx, e.lam = lam_loc, e.m = g.m, e.nP = g.nP, e.s = g.s, e.rank = rank, e.P = g.P;
    for (int a = 0; a < 3; ++a) e.rates[a] = g.rates[a];
    const auto nr = diff_norm_table(g.m), ns = diff_norm_table(g.s), ncg = diff_norm_table(g.n);
    std::vector<double> nc((size_t)g.nP);
    for (long long jl = 0; jl < g.nP; ++jl) nc[(size_t)jl] = ncg[(size_t)row_of(jl, rank, g.nlP, g.nl)];
    VSR_CUDA(cudaMalloc(&e.nr, nr.size() * sizeof(double)));
    VSR_CUDA(cudaMalloc(&e.nc, nc.size() * sizeof(double)));
    VSR_CUDA(cudaMalloc(&e.ns, ns.size() * sizeof(double)));
    VSR_CUDA(cudaMemcpyAsync(e.nr, nr.data(), nr.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    VSR_CUDA(cudaMemcpyAsync(e.nc, nc.data(), nc.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    VSR_CUDA(cudaMemcpyAsync(e.ns, ns.data(), ns.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    e.nb = fused_axis3_ok(G) ? tv_sandwich_blocks(G) : tv_fold_blocks(G);
    VSR_CUDA(cudaMalloc(&e.fitp, std::max<size_t>(e.nb, 1) * sizeof(double)));
    if (fused_axis3_ok(G)) {
        const Dims ld{(size_t)g.m, (size_t)g.nP, (size_t)g.s};
        VSR_CUDA(cudaMalloc(&e.sep, (ld.m + ld.n + ld.s) * sizeof(double2)));
        if (!detect_separable(ld, reinterpret_cast<const double2*>(lam_loc), e.sep, e.sep + ld.m,
                              e.sep + ld.m + ld.n, 1e-13, st)) {
            VSR_CUDA(cudaFree(e.sep));
            e.sep = nullptr;
        }
    }
    cache.push_back(e);
    return cache.back();
}

}  // namespace

// Frees the cached fold tables of one context (vsr_ctx_destroy), or of one
// Lambda slice of it (lam_loc != nullptr; vsr_slab_tv_release_d, called when a
// slab ADMM-TV program is torn down).
namespace vsr_capi {
void release_slab_state(vsr_ctx* ctx, const double* lam_loc) {
    auto& cache = state_cache();
    std::lock_guard<std::mutex> lock(state_mutex());
    for (auto it = cache.begin(); it != cache.end();) {
        if (it->ctx == ctx && (lam_loc == nullptr || it->lam == lam_loc)) {
            free_state(*it);
            it = cache.erase(it);
        } else {
            ++it;
        }
    }
}
}  // namespace vsr_capi

extern "C" {

int vsr_fft3_d(vsr_ctx* ctx, const size_t dims[3], const double* in, int in_real, double* out_c,
               double scale) {
    return vsr_capi::guard_call([&] {
        DevGuard dg(vsr_capi::device_of(ctx));
        const Dims d{dims[0], dims[1], dims[2]};
        if (d.count() == 0) throw shape_error("fft3: empty volume");
        fft_engine().forward3(d, in, in_real ? IN_REAL : IN_COMPLEX, reinterpret_cast<double2*>(out_c), scale,
                              vsr_capi::stream_of(ctx));
    });
}

int vsr_slab_fwd_xy_pack_d(vsr_ctx* ctx, const size_t hr[3], const size_t rates[3], int P, const double* in,
                           int in_real, double* work_c, double* send_c) {
    return vsr_capi::guard_call([&] {
        DevGuard dg(vsr_capi::device_of(ctx));
        const Slab g = make_slab(hr, rates, P);
        cudaStream_t st = vsr_capi::stream_of(ctx);
        const Dims sd{(size_t)g.m, (size_t)g.n, (size_t)g.sz};
        auto* W = reinterpret_cast<double2*>(work_c);
        fft_engine().forward12(sd, in, in_real ? IN_REAL : IN_COMPLEX, W, st);
        pack_kernel<<<blocks(g.m * g.n * g.sz), 256, 0, st>>>(g, W, reinterpret_cast<double2*>(send_c));
        VSR_LAUNCH_CHECK();
    });
}

int vsr_slab_axis3_d(vsr_ctx* ctx, const size_t hr[3], const size_t rates[3], int P, double* W, int inverse,
                     double scale) {
    return vsr_capi::guard_call([&] {
        DevGuard dg(vsr_capi::device_of(ctx));
        const Slab g = make_slab(hr, rates, P);
        const Dims ld{(size_t)g.m, (size_t)g.nP, (size_t)g.s};
        fft_engine().axis_pass(ld, 2, inverse != 0, W, IN_COMPLEX, W, OUT_COMPLEX, scale, nullptr,
                               vsr_capi::stream_of(ctx));
    });
}

int vsr_slab_lr_slice_d(vsr_ctx* ctx, const size_t hr[3], const size_t rates[3], int P, int rank,
                        const double* Yl_full, double* Yl_loc) {
    return vsr_capi::guard_call([&] {
        DevGuard dg(vsr_capi::device_of(ctx));
        const Slab g = make_slab(hr, rates, P);
        lr_slice_kernel<<<blocks(g.ml * g.nlP * g.sl), 256, 0, vsr_capi::stream_of(ctx)>>>(
            g, rank, reinterpret_cast<const double2*>(Yl_full), reinterpret_cast<double2*>(Yl_loc));
        VSR_LAUNCH_CHECK();
    });
}

// Tikhonov fold on the local geometry + inverse axis-3 FFT -> W_out (local spectral layout)
int vsr_slab_tik_fold_d(vsr_ctx* ctx, const size_t hr[3], const size_t rates[3], int P, const double* Yl_loc,
                        const double* lam_loc, const double* xbh_loc, double reg, double* W_out) {
    return vsr_capi::guard_call([&] {
        DevGuard dg(vsr_capi::device_of(ctx));
        if (!(reg > 0.0)) throw std::invalid_argument("lambda must be positive, got " + std::to_string(reg));
        const Slab g = make_slab(hr, rates, P);
        const FoldGeom G = local_geom(g);
        cudaStream_t st = vsr_capi::stream_of(ctx);
        auto* out = reinterpret_cast<double2*>(W_out);
        const auto* Y = reinterpret_cast<const double2*>(Yl_loc);
        const auto* L = reinterpret_cast<const double2*>(lam_loc);
        const auto* X = reinterpret_cast<const double2*>(xbh_loc);
        if (fused_axis3_ok(G)) {
            launch_tik_fold_ifft3(G, Y, L, X, out, reg, st);
        } else {
            launch_tik_fold(G, Y, L, X, out, reg, st);
            const Dims ld{(size_t)g.m, (size_t)g.nP, (size_t)g.s};
            fft_engine().axis_pass(ld, 2, true, out, IN_COMPLEX, out, OUT_COMPLEX, 1.0, nullptr, st);
        }
    });
}


int vsr_slab_tv_release_d(vsr_ctx* ctx, const double* lam_loc) {
    return vsr_capi::guard_call([&] {
        DevGuard dg(vsr_capi::device_of(ctx));
        VSR_CUDA(cudaStreamSynchronize(vsr_capi::stream_of(ctx)));  // no queued fold still reads them
        vsr_capi::release_slab_state(ctx, lam_loc);
    });
}

// TV: forward axis-3 FFT (scaled) + fold + inverse axis-3 FFT in place on W;
// (Re)builds the rank's cached fold tables for the Lambda slice at lam_loc
// (call after computing it; a later fold with the same pointer reuses them).
int vsr_slab_tv_prepare_d(vsr_ctx* ctx, const size_t hr[3], const size_t rates[3], int P, int rank,
                          const double* lam_loc) {
    return vsr_capi::guard_call([&] {
        DevGuard dg(vsr_capi::device_of(ctx));
        const Slab g = make_slab(hr, rates, P);
        tv_fold_state(ctx, g, rank, lam_loc, local_geom(g), vsr_capi::stream_of(ctx), true);
    });
}

// fit_out (device double) receives this rank's share of ||y - D H x||^2.
int vsr_slab_tv_fold_d(vsr_ctx* ctx, const size_t hr[3], const size_t rates[3], int P, int rank,
                       const double* Yl_loc, const double* lam_loc, double* W, double mu, double tau,
                       double fwd_scale, double* fit_out) {
    return vsr_capi::guard_call([&] {
        DevGuard dg(vsr_capi::device_of(ctx));
        if (!(mu > 0.0)) throw std::invalid_argument("mu must be positive, got " + std::to_string(mu));
        if (!(tau > 0.0)) throw numeric_error(
            "make_gamma: difference-operator gram is singular at the zero frequency (DC); "
            "a positive tau floor is required");
        const Slab g = make_slab(hr, rates, P);
        const FoldGeom G = local_geom(g);
        cudaStream_t st = vsr_capi::stream_of(ctx);
        const TvFoldState& fs = tv_fold_state(ctx, g, rank, lam_loc, G, st);
        GammaTables tabs{fs.nr, fs.nc, fs.ns, tau};
        auto* Wc = reinterpret_cast<double2*>(W);
        const auto* Y = reinterpret_cast<const double2*>(Yl_loc);
        const auto* L = reinterpret_cast<const double2*>(lam_loc);
        const Dims ld{(size_t)g.m, (size_t)g.nP, (size_t)g.s};
        if (fused_axis3_ok(G)) {
            SepTables sep;
            if (fs.sep) sep = SepTables{fs.sep, fs.sep + ld.m, fs.sep + ld.m + ld.n};
            launch_tv_sandwich(G, Y, L, Wc, tabs, mu, fwd_scale, fs.fitp, st, sep);
        } else {
            fft_engine().axis_pass(ld, 2, false, Wc, IN_COMPLEX, Wc, OUT_COMPLEX, fwd_scale, nullptr, st);
            launch_tv_fold(G, Y, L, Wc, Wc, nullptr, tabs, mu, fs.fitp, st);
            fft_engine().axis_pass(ld, 2, true, Wc, IN_COMPLEX, Wc, OUT_COMPLEX, 1.0, nullptr, st);
        }
        sum_partials_kernel<<<1, 1024, 0, st>>>(fs.fitp, 1, 1, (long long)fs.nb, fit_out);
        VSR_LAUNCH_CHECK();
    });
}

// recv [q][z][jl][f1] -> slab [z][f2][f1] -> inverse axes 2, 1 -> out real slab (scaled);
// sums_out (device double[2]): sum imag^2, sum |z|^2; bad_out (device u64): min
// non-finite slab index (caller initialises to ULLONG_MAX).
int vsr_slab_unpack_inv_xy_d(vsr_ctx* ctx, const size_t hr[3], const size_t rates[3], int P,
                             const double* recv_c, double* work_c, double* out_real, double scale,
                             double* sums_out, unsigned long long* bad_out) {
    return vsr_capi::guard_call([&] {
        DevGuard dg(vsr_capi::device_of(ctx));
        const Slab g = make_slab(hr, rates, P);
        cudaStream_t st = vsr_capi::stream_of(ctx);
        auto* Wk = reinterpret_cast<double2*>(work_c);
        unpack_kernel<<<blocks(g.m * g.n * g.sz), 256, 0, st>>>(g, reinterpret_cast<const double2*>(recv_c), Wk);
        VSR_LAUNCH_CHECK();
        const Dims sd{(size_t)g.m, (size_t)g.n, (size_t)g.sz};
        const size_t nb = fft_engine().inverse_final_blocks(sd);
        double* part = nullptr;
        VSR_CUDA(cudaMallocAsync(&part, 2 * std::max<size_t>(nb, 1) * sizeof(double), st));
        PassReduce red{part, bad_out};
        fft_engine().inverse21(sd, Wk, out_real, OUT_REAL, scale, &red, st);
        sum_partials_kernel<<<1, 1024, 0, st>>>(part, 2, 2, (long long)nb, sums_out);
        VSR_LAUNCH_CHECK();
        cudaFreeAsync(part, st);
    });
}

// TV stencil on a slab with halo planes; sums_out (device double[4]):
// residual^2, TV, 0, 0 summed over this rank's voxels.
int vsr_slab_tv_stencil_d(vsr_ctx* ctx, const size_t hr[3], const size_t rates[3], int P, int init,
                          const double* x_ext, const double* dual_in_ext, double* dual_out_ext, double* theta,
                          double thr, double* sums_out) {
    return vsr_capi::guard_call([&] {
        DevGuard dg(vsr_capi::device_of(ctx));
        const Slab g = make_slab(hr, rates, P);
        cudaStream_t st = vsr_capi::stream_of(ctx);
        const Dims sd{(size_t)g.m, (size_t)g.n, (size_t)g.sz};
        const size_t nb = stencil_geom(sd).blocks();
        double* part = nullptr;
        VSR_CUDA(cudaMallocAsync(&part, kStencilVals * nb * sizeof(double), st));
        launch_tv_stencil_slab(sd, init != 0, x_ext, dual_in_ext, dual_out_ext, theta, thr, part, st);
        sum_partials_kernel<<<1, 1024, 0, st>>>(part, kStencilVals, kStencilVals, (long long)nb, sums_out);
        VSR_LAUNCH_CHECK();
        cudaFreeAsync(part, st);
    });
}

// Per-rank data-fit share for an arbitrary local spectrum (initial objective):
// Xh_loc = local spectral layout of fft3(x) (unitary).
int vsr_slab_fit_d(vsr_ctx* ctx, const size_t hr[3], const size_t rates[3], int P, const double* Yl_loc,
                   const double* lam_loc, const double* xh_loc, double* fit_out) {
    return vsr_capi::guard_call([&] {
        DevGuard dg(vsr_capi::device_of(ctx));
        const Slab g = make_slab(hr, rates, P);
        const FoldGeom G = local_geom(g);
        cudaStream_t st = vsr_capi::stream_of(ctx);
        const size_t nb = fit_blocks(G);
        double* part = nullptr;
        VSR_CUDA(cudaMallocAsync(&part, std::max<size_t>(nb, 1) * sizeof(double), st));
        launch_fit_partials(G, reinterpret_cast<const double2*>(Yl_loc), reinterpret_cast<const double2*>(lam_loc),
                            reinterpret_cast<const double2*>(xh_loc), part, st);
        sum_partials_kernel<<<1, 1024, 0, st>>>(part, 1, 1, (long long)nb, fit_out);
        VSR_LAUNCH_CHECK();
        cudaFreeAsync(part, st);
    });
}

}  // extern "C"
