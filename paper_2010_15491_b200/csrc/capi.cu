// C ABI of the volsr B200 path (include/vsr.h).  Host-side orchestration of
// the FFT engine (fft.cu), the spectral fold kernels (fold.cu) and the TV
// stencil (tv.cu); the reference behaviour each entry point reproduces is
// cited beside it.  Nothing here falls back to the CPU: every numeric step
// runs in a kernel on the context's device.
#include <atomic>
#include <random>
#include <thread>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <utility>
#include <vector>

#include "../../include/vsr.h"
#include "fft.cuh"
#include "fold.cuh"
#include "host_util.cuh"
#include "fused.cuh"
#include "spatial.cuh"
#include "l2l2.cuh"
#include "rfft.cuh"
#include "tv.cuh"

using namespace vsr;
using namespace vsr_host;

namespace vsr {
static std::atomic<uint64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// CUDA-event stage profiler owned by a context (see Profiler in vsr_common.cuh).
class EventProfiler : public Profiler {
public:
    struct Rec {
        std::string name;
        cudaEvent_t b, e;
    };
    void begin(const char* name, cudaStream_t st) override {
        Rec r{name, take(), take()};
        VSR_CUDA(cudaEventRecord(r.b, st));
        open_.push_back(r);
    }
    void end(cudaStream_t st) override {
        Rec r = open_.back();
        open_.pop_back();
        VSR_CUDA(cudaEventRecord(r.e, st));
        done_.push_back(r);
    }
    // aggregate (name -> total ms, count); recycles the events
    std::vector<std::pair<std::string, std::pair<double, uint64_t>>> drain() {
        std::vector<std::pair<std::string, std::pair<double, uint64_t>>> agg;
        for (auto& r : done_) {
            VSR_CUDA(cudaEventSynchronize(r.e));
            float ms = 0.f;
            VSR_CUDA(cudaEventElapsedTime(&ms, r.b, r.e));
            bool found = false;
            for (auto& a : agg)
                if (a.first == r.name) {
                    a.second.first += ms;
                    a.second.second += 1;
                    found = true;
                }
            if (!found) agg.push_back({r.name, {(double)ms, 1}});
            pool_.push_back(r.b);
            pool_.push_back(r.e);
        }
        done_.clear();
        return agg;
    }
    ~EventProfiler() override {
        for (auto& r : done_) {
            cudaEventDestroy(r.b);
            cudaEventDestroy(r.e);
        }
        for (auto e : pool_) cudaEventDestroy(e);
    }

private:
    cudaEvent_t take() {
        if (!pool_.empty()) {
            cudaEvent_t e = pool_.back();
            pool_.pop_back();
            return e;
        }
        cudaEvent_t e;
        VSR_CUDA(cudaEventCreate(&e));
        return e;
    }
    std::vector<Rec> open_, done_;
    std::vector<cudaEvent_t> pool_;
};
}  // namespace vsr

// ============================================================ errors / state
namespace {

thread_local std::string g_last_error;
std::atomic<uint64_t> g_fwd{0}, g_inv{0};  // reference src/fft.cpp:15-16

template <class F>
int guarded(F&& f) {
    try {
        f();
        return VSR_OK;
    } catch (const vsr::shape_error& e) {
        g_last_error = e.what();
        return VSR_ERR_SHAPE;
    } catch (const vsr::numeric_error& e) {
        g_last_error = e.what();
        return VSR_ERR_NUMERIC;
    } catch (const std::out_of_range& e) {
        g_last_error = e.what();
        return VSR_ERR_OUT_OF_RANGE;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return VSR_ERR_INVALID;
    } catch (const vsr::cuda_error& e) {
        g_last_error = e.what();
        return VSR_ERR_CUDA;
    } catch (const vsr::io_error& e) {
        g_last_error = e.what();
        return VSR_ERR_IO;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return VSR_ERR_INTERNAL;
    } catch (...) {
        g_last_error = "unknown error";
        return VSR_ERR_INTERNAL;
    }
}

std::string residue_message(double ratio, double max_rel_imag) {  // src/fft.cpp:90-93
    return "ifft3_real: imaginary residue " + std::to_string(ratio) + " exceeds " +
           std::to_string(max_rel_imag) + " (spectral bookkeeping bug?)";
}

// ---- small kernels local to the ABI layer
__global__ void residue_status_kernel(const double* __restrict__ partials, long long nblocks,
                                      double tol, double* __restrict__ status) {
    __shared__ double red[64];
    double v[2] = {0.0, 0.0};
    for (long long i = threadIdx.x; i < nblocks; i += blockDim.x) {
        v[0] += partials[2 * i];
        v[1] += partials[2 * i + 1];
    }
    block_reduce_sum<2>(v, red);
    if (threadIdx.x == 0) {
        const double ratio = v[1] > 0.0 ? sqrt(v[0] / v[1]) : 0.0;
        status[2] = ratio;
        if (v[1] > 0.0 && ratio > tol && status[0] == 0.0) {
            status[0] = 1.0;
            status[1] = ratio;
        }
    }
}

// 1 if any entry of x off the decimation lattice (i % dr, j % dc, k % ds not all 0) is non-zero
__global__ void off_lattice_kernel(long long m, long long n, long long N, int dr, int dc, int ds,
                                   const double* __restrict__ x, int* __restrict__ flag) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= N) return;
    const long long i = p % m, j = (p / m) % n, k = p / (m * n);
    if ((i % dr || j % dc || k % ds) && x[p] != 0.0) *flag = 1;
}

// degrade (sim.cpp:106-127): per-block sums of y, then of (y - mean)^2
__global__ void __launch_bounds__(256) blocksum_kernel(const double* __restrict__ y, long long n,
                                                       const double* __restrict__ mean, double* __restrict__ partials) {
    __shared__ double red[32];
    double v[1] = {0.0};
    const double mu = mean ? *mean : 0.0;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
        const double t = y[i] - mu;
        v[0] += mean ? t * t : y[i];
    }
    block_reduce_sum<1>(v, red);
    if (threadIdx.x == 0) partials[blockIdx.x] = v[0];
}
__global__ void add_noise_kernel(double* __restrict__ y, const double* __restrict__ noise, long long n, double sigma,
                                 unsigned long long* __restrict__ bad) {
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)gridDim.x * 256) {
        const double v = noise ? y[i] + sigma * noise[i] : y[i];
        y[i] = v;
        if (!isfinite(v)) atomicMin(bad, (unsigned long long)i);
    }
}

// nn_upsample (operators.cpp:155-164): x[i,j,k] = y[i/dr, j/dc, k/ds]
__global__ void nn_upsample_kernel(long long m, long long n, long long N, int dr, int dc, int ds, long long ml,
                                   long long nl, const double* __restrict__ y, double* __restrict__ x) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= N) return;
    const long long i = p % m, j = (p / m) % n, k = p / (m * n);
    x[p] = y[(i / dr) + ml * ((j / dc) + nl * (k / ds))];
}

// finite_diff_spectra (operators.cpp:225-243): (cos(2 pi f/len) - 1, sin(2 pi f/len)),
// exactly 0 at f = 0, per axis over the whole HR grid
__global__ void diff_spectra_kernel(long long m, long long n, long long N, long long s, double2* __restrict__ rows,
                                    double2* __restrict__ cols, double2* __restrict__ slices) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= N) return;
    const long long f[3] = {p % m, (p / m) % n, p / (m * n)};
    const long long len[3] = {m, n, s};
    double2* out[3] = {rows, cols, slices};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double2 v = make_double2(0.0, 0.0);
        if (f[a] != 0) {
            const double ang = 6.283185307179586 * (double)f[a] / (double)len[a];  // 2 * std::numbers::pi
            v = make_double2(cos(ang) - 1.0, sin(ang));
        }
        out[a][p] = v;
    }
}

// make_gamma (solvers.cpp:191-205) from three given difference spectra:
// gamma = 1 / (|r|^2 + |c|^2 + |s|^2 + tau); the first non-positive
// denominator's index goes to *bad (atomicMin)
__global__ void gamma_spectra_kernel(long long N, const double2* __restrict__ r, const double2* __restrict__ c,
                                     const double2* __restrict__ s, double tau, double* __restrict__ g,
                                     unsigned long long* __restrict__ bad) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= N) return;
    const double2 a = r[p], b = c[p], e = s[p];
    const double den = (((a.x * a.x + a.y * a.y) + (b.x * b.x + b.y * b.y)) + (e.x * e.x + e.y * e.y)) + tau;
    if (!(den > 0.0)) atomicMin(bad, (unsigned long long)p);
    g[p] = 1.0 / den;
}

__global__ void scale_kernel(double* v, double s) { *v *= s; }
__global__ void narrow_f64_kernel(const double* __restrict__ in, float* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = (float)in[i];
}
__global__ void widen_f32_kernel(const float* __restrict__ in, double* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = (double)in[i];
}
__global__ void cmul_kernel(long long n, double2* __restrict__ a, const double2* __restrict__ b,
                            bool conj_b) {
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const double2 bb = conj_b ? make_double2(b[p].x, -b[p].y) : b[p];
    a[p] = cmul(a[p], bb);  // operators.cpp:129 xh[p] *= lambda[p]
}

void launch_narrow(const double* in, float* out, size_t n, cudaStream_t st) {
    if (!n) return;
    const unsigned b = (unsigned)std::min<size_t>((n + 255) / 256, 148 * 16);
    narrow_f64_kernel<<<b, 256, 0, st>>>(in, out, (long long)n);
    VSR_LAUNCH_CHECK();
}
void launch_widen(const float* in, double* out, size_t n, cudaStream_t st) {
    if (!n) return;
    const unsigned b = (unsigned)std::min<size_t>((n + 255) / 256, 148 * 16);
    widen_f32_kernel<<<b, 256, 0, st>>>(in, out, (long long)n);
    VSR_LAUNCH_CHECK();
}

}  // namespace

// ============================================================ context
struct vsr_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    DevBuf<double> scal;                // 8 doubles: [0..3] residue status
    DevBuf<unsigned long long> bad;     // non-finite index slot
    EventProfiler profiler;
    bool profiling = false;
    Profiler* prof() { return profiling ? &profiler : nullptr; }
    struct Guard {
        int prev = 0;
        explicit Guard(int dev) {
            cudaGetDevice(&prev);
            if (prev != dev) VSR_CUDA(cudaSetDevice(dev));
        }
        ~Guard() {
            int cur = 0;
            cudaGetDevice(&cur);
            if (cur != prev) cudaSetDevice(prev);
        }
    };
};

namespace {

// Run an ifft3_real-style final-pass reduction check synchronously.
struct ResidueCheck {
    DevBuf<double> partials;
    size_t blocks = 0;
    PassReduce red;
    ResidueCheck(vsr_ctx* ctx, const Dims& d) {
        blocks = fft_engine().inverse_final_blocks(d);
        partials.alloc(2 * std::max<size_t>(blocks, 1));
        red.partials = partials.p;
        red.bad_index = ctx->bad.p;
        VSR_CUDA(cudaMemsetAsync(ctx->scal.p, 0, 8 * sizeof(double), ctx->stream));
        VSR_CUDA(cudaMemsetAsync(ctx->bad.p, 0xff, sizeof(unsigned long long), ctx->stream));
    }
    // returns (violated, ratio) and the non-finite index (ULLONG_MAX = none)
    void finish(vsr_ctx* ctx, double tol, double* status_out, unsigned long long* bad_out) {
        residue_status_kernel<<<1, 1024, 0, ctx->stream>>>(partials.p, (long long)blocks, tol,
                                                           ctx->scal.p);
        VSR_LAUNCH_CHECK();
        VSR_CUDA(cudaMemcpyAsync(status_out, ctx->scal.p, 4 * sizeof(double),
                                 cudaMemcpyDeviceToHost, ctx->stream));
        VSR_CUDA(cudaMemcpyAsync(bad_out, ctx->bad.p, sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, ctx->stream));
        VSR_CUDA(cudaStreamSynchronize(ctx->stream));
    }
};

void h2d(vsr_ctx* ctx, void* dst, const void* src, size_t bytes) {
    if (bytes) VSR_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
}
void d2h(vsr_ctx* ctx, void* dst, const void* src, size_t bytes) {
    if (bytes) VSR_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
}
void sync(vsr_ctx* ctx) { VSR_CUDA(cudaStreamSynchronize(ctx->stream)); }

void require_ctx(vsr_ctx* ctx) {
    if (!ctx) throw std::invalid_argument("vsr: null context");
}

double inv_sqrt_count(const Dims& d) { return 1.0 / std::sqrt((double)d.count()); }

// Which pass the fold is fused with: 1 (contiguous rows), 3 (strided lines) or
// 0 (none).  Measured at 256^3 (r01): Tikhonov fold+axis3 220 us vs
// fold+axis1 285 us; TV sandwich on axis 1 358 us vs axis 3 470 us.  So the
// default is axis 3 for Tikhonov and axis 1 for TV (VSR_FUSE_AXIS overrides).
int fuse_axis(const FoldGeom& G, int dflt) {
    static const int env = [] {
        const char* e = std::getenv("VSR_FUSE_AXIS");
        return e ? std::atoi(e) : -1;
    }();
    const int pref = env >= 0 ? env : dflt;
    static const bool off = [] {
        const char* e = std::getenv("VSR_NO_FUSE");
        return e && e[0] == '1';
    }();
    if (off || pref == 0) return 0;
    if (pref == 1 && fused_axis1_ok(G)) return 1;
    if (fused_axis3_ok(G)) return 3;
    if (fused_axis1_ok(G)) return 1;
    return 0;
}

// Separable-spectrum tables (fold.cuh SepTables); VSR_NO_SEP=1 disables.
struct SepState {
    DevBuf<double2> tab;  // a[m], b[n], c[s]
    SepTables t;
    void detect(const Dims& hr, const double2* lam, cudaStream_t st) {
        static const bool off = [] {
            const char* e = std::getenv("VSR_NO_SEP");
            return e && e[0] == '1';
        }();
        t = SepTables{};
        if (off) return;
        tab.alloc(hr.m + hr.n + hr.s);
        if (detect_separable(hr, lam, tab.p, tab.p + hr.m, tab.p + hr.m + hr.n, 1e-13, st))
            t = SepTables{tab.p, tab.p + hr.m, tab.p + hr.m + hr.n};
        else
            tab.release();
    }
};

bool use_fused(const FoldGeom& G) {
    static const bool off = [] {
        const char* e = std::getenv("VSR_NO_FUSE");
        return e && e[0] == '1';
    }();
    return !off && fused_axis3_ok(G);
}

}  // namespace

// hooks for the other C-ABI translation units (slab.cu, volio.cu)
namespace vsr_capi {
cudaStream_t stream_of(vsr_ctx* ctx) {
    if (!ctx) throw std::invalid_argument("vsr: null context");
    return ctx->stream;
}
int device_of(vsr_ctx* ctx) {
    if (!ctx) throw std::invalid_argument("vsr: null context");
    return ctx->device;
}
int guard_call(const std::function<void()>& f) { return guarded(f); }
void add_fft_counts(uint64_t forward, uint64_t inverse) {  // fft_counters (src/fft.cpp:103-111)
    g_fwd += forward;
    g_inv += inverse;
}
}  // namespace vsr_capi

extern "C" {

const char* vsr_last_error_message(void) { return g_last_error.c_str(); }
int vsr_version(void) { return 1; }

int vsr_ctx_create(int device, vsr_ctx** out) {
    return guarded([&] {
        if (!out) throw std::invalid_argument("vsr_ctx_create: null out");
        int ndev = 0;
        VSR_CUDA(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev)
            throw std::invalid_argument("vsr_ctx_create: device " + std::to_string(device) +
                                        " not present (" + std::to_string(ndev) + " devices)");
        auto* c = new vsr_ctx();
        c->device = device;
        vsr_ctx::Guard g(device);
        VSR_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        c->scal.alloc(8);
        c->bad.alloc(1);
        *out = c;
    });
}

int vsr_ctx_destroy(vsr_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        vsr_ctx::Guard g(ctx->device);
        cudaStreamSynchronize(ctx->stream);
        ctx->scal.release();
        ctx->bad.release();
        cudaStreamDestroy(ctx->stream);
        delete ctx;
    });
}

int vsr_ctx_synchronize(vsr_ctx* ctx) {
    return guarded([&] {
        require_ctx(ctx);
        sync(ctx);
    });
}

void* vsr_ctx_stream(vsr_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }
int vsr_ctx_device(vsr_ctx* ctx) { return ctx ? ctx->device : -1; }

int vsr_host_alloc(size_t bytes, void** out) {
    return guarded([&] { VSR_CUDA(cudaHostAlloc(out, bytes, cudaHostAllocDefault)); });
}
int vsr_host_free(void* p) {
    return guarded([&] { VSR_CUDA(cudaFreeHost(p)); });
}
int vsr_device_alloc(vsr_ctx* ctx, size_t bytes, void** out) {
    return guarded([&] {
        require_ctx(ctx);
        vsr_ctx::Guard g(ctx->device);
        VSR_CUDA(cudaMalloc(out, bytes));
    });
}
int vsr_device_free(vsr_ctx* ctx, void* p) {
    return guarded([&] {
        require_ctx(ctx);
        vsr_ctx::Guard g(ctx->device);
        VSR_CUDA(cudaFree(p));
    });
}
int vsr_memcpy_h2d(vsr_ctx* ctx, void* dst, const void* src, size_t bytes) {
    return guarded([&] {
        require_ctx(ctx);
        vsr_ctx::Guard g(ctx->device);
        h2d(ctx, dst, src, bytes);
        sync(ctx);
    });
}
int vsr_memcpy_d2h(vsr_ctx* ctx, void* dst, const void* src, size_t bytes) {
    return guarded([&] {
        require_ctx(ctx);
        vsr_ctx::Guard g(ctx->device);
        d2h(ctx, dst, src, bytes);
        sync(ctx);
    });
}

// ============================================================ FFT contract
// src/fft.cpp:66-101
static void fft_host(vsr_ctx* ctx, const size_t dims[3], const void* in, bool real_in, double* out,
                     double scale_override) {
    require_ctx(ctx);
    const Dims d = to_dims(dims);
    require_nonempty(d, "fft3");
    vsr_ctx::Guard g(ctx->device);
    DevBuf<double2> buf(d.count());
    DevBuf<double> rin;
    if (real_in) {
        rin.alloc(d.count());
        h2d(ctx, rin.p, in, rin.bytes());
        fft_engine().forward3(d, rin.p, IN_REAL, buf.p, scale_override, ctx->stream);
    } else {
        h2d(ctx, buf.p, in, buf.bytes());
        fft_engine().forward3(d, buf.p, IN_COMPLEX, buf.p, scale_override, ctx->stream);
    }
    ++g_fwd;
    d2h(ctx, out, buf.p, buf.bytes());
    sync(ctx);
}

int vsr_fft3(vsr_ctx* ctx, const size_t dims[3], const double* in_c, double* out_c) {
    return guarded([&] { fft_host(ctx, dims, in_c, false, out_c, inv_sqrt_count(to_dims(dims))); });
}
int vsr_fft3_real(vsr_ctx* ctx, const size_t dims[3], const double* in_r, double* out_c) {
    return guarded([&] { fft_host(ctx, dims, in_r, true, out_c, inv_sqrt_count(to_dims(dims))); });
}
int vsr_dft3_unnormalized(vsr_ctx* ctx, const size_t dims[3], const double* in_r, double* out_c) {
    return guarded([&] { fft_host(ctx, dims, in_r, true, out_c, 1.0); });
}
int vsr_psf_to_spectrum(vsr_ctx* ctx, const size_t dims[3], const double* psf_r, double* lambda_c) {
    return vsr_dft3_unnormalized(ctx, dims, psf_r, lambda_c);
}

int vsr_ifft3(vsr_ctx* ctx, const size_t dims[3], const double* in_c, double* out_c) {
    return guarded([&] {
        require_ctx(ctx);
        const Dims d = to_dims(dims);
        require_nonempty(d, "fft3");
        vsr_ctx::Guard g(ctx->device);
        DevBuf<double2> buf(d.count());
        h2d(ctx, buf.p, in_c, buf.bytes());
        fft_engine().inverse3(d, buf.p, buf.p, OUT_COMPLEX, inv_sqrt_count(d), nullptr, ctx->stream);
        ++g_inv;
        d2h(ctx, out_c, buf.p, buf.bytes());
        sync(ctx);
    });
}

int vsr_ifft3_real(vsr_ctx* ctx, const size_t dims[3], const double* in_c, double* out_r,
                   double max_rel_imag) {
    return guarded([&] {
        require_ctx(ctx);
        const Dims d = to_dims(dims);
        require_nonempty(d, "fft3");
        vsr_ctx::Guard g(ctx->device);
        DevBuf<double2> buf(d.count());
        DevBuf<double> xr(d.count());
        h2d(ctx, buf.p, in_c, buf.bytes());
        ResidueCheck rc(ctx, d);
        fft_engine().inverse3(d, buf.p, xr.p, OUT_REAL, inv_sqrt_count(d), &rc.red, ctx->stream);
        ++g_inv;
        double status[4];
        unsigned long long bad;
        rc.finish(ctx, max_rel_imag, status, &bad);
        if (status[0] != 0.0) throw numeric_error(residue_message(status[1], max_rel_imag));
        d2h(ctx, out_r, xr.p, xr.bytes());
        sync(ctx);
    });
}

int vsr_fft_counters(uint64_t* forward, uint64_t* inverse) {
    if (forward) *forward = g_fwd.load(std::memory_order_relaxed);
    if (inverse) *inverse = g_inv.load(std::memory_order_relaxed);
    return VSR_OK;
}
int vsr_reset_fft_counters(void) {
    g_fwd.store(0);
    g_inv.store(0);
    return VSR_OK;
}

// ============================================================ operators
int vsr_decimate(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3], const double* x,
                 double* y) {
    return guarded([&] {
        require_ctx(ctx);
        const Spec sp = make_spec(hr_dims, rates);
        vsr_ctx::Guard g(ctx->device);
        DevBuf<double> dx(sp.hr.count()), dy(sp.lr.count());
        h2d(ctx, dx.p, x, dx.bytes());
        launch_decimate(sp.hr, sp.rates, dx.p, dy.p, ctx->stream);
        d2h(ctx, y, dy.p, dy.bytes());
        sync(ctx);
    });
}

int vsr_decimate_adjoint(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3],
                         const double* y, double* x) {
    return guarded([&] {
        require_ctx(ctx);
        const Spec sp = make_spec(hr_dims, rates);
        vsr_ctx::Guard g(ctx->device);
        DevBuf<double> dx(sp.hr.count()), dy(sp.lr.count());
        h2d(ctx, dy.p, y, dy.bytes());
        launch_decimate_adjoint(sp.hr, sp.rates, dy.p, dx.p, 1.0, ctx->stream);
        d2h(ctx, x, dx.p, dx.bytes());
        sync(ctx);
    });
}

int vsr_nn_upsample(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3], const double* y, double* x) {
    return guarded([&] {
        require_ctx(ctx);
        const Spec sp = make_spec(hr_dims, rates);
        vsr_ctx::Guard g(ctx->device);
        DevBuf<double> dx(sp.hr.count()), dy(sp.lr.count());
        h2d(ctx, dy.p, y, dy.bytes());
        const long long N = (long long)sp.hr.count();
        if (N) {
            nn_upsample_kernel<<<(unsigned)((N + 255) / 256), 256, 0, ctx->stream>>>(
                (long long)sp.hr.m, (long long)sp.hr.n, N, sp.rates[0], sp.rates[1], sp.rates[2],
                (long long)sp.lr.m, (long long)sp.lr.n, dy.p, dx.p);
            VSR_LAUNCH_CHECK();
        }
        d2h(ctx, x, dx.p, dx.bytes());
        sync(ctx);
    });
}

int vsr_finite_diff_spectra(vsr_ctx* ctx, const size_t hr_dims[3], double* rows_c, double* cols_c,
                            double* slices_c) {
    return guarded([&] {
        require_ctx(ctx);
        const Dims d = to_dims(hr_dims);
        vsr_ctx::Guard g(ctx->device);
        const long long N = (long long)d.count();
        DevBuf<double2> r(d.count()), c(d.count()), z(d.count());
        if (N) {
            diff_spectra_kernel<<<(unsigned)((N + 255) / 256), 256, 0, ctx->stream>>>(
                (long long)d.m, (long long)d.n, N, (long long)d.s, r.p, c.p, z.p);
            VSR_LAUNCH_CHECK();
        }
        d2h(ctx, rows_c, r.p, r.bytes());
        d2h(ctx, cols_c, c.p, c.bytes());
        d2h(ctx, slices_c, z.p, z.bytes());
        sync(ctx);
    });
}

int vsr_make_gamma_spectra(vsr_ctx* ctx, const size_t hr_dims[3], const double* rows_c, const double* cols_c,
                           const double* slices_c, double tau, double* gamma_r) {
    return guarded([&] {
        require_ctx(ctx);
        if (tau < 0.0) throw std::invalid_argument("make_gamma: tau must be nonnegative");  // solvers.cpp:192
        const Dims d = to_dims(hr_dims);
        vsr_ctx::Guard g(ctx->device);
        const long long N = (long long)d.count();
        DevBuf<double2> r(d.count()), c(d.count()), z(d.count());
        DevBuf<double> out(d.count());
        h2d(ctx, r.p, rows_c, r.bytes());
        h2d(ctx, c.p, cols_c, c.bytes());
        h2d(ctx, z.p, slices_c, z.bytes());
        VSR_CUDA(cudaMemsetAsync(ctx->bad.p, 0xff, sizeof(unsigned long long), ctx->stream));
        if (N) {
            gamma_spectra_kernel<<<(unsigned)((N + 255) / 256), 256, 0, ctx->stream>>>(N, r.p, c.p, z.p, tau, out.p,
                                                                                      ctx->bad.p);
            VSR_LAUNCH_CHECK();
        }
        unsigned long long bad = 0;
        d2h(ctx, &bad, ctx->bad.p, sizeof(bad));
        sync(ctx);
        if (bad != ULLONG_MAX)
            throw numeric_error(
                "make_gamma: difference-operator gram is singular at the zero frequency (DC); "
                "a positive tau floor is required");
        d2h(ctx, gamma_r, out.p, out.bytes());
        sync(ctx);
    });
}

static int diff_host(vsr_ctx* ctx, const size_t dims[3], int axis, const double* x, double* out,
                     bool adjoint) {
    return guarded([&] {
        require_ctx(ctx);
        const Dims d = to_dims(dims);
        if (axis < 0 || axis > 2) throw std::invalid_argument("diff: axis must be 0, 1 or 2");
        vsr_ctx::Guard g(ctx->device);
        DevBuf<double> dx(d.count()), dout(d.count());
        h2d(ctx, dx.p, x, dx.bytes());
        launch_diff(d, axis, adjoint, dx.p, dout.p, ctx->stream);
        d2h(ctx, out, dout.p, dout.bytes());
        sync(ctx);
    });
}
int vsr_diff_forward(vsr_ctx* ctx, const size_t dims[3], int axis, const double* x, double* out) {
    return diff_host(ctx, dims, axis, x, out, false);
}
int vsr_diff_adjoint(vsr_ctx* ctx, const size_t dims[3], int axis, const double* x, double* out) {
    return diff_host(ctx, dims, axis, x, out, true);
}

int vsr_blur_apply(vsr_ctx* ctx, const size_t dims[3], const double* x, const double* lambda_c,
                   int conjugate, double* out) {
    return guarded([&] {
        require_ctx(ctx);
        const Dims d = to_dims(dims);
        require_nonempty(d, "fft3");
        vsr_ctx::Guard g(ctx->device);
        DevBuf<double> dx(d.count());
        DevBuf<double2> W(d.count()), lam(d.count());
        h2d(ctx, dx.p, x, dx.bytes());
        h2d(ctx, lam.p, lambda_c, lam.bytes());
        fft_engine().forward3(d, dx.p, IN_REAL, W.p, inv_sqrt_count(d), ctx->stream);
        ++g_fwd;
        cmul_kernel<<<(unsigned)((d.count() + 255) / 256), 256, 0, ctx->stream>>>(
            (long long)d.count(), W.p, lam.p, conjugate != 0);
        VSR_LAUNCH_CHECK();
        ResidueCheck rc(ctx, d);
        fft_engine().inverse3(d, W.p, dx.p, OUT_REAL, inv_sqrt_count(d), &rc.red, ctx->stream);
        ++g_inv;
        double status[4];
        unsigned long long bad;
        rc.finish(ctx, 1e-8, status, &bad);
        if (status[0] != 0.0) throw numeric_error(residue_message(status[1], 1e-8));
        d2h(ctx, out, dx.p, dx.bytes());
        sync(ctx);
    });
}

// ============================================================ degrade (input synthesis)
namespace {
// sim.cpp:88-104 gaussian_noise: the reference's sequential mt19937_64 +
// Box-Muller stream, (u1, u2) = ((r >> 11) + 1) * 2^-53 per draw (host: the
// generator is inherently serial; it runs on a host thread while the device
// blurs and decimates)
void gaussian_noise_host(size_t n, uint64_t seed, double* out) {
    std::mt19937_64 rng(seed);
    auto uniform = [&rng]() { return (static_cast<double>(rng() >> 11) + 1.0) * 0x1p-53; };
    constexpr double two_pi = 2.0 * 3.141592653589793;  // 2 * std::numbers::pi
    for (size_t p = 0; p < n; p += 2) {
        const double u1 = uniform();
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        out[p] = r * std::cos(two_pi * u2);
        if (p + 1 < n) out[p + 1] = r * std::sin(two_pi * u2);
    }
}
}  // namespace

// degrade (sim.cpp:106-127): y = decimate(blur_apply(x, Lambda(psf))) + sigma n,
// sigma^2 = var(y) / 10^(bsnr/10) over the mean-removed noiseless y.  The
// blur-and-decimate runs as ONE HR forward transform, the alias fold of
// Lambda X (F_l(D v)[g] = d^-1/2 sum_b F(v)[g + b lr]) and ONE LR inverse.
int vsr_degrade(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3], const double* x, const double* psf,
                int has_bsnr, double bsnr_db, uint64_t seed, double* y_out, double* sigma_out) {
    return guarded([&] {
        require_ctx(ctx);
        const Spec sp = make_spec(hr_dims, rates);
        vsr_ctx::Guard g(ctx->device);
        cudaStream_t st = ctx->stream;
        const long long Nl = (long long)sp.lr.count();
        std::vector<double> noise;
        std::thread gen;
        if (has_bsnr) {
            noise.resize((size_t)Nl);
            gen = std::thread([&] { gaussian_noise_host((size_t)Nl, seed, noise.data()); });
        }
        struct Join {
            std::thread& t;
            ~Join() {
                if (t.joinable()) t.join();
            }
        } join{gen};
        const FoldGeom G = make_geom(sp.hr, sp.rates);
        DevBuf<double> dx(sp.hr.count()), y(sp.lr.count());
        DevBuf<double2> X(sp.hr.count()), lam(sp.hr.count()), Yl(sp.lr.count());
        h2d(ctx, dx.p, psf, dx.bytes());
        fft_engine().forward3(sp.hr, dx.p, IN_REAL, lam.p, 1.0, st);  // Lambda: unnormalised DFT (operators.cpp:121-123)
        h2d(ctx, dx.p, x, dx.bytes());
        fft_engine().forward3(sp.hr, dx.p, IN_REAL, X.p, inv_sqrt_count(sp.hr), st);
        g_fwd += 2;
        launch_fold_apply(G, lam.p, nullptr, X.p, Yl.p, st);  // sum_b Lambda_b X_b
        ResidueCheck rc(ctx, sp.lr);
        fft_engine().inverse3(sp.lr, Yl.p, y.p, OUT_REAL, inv_sqrt_count(sp.lr) / std::sqrt((double)sp.rate()), &rc.red,
                              st);
        ++g_inv;
        double status[4];
        unsigned long long bad;
        rc.finish(ctx, 1e-8, status, &bad);
        if (status[0] != 0.0) throw numeric_error(residue_message(status[1], 1e-8));
        double sigma = 0.0;
        DevBuf<double> nz;
        if (has_bsnr) {
            const unsigned nb = (unsigned)std::min<long long>((Nl + 255) / 256, 148LL * 8);
            DevBuf<double> part(nb), mv(2);
            blocksum_kernel<<<nb, 256, 0, st>>>(y.p, Nl, nullptr, part.p);
            VSR_LAUNCH_CHECK();
            launch_finalize_sum(part.p, 1, 1, nb, mv.p, st);
            scale_kernel<<<1, 1, 0, st>>>(mv.p, 1.0 / (double)Nl);
            VSR_LAUNCH_CHECK();
            blocksum_kernel<<<nb, 256, 0, st>>>(y.p, Nl, mv.p, part.p);
            VSR_LAUNCH_CHECK();
            launch_finalize_sum(part.p, 1, 1, nb, mv.p + 1, st);
            double h[2];
            d2h(ctx, h, mv.p, sizeof(h));
            sync(ctx);
            const double var = h[1] / (double)Nl;
            sigma = std::sqrt(var / std::pow(10.0, bsnr_db / 10.0));
            gen.join();
            nz.alloc((size_t)Nl);
            h2d(ctx, nz.p, noise.data(), nz.bytes());
        }
        VSR_CUDA(cudaMemsetAsync(ctx->bad.p, 0xff, sizeof(unsigned long long), st));
        add_noise_kernel<<<(unsigned)std::min<long long>((Nl + 255) / 256, 148LL * 16), 256, 0, st>>>(
            y.p, has_bsnr ? nz.p : nullptr, Nl, sigma, ctx->bad.p);
        VSR_LAUNCH_CHECK();
        d2h(ctx, &bad, ctx->bad.p, sizeof(bad));
        d2h(ctx, y_out, y.p, y.bytes());
        sync(ctx);
        if (bad != ULLONG_MAX) throw numeric_error("degrade: non-finite value at flat index " + std::to_string(bad));
        if (sigma_out) *sigma_out = sigma;
    });
}

// ============================================================ spectral fold
int vsr_alias_fold(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3],
                   const double* hr_c, double* lr_c) {
    return guarded([&] {
        require_ctx(ctx);
        const Spec sp = make_spec(hr_dims, rates);
        vsr_ctx::Guard g(ctx->device);
        const FoldGeom G = make_geom(sp.hr, sp.rates);
        DevBuf<double2> hi(sp.hr.count()), lo(sp.lr.count());
        h2d(ctx, hi.p, hr_c, hi.bytes());
        launch_fold_apply(G, nullptr, nullptr, hi.p, lo.p, ctx->stream);
        d2h(ctx, lr_c, lo.p, lo.bytes());
        sync(ctx);
    });
}

int vsr_alias_expand(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3],
                     const double* lr_c, double* hr_c) {
    return guarded([&] {
        require_ctx(ctx);
        const Spec sp = make_spec(hr_dims, rates);
        vsr_ctx::Guard g(ctx->device);
        const FoldGeom G = make_geom(sp.hr, sp.rates);
        DevBuf<double2> hi(sp.hr.count()), lo(sp.lr.count());
        h2d(ctx, lo.p, lr_c, lo.bytes());
        launch_fold_adjoint(G, nullptr, nullptr, lo.p, hi.p, ctx->stream);
        d2h(ctx, hr_c, hi.p, hi.bytes());
        sync(ctx);
    });
}

struct vsr_folded {
    vsr_ctx* ctx;
    Spec sp;
    FoldGeom G;
    DevBuf<double2> lam;
};

int vsr_folded_create(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3],
                      const double* lambda_c, vsr_folded** out) {
    return guarded([&] {
        require_ctx(ctx);
        const Spec sp = make_spec(hr_dims, rates);
        vsr_ctx::Guard g(ctx->device);
        auto* f = new vsr_folded();
        f->ctx = ctx;
        f->sp = sp;
        f->G = make_geom(sp.hr, sp.rates);
        f->lam.alloc(sp.hr.count());
        h2d(ctx, f->lam.p, lambda_c, f->lam.bytes());
        sync(ctx);
        *out = f;
    });
}

// an independent copy (FoldedSpectrum is a value type in the reference)
int vsr_folded_clone(const vsr_folded* src, vsr_folded** out) {
    return guarded([&] {
        if (!src || !out) throw std::invalid_argument("vsr_folded_clone: null handle");
        vsr_ctx::Guard g(src->ctx->device);
        auto* f = new vsr_folded();
        f->ctx = src->ctx;
        f->sp = src->sp;
        f->G = src->G;
        f->lam.alloc(src->sp.hr.count());
        VSR_CUDA(cudaMemcpyAsync(f->lam.p, src->lam.p, f->lam.bytes(), cudaMemcpyDeviceToDevice, src->ctx->stream));
        sync(src->ctx);
        *out = f;
    });
}

int vsr_folded_destroy(vsr_folded* f) {
    return guarded([&] {
        if (!f) return;
        vsr_ctx::Guard g(f->ctx->device);
        delete f;
    });
}

int vsr_folded_block_value(vsr_folded* f, size_t br, size_t bc, size_t bs, size_t gi,
                           double out_c[2]) {
    return guarded([&] {
        if (br >= (size_t)f->sp.rates[0] || bc >= (size_t)f->sp.rates[1] ||
            bs >= (size_t)f->sp.rates[2] || gi >= f->sp.lr.count())
            throw std::out_of_range("FoldedSpectrum::block_value: block offset out of range");
        vsr_ctx::Guard g(f->ctx->device);
        const Dims& lr = f->sp.lr;
        const size_t g1 = gi % lr.m, g2 = (gi / lr.m) % lr.n, g3 = gi / (lr.m * lr.n);
        const size_t hr = (g1 + br * lr.m) + f->sp.hr.m * ((g2 + bc * lr.n) + f->sp.hr.n * (g3 + bs * lr.s));
        d2h(f->ctx, out_c, f->lam.p + hr, sizeof(double2));
        sync(f->ctx);
    });
}

static int folded_apply_host(vsr_folded* f, const double* in_c, const double* w, double* out_c,
                             bool adjoint) {
    return guarded([&] {
        vsr_ctx* ctx = f->ctx;
        vsr_ctx::Guard g(ctx->device);
        DevBuf<double2> hi(f->sp.hr.count()), lo(f->sp.lr.count());
        DevBuf<double> dw;
        if (w) {
            dw.alloc(f->sp.hr.count());
            h2d(ctx, dw.p, w, dw.bytes());
        }
        if (!adjoint) {
            h2d(ctx, hi.p, in_c, hi.bytes());
            launch_fold_apply(f->G, f->lam.p, dw.p, hi.p, lo.p, ctx->stream);
            d2h(ctx, out_c, lo.p, lo.bytes());
        } else {
            h2d(ctx, lo.p, in_c, lo.bytes());
            launch_fold_adjoint(f->G, f->lam.p, dw.p, lo.p, hi.p, ctx->stream);
            d2h(ctx, out_c, hi.p, hi.bytes());
        }
        sync(ctx);
    });
}
int vsr_folded_apply(vsr_folded* f, const double* hr_c, double* lr_c) {
    return folded_apply_host(f, hr_c, nullptr, lr_c, false);
}
int vsr_folded_apply_adjoint(vsr_folded* f, const double* lr_c, double* hr_c) {
    return folded_apply_host(f, lr_c, nullptr, hr_c, true);
}
int vsr_folded_apply_weighted(vsr_folded* f, const double* hr_c, const double* hr_w, double* lr_c) {
    return folded_apply_host(f, hr_c, hr_w, lr_c, false);
}
int vsr_folded_apply_adjoint_weighted(vsr_folded* f, const double* lr_c, const double* hr_w,
                                      double* hr_c) {
    return folded_apply_host(f, lr_c, hr_w, hr_c, true);
}

static int gram_host(vsr_folded* f, const double* w, double* lr_r) {
    return guarded([&] {
        vsr_ctx* ctx = f->ctx;
        vsr_ctx::Guard g(ctx->device);
        DevBuf<double> lo(f->sp.lr.count()), dw;
        if (w) {
            dw.alloc(f->sp.hr.count());
            h2d(ctx, dw.p, w, dw.bytes());
        }
        launch_gram(f->G, f->lam.p, dw.p, lo.p, ctx->stream);
        d2h(ctx, lr_r, lo.p, lo.bytes());
        sync(ctx);
    });
}
int vsr_folded_gram_diag(vsr_folded* f, double* lr_r) { return gram_host(f, nullptr, lr_r); }
int vsr_folded_gram_diag_weighted(vsr_folded* f, const double* hr_w, double* lr_r) {
    return gram_host(f, hr_w, lr_r);
}
int vsr_folded_swap_blocks_for_fault_injection(vsr_folded* f) {
    return guarded([&] {
        if (f->sp.rate() < 2) return;  // spectral.cpp:116
        vsr_ctx::Guard g(f->ctx->device);
        launch_swap_blocks(f->G, f->lam.p, f->ctx->stream);
        sync(f->ctx);
    });
}

// ============================================================ Tikhonov
// TikhonovOperator (src/solvers.cpp:36-67).  Device state: Lambda (16N),
// X̄ = fft3(xbar) (16N), x̂ work (16N), LR spectrum of y, y and x staging.
struct vsr_tikhonov {
    vsr_ctx* ctx = nullptr;
    Spec sp;
    FoldGeom G;
    double reg = 0.0;
    DevBuf<double2> lam, xbh, Yl, xh;
    DevBuf<double> y, x;
    DevBuf<double> partials, status;  // status: [violated, ratio, last ratio, pad]
    DevBuf<unsigned long long> bad;
    size_t res_blocks = 0;
    SepState sep;                     // Lambda = a[f1] b[f2] c[f3] when the PSF is separable
    DevBuf<double2> Zl;               // LR spectrum of decimate(xbar) when xbar lives on the lattice
    DevBuf<double> zlat;              // decimate(xbar) (lattice prior)
    SpatialPlan spl;                  // spatial expansion (separable compact PSF + lattice prior)
    DevBuf<double> sp_taps, sp_s2, u;
    DevBuf<double> q;                 // constant LR prior term sqrt(d) F_l^-1(Z G1 / (G2 + 2 reg d))
    bool half = false;                // LR stage on the Hermitian half spectrum
    // CUDA graph of one solve for a given (y, x) pair (replayed while they repeat)
    cudaGraphExec_t gexec = nullptr;
    const void* g_y = nullptr;
    void* g_x = nullptr;
    uint64_t g_kernels = 0;
    uint64_t solves = 0;
    ~vsr_tikhonov() {
        if (gexec) cudaGraphExecDestroy(gexec);
    }
    DevBuf<double2> sp_s1, U;
    DevBuf<unsigned long long> lrbad;
    // fp32 solves (vsr_tikhonov_solve_f32*): fp32 y staging / x, and the graph's precision
    DevBuf<float> yf, xf;
    bool g_f32 = false;
};

static void tik_reset_status(vsr_tikhonov* t) {
    VSR_CUDA(cudaMemsetAsync(t->status.p, 0, 4 * sizeof(double), t->ctx->stream));
    VSR_CUDA(cudaMemsetAsync(t->bad.p, 0xff, sizeof(unsigned long long), t->ctx->stream));
}

// xbar_hat_ = fft3(cfg.xbar) (solvers.cpp:45).  When the prior is supported on
// the decimation lattice (the CLI default xbar = zero_fill_upsample(y),
// volsr_main.cpp:208) and a fused fold runs, only its LR spectrum is kept:
// fft3(D^H z)[g + b lr] = fft_LR(z)[g] / sqrt(d) for every alias b.
static void tik_prior(vsr_tikhonov* t, const double* xbar_dev, cudaStream_t st);
static void tik_spatial(vsr_tikhonov* t, cudaStream_t st);

static vsr_tikhonov* tik_new(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3],
                             double reg) {
    require_ctx(ctx);
    const Spec sp = make_spec(hr_dims, rates);
    require_positive(reg, "lambda");  // solvers.cpp:39
    require_nonempty(sp.hr, "fft3");
    auto* t = new vsr_tikhonov();
    t->ctx = ctx;
    t->sp = sp;
    t->G = make_geom(sp.hr, sp.rates);
    t->reg = reg;
    const size_t N = sp.hr.count(), Nl = sp.lr.count();
    t->lam.alloc(N);
    t->xh.alloc(N);
    t->Yl.alloc(Nl);
    t->y.alloc(Nl);
    t->x.alloc(N);
    t->res_blocks = std::max(fft_engine().inverse_final_blocks(sp.hr), fft_engine().pass_blocks(sp.hr, 2));
    t->partials.alloc(2 * std::max<size_t>(t->res_blocks, 1));
    t->status.alloc(4);
    t->bad.alloc(1);
    tik_reset_status(t);
    return t;
}

static void tik_prior(vsr_tikhonov* t, const double* xbar_dev, cudaStream_t st) {
    static const bool off = [] {
        const char* e = std::getenv("VSR_NO_LATTICE");
        return e && e[0] == '1';
    }();
    const Dims& hr = t->sp.hr;
    bool lattice = false;
    if (!off && t->sp.rate() > 1) {
        DevBuf<int> flag(1);
        VSR_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), st));
        const long long N = (long long)hr.count();
        off_lattice_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(
            (long long)hr.m, (long long)hr.n, N, t->sp.rates[0], t->sp.rates[1], t->sp.rates[2], xbar_dev, flag.p);
        VSR_LAUNCH_CHECK();
        int h = 1;
        VSR_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        VSR_CUDA(cudaStreamSynchronize(st));
        lattice = h == 0;
    }
    if (lattice) {
        DevBuf<double>& z = t->zlat;
        z.alloc(t->sp.lr.count());
        launch_decimate(hr, t->sp.rates, xbar_dev, z.p, st);
        t->Zl.alloc(t->sp.lr.count());
        fft_engine().forward3(t->sp.lr, z.p, IN_REAL, t->Zl.p,
                              inv_sqrt_count(t->sp.lr) / std::sqrt((double)t->sp.rate()), st);
        VSR_CUDA(cudaStreamSynchronize(st));
        tik_spatial(t, st);
        if (!t->spl.ok && !use_fused(t->G)) {  // the unfused fold reads the HR fft3(xbar)
            t->Zl.release();
            t->zlat.release();
            lattice = false;
        }
    }
    if (!lattice) {
        t->xbh.alloc(hr.count());
        fft_engine().forward3(hr, xbar_dev, IN_REAL, t->xbh.p, inv_sqrt_count(hr), st);
    }
    ++g_fwd;  // the ctor's fft3(cfg.xbar)
}

// Spatial expansion (spatial.cuh) when Lambda is separable with a compact
// real 1-D factor per axis and xbar lives on the decimation lattice.
// VSR_NO_SPATIAL=1 keeps the FFT path.
static void tik_spatial(vsr_tikhonov* t, cudaStream_t st) {
    const char* env = std::getenv("VSR_NO_SPATIAL");  // read per operator (bench compares both paths)
    const bool off = env && env[0] == '1';
    if (off || !t->sep.t.a || !t->Zl.p || t->sp.rate() < 2) return;
    const Dims& hr = t->sp.hr;
    std::vector<double2> tabs(hr.m + hr.n + hr.s);
    VSR_CUDA(cudaMemcpyAsync(tabs.data(), t->sep.tab.p, tabs.size() * sizeof(double2), cudaMemcpyDeviceToHost, st));
    VSR_CUDA(cudaStreamSynchronize(st));
    std::vector<double> taps, s2;
    std::vector<double2> s1;
    SpatialPlan p;
    if (!spatial_plan_host(hr, t->sp.rates, tabs, taps, p.h, s1, s2)) return;
    for (int a = 0; a < 3; ++a) {
        const int r = t->sp.rates[a], h = p.h[a];
        p.dmin[a] = -(h / r);
        p.ndelta[a] = (r - 1 + h) / r - p.dmin[a] + 1;
    }
    p.dm = spatial_tile(p, t->sp.rates);
    if (!p.dm) return;
    std::vector<double> kp;
    spatial_phase_taps(t->sp.rates, p.h, p.dmin, taps, p.dm, kp);
    taps.swap(kp);
    p.kp_host = taps;
    t->sp_taps.alloc(taps.size());
    t->sp_s1.alloc(s1.size());
    t->sp_s2.alloc(s2.size());
    VSR_CUDA(cudaMemcpyAsync(t->sp_taps.p, taps.data(), taps.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    VSR_CUDA(cudaMemcpyAsync(t->sp_s1.p, s1.data(), s1.size() * sizeof(double2), cudaMemcpyHostToDevice, st));
    VSR_CUDA(cudaMemcpyAsync(t->sp_s2.p, s2.data(), s2.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    const size_t L[3] = {t->sp.lr.m, t->sp.lr.n, t->sp.lr.s};
    size_t so = 0;
    p.kp = t->sp_taps.p;
    for (int a = 0; a < 3; ++a) {
        p.s1[a] = t->sp_s1.p + so;
        p.s2[a] = t->sp_s2.p + so;
        so += L[a];
    }
    p.ok = true;
    const Dims& lr = t->sp.lr;
    const Dims lrh{(size_t)half_pitch(lr.m), lr.n, lr.s};
    const char* henv = std::getenv("VSR_NO_HALF");
    if (!(henv && henv[0] == '1') && rfft_rows_ok(lr.m) && spatial_sandwich_ok(lrh)) {
        // U = (d yv - Z G1) / (G2 + s) splits into a real even filter of y and a
        // constant: u = (d / N_l) F^-1(F(y) / (G2 + s)) - q with
        // q = sqrt(d) F_l^-1(Z G1 / (G2 + s)), formed here once.
        const size_t Nl = lr.count();
        DevBuf<double2> yz(Nl), uq(Nl);
        VSR_CUDA(cudaMemsetAsync(yz.p, 0, yz.bytes(), st));
        launch_spatial_v(lr, t->sp.rate(), p, yz.p, t->Zl.p, t->reg, uq.p, st);  // -Z G1 / (G2 + s)
        t->q.alloc(Nl);
        // q is real by construction (Z is the spectrum of a real lattice
        // prior, G1 and G2 are real even filters): check it like ifft3_real
        // (fft.cpp:86-96) before it enters every solve
        ResidueCheck qc(t->ctx, lr);
        fft_engine().inverse3(lr, uq.p, t->q.p, OUT_REAL,
                              -inv_sqrt_count(lr) * std::sqrt((double)t->sp.rate()), &qc.red, st);
        double qstat[4];
        unsigned long long qbad = 0;
        qc.finish(t->ctx, 1e-8, qstat, &qbad);
        if (qstat[0] != 0.0) throw numeric_error(residue_message(qstat[1], 1e-8));
        if (qbad != ULLONG_MAX)
            throw numeric_error("tikhonov_fast: non-finite value at flat index " + std::to_string(qbad) +
                                " of the prior's LR term");
        t->half = true;
    } else if (!spatial_sandwich_ok(lr)) {
        t->U.alloc(lr.count());  // unfused LR stage: U kernel + inverse3
    }
    t->u.alloc(t->sp.lr.count());
    t->lrbad.alloc(1);
    t->xh.release();  // the HR spectrum is never formed on this path
    const size_t nres = fft_engine().inverse_final_blocks(t->sp.lr);
    if (nres > t->res_blocks) {
        t->res_blocks = nres;
        t->partials.alloc(2 * nres);
    }
    VSR_CUDA(cudaStreamSynchronize(st));
    t->spl = p;
}

int vsr_tikhonov_create(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3],
                        const double* lambda_c, double reg, const double* xbar_r,
                        vsr_tikhonov** out) {
    return guarded([&] {
        require_ctx(ctx);
        vsr_ctx::Guard g(ctx->device);
        vsr_tikhonov* t = tik_new(ctx, hr_dims, rates, reg);
        try {
            h2d(ctx, t->lam.p, lambda_c, t->lam.bytes());
            h2d(ctx, t->x.p, xbar_r, t->x.bytes());
            t->sep.detect(t->sp.hr, t->lam.p, ctx->stream);
            tik_prior(t, t->x.p, ctx->stream);
            sync(ctx);
        } catch (...) {
            delete t;
            throw;
        }
        *out = t;
    });
}

int vsr_tikhonov_create_d(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3],
                          const double* lambda_c_dev, double reg, const double* xbar_r_dev,
                          vsr_tikhonov** out) {
    return guarded([&] {
        require_ctx(ctx);
        vsr_ctx::Guard g(ctx->device);
        vsr_tikhonov* t = tik_new(ctx, hr_dims, rates, reg);
        try {
            VSR_CUDA(cudaMemcpyAsync(t->lam.p, lambda_c_dev, t->lam.bytes(),
                                     cudaMemcpyDeviceToDevice, ctx->stream));
            t->sep.detect(t->sp.hr, t->lam.p, ctx->stream);
            tik_prior(t, xbar_r_dev, ctx->stream);
            sync(ctx);
        } catch (...) {
            delete t;
            throw;
        }
        *out = t;
    });
}

int vsr_tikhonov_destroy(vsr_tikhonov* t) {
    return guarded([&] {
        if (!t) return;
        vsr_ctx::Guard g(t->ctx->device);
        cudaStreamSynchronize(t->ctx->stream);
        delete t;
    });
}

// Enqueue one solve: LR FFT of y (== F D^H y up to the alias replication and
// 1/sqrt(d)) -> fused fold -> inverse FFT to real x with
// the residue / finiteness reductions.
static bool tik_fp32_ok(const vsr_tikhonov* t) {
    return t->spl.ok && t->half && spatial_march_ok(t->sp.hr, t->sp.rates, t->spl);
}

// xf_dev / yf_dev (fp32 solves, spatial half-spectrum path only): y arrives
// as fp32 and is widened for the fp64 LR stage; the expansion writes fp32 x.
static void tik_enqueue(vsr_tikhonov* t, const double* y_dev, double* x_dev, const float* yf_dev = nullptr,
                        float* xf_dev = nullptr) {
    cudaStream_t st = t->ctx->stream;
    Profiler* prof = t->ctx->prof();
    if (yf_dev) {
        launch_widen(yf_dev, t->y.p, t->y.n, st);
        y_dev = t->y.p;
    }
    if (t->spl.ok && t->half) {
        // half-spectrum LR stage: r2c rows, axis 2, filter sandwich on axis 3,
        // inverse axis 2, c2r rows minus the constant prior term -> u
        const Dims& lr = t->sp.lr;
        const Dims lrh{(size_t)half_pitch(lr.m), lr.n, lr.s};
        const long long rows = (long long)(lr.n * lr.s);
        {
            {
                ProfScope ps(prof, "lr_r2c_axis1", st);
                rfft_rows_forward(lr.m, y_dev, t->Yl.p, rows, st);
            }
            ProfScope ps(prof, "lr_fft_axis2_half", st);
            fft_engine().axis_pass(lrh, 1, false, t->Yl.p, IN_COMPLEX, t->Yl.p, OUT_COMPLEX, 1.0, nullptr, st);
        }
        ++g_fwd;
        {
            ProfScope ps(prof, "lr_filter_axis3_half", st);
            launch_spatial_sandwich(lrh, t->sp.rate(), t->spl, t->Yl.p, nullptr, t->reg, inv_sqrt_count(lr),
                                    inv_sqrt_count(lr) * std::sqrt((double)t->sp.rate()), st);
        }
        {
            {
                ProfScope ps(prof, "lr_ifft_axis2_half", st);
                fft_engine().axis_pass(lrh, 1, true, t->Yl.p, IN_COMPLEX, t->Yl.p, OUT_COMPLEX, 1.0, nullptr, st);
            }
            ProfScope ps(prof, "lr_c2r_axis1", st);
            rfft_rows_inverse(lr.m, t->Yl.p, t->u.p, rows, 1.0, t->q.p, st);
        }
        ++g_inv;
        {
            ProfScope ps(prof, "spatial_expand", st);
            if (xf_dev)
                launch_spatial_expand_f32(t->sp.hr, t->sp.rates, t->spl, t->u.p, t->zlat.p, xf_dev, t->bad.p, st);
            else
                launch_spatial_expand(t->sp.hr, t->sp.rates, t->spl, t->u.p, t->zlat.p, 1.0, x_dev, t->bad.p, st);
        }
        return;  // real by construction: no imaginary residue to reduce
    }
    if (xf_dev) throw std::logic_error("tikhonov fp32: not the spatial path");
    if (t->spl.ok && t->U.p == nullptr) {
        ProfScope ps(prof, "lr_fft12", st);
        fft_engine().forward12(t->sp.lr, y_dev, IN_REAL, t->Yl.p, st);
    } else {
        ProfScope ps(prof, "lr_fft3", st);
        fft_engine().forward3(t->sp.lr, y_dev, IN_REAL, t->Yl.p, inv_sqrt_count(t->sp.lr), st);
    }
    ++g_fwd;  // the one forward transform of solve() (solvers.cpp:52)
    PassReduce red{t->partials.p, t->bad.p};
    if (t->spl.ok) {
        // U on the LR grid -> u = sqrt(d) F_l^-1(U) -> x = D^H z + H^T D^H u
        PassReduce lred{t->partials.p, t->lrbad.p};
        const double usc = inv_sqrt_count(t->sp.lr) * std::sqrt((double)t->sp.rate());
        if (t->U.p == nullptr) {
            // fused: lr_fft3 ran the forward axis-1/2 passes only (unscaled)
            {
                ProfScope ps(prof, "lr_sandwich_axis3", st);
                launch_spatial_sandwich(t->sp.lr, t->sp.rate(), t->spl, t->Yl.p, t->Zl.p, t->reg,
                                        inv_sqrt_count(t->sp.lr), usc, st);
            }
            {
                ProfScope ps(prof, "lr_ifft_axis2", st);
                fft_engine().axis_pass(t->sp.lr, 1, true, t->Yl.p, IN_COMPLEX, t->Yl.p, OUT_COMPLEX, 1.0, nullptr, st);
            }
            {
                ProfScope ps(prof, "lr_ifft_axis1_c2r", st);
                fft_engine().axis_pass(t->sp.lr, 0, true, t->Yl.p, IN_COMPLEX, t->u.p, OUT_REAL, 1.0, &lred, st);
            }
        } else {
            {
                ProfScope ps(prof, "spatial_u", st);
                launch_spatial_v(t->sp.lr, t->sp.rate(), t->spl, t->Yl.p, t->Zl.p, t->reg, t->U.p, st);
            }
            ProfScope ps(prof, "lr_ifft3", st);
            fft_engine().inverse3(t->sp.lr, t->U.p, t->u.p, OUT_REAL, usc, &lred, st);
        }
        {
            ProfScope ps(prof, "spatial_expand", st);
            launch_spatial_expand(t->sp.hr, t->sp.rates, t->spl, t->u.p, t->zlat.p, 1.0, x_dev, t->bad.p, st);
        }
    } else if (fuse_axis(t->G, 3) == 1) {
        // fold + inverse axis 1 (contiguous rows), then axis 2, then axis 3 -> real x
        {
            ProfScope ps(prof, "tik_fold_ifft_axis1", st);
            launch_tik_fold_ifft1(t->G, t->Yl.p, t->lam.p, t->xbh.p, t->xh.p, t->reg, st, t->sep.t, t->Zl.p);
        }
        {
            ProfScope ps(prof, "fft_inv_axis2", st);
            fft_engine().axis_pass(t->sp.hr, 1, true, t->xh.p, IN_COMPLEX, t->xh.p, OUT_COMPLEX, 1.0, nullptr, st);
        }
        {
            ProfScope ps(prof, "fft_inv_axis3_c2r", st);
            fft_engine().axis_pass(t->sp.hr, 2, true, t->xh.p, IN_COMPLEX, x_dev, OUT_REAL,
                                   inv_sqrt_count(t->sp.hr), &red, st);
        }
    } else if (use_fused(t->G)) {
        {
            ProfScope ps(prof, "tik_fold_ifft_axis3", st);
            launch_tik_fold_ifft3(t->G, t->Yl.p, t->lam.p, t->xbh.p, t->xh.p, t->reg, st, t->sep.t, t->Zl.p);
        }
        fft_engine().inverse21(t->sp.hr, t->xh.p, x_dev, OUT_REAL, inv_sqrt_count(t->sp.hr), &red, st, prof);
    } else {
        {
            ProfScope ps(prof, "tik_fold", st);
            launch_tik_fold(t->G, t->Yl.p, t->lam.p, t->xbh.p, t->xh.p, t->reg, st);
        }
        fft_engine().inverse3(t->sp.hr, t->xh.p, x_dev, OUT_REAL, inv_sqrt_count(t->sp.hr), &red,
                              st, prof);
    }
    ++g_inv;  // the one inverse transform (solvers.cpp:64)
    {
        ProfScope ps(prof, "residue_status", st);
        const size_t nres = t->spl.ok ? fft_engine().pass_blocks(t->sp.lr, 0)
                            : fuse_axis(t->G, 3) == 1 ? fft_engine().pass_blocks(t->sp.hr, 2)
                                                 : fft_engine().inverse_final_blocks(t->sp.hr);
        residue_status_kernel<<<1, 1024, 0, st>>>(t->partials.p, (long long)nres, 1e-8, t->status.p);
        VSR_LAUNCH_CHECK();
    }
}

// One solve through a CUDA graph (launch gaps removed).  The first solve of an
// operator runs eagerly (lazy twiddle tables, attribute setup); the next one is
// captured for its (y, x) pair and replayed while the pair repeats.  The event
// profiler and VSR_NO_GRAPH=1 keep the eager path.
static void tik_run(vsr_tikhonov* t, const double* y_dev, double* x_dev, const float* yf_dev = nullptr,
                    float* xf_dev = nullptr) {
    static const bool off = [] {
        const char* e = std::getenv("VSR_NO_GRAPH");
        return e && e[0] == '1';
    }();
    cudaStream_t st = t->ctx->stream;
    const bool eager = off || t->ctx->prof() != nullptr || t->solves++ == 0;
    if (eager) {
        tik_enqueue(t, y_dev, x_dev, yf_dev, xf_dev);
        return;
    }
    const bool f32 = xf_dev != nullptr;
    const void* gy = f32 ? (const void*)yf_dev : (const void*)y_dev;
    void* gx = f32 ? (void*)xf_dev : (void*)x_dev;
    if (!(t->gexec && t->g_y == gy && t->g_x == gx && t->g_f32 == f32)) {
        if (t->gexec) {
            cudaGraphExecDestroy(t->gexec);
            t->gexec = nullptr;
        }
        const uint64_t l0 = g_launches.load();
        const uint64_t f0 = g_fwd.load(), i0 = g_inv.load();
        cudaGraph_t graph = nullptr;
        VSR_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        try {
            tik_enqueue(t, y_dev, x_dev, yf_dev, xf_dev);
        } catch (...) {
            cudaStreamEndCapture(st, &graph);
            if (graph) cudaGraphDestroy(graph);
            throw;
        }
        VSR_CUDA(cudaStreamEndCapture(st, &graph));
        const cudaError_t e = cudaGraphInstantiate(&t->gexec, graph, 0);
        cudaGraphDestroy(graph);
        VSR_CUDA(e);
        t->g_kernels = g_launches.load() - l0;
        g_launches.fetch_sub(t->g_kernels);  // counted when the graph runs
        g_fwd.fetch_sub(g_fwd.load() - f0);
        g_inv.fetch_sub(g_inv.load() - i0);
        t->g_y = gy;
        t->g_x = gx;
        t->g_f32 = f32;
    }
    VSR_CUDA(cudaGraphLaunch(t->gexec, st));
    g_launches.fetch_add(t->g_kernels);
    ++g_fwd;  // the solve's transform budget (solvers.cpp:52,64)
    ++g_inv;
}

static void tik_check(vsr_tikhonov* t) {
    double status[4];
    unsigned long long bad = 0;
    d2h(t->ctx, status, t->status.p, sizeof(status));
    d2h(t->ctx, &bad, t->bad.p, sizeof(bad));
    sync(t->ctx);
    if (status[0] != 0.0 || bad != ULLONG_MAX) {
        tik_reset_status(t);
        sync(t->ctx);
        if (status[0] != 0.0) throw numeric_error(residue_message(status[1], 1e-8));
        throw numeric_error("tikhonov_fast: non-finite value at flat index " + std::to_string(bad));
    }
}

int vsr_tikhonov_solve(vsr_tikhonov* t, const double* y_r, double* x_r) {
    return guarded([&] {
        if (!t) throw std::invalid_argument("vsr_tikhonov_solve: null operator");
        vsr_ctx::Guard g(t->ctx->device);
        h2d(t->ctx, t->y.p, y_r, t->y.bytes());
        tik_run(t, t->y.p, t->x.p);
        d2h(t->ctx, x_r, t->x.p, t->x.bytes());
        tik_check(t);
    });
}

int vsr_tikhonov_solve_d(vsr_tikhonov* t, const double* y_dev, double* x_dev) {
    return guarded([&] {
        if (!t) throw std::invalid_argument("vsr_tikhonov_solve_d: null operator");
        vsr_ctx::Guard g(t->ctx->device);
        tik_run(t, y_dev, x_dev);
    });
}

// fp32 solves (BASELINE north_star's optional fp32 mode): y and x in fp32,
// the LR stage in fp64, the expansion in fp32 arithmetic
static void tik_require_fp32(vsr_tikhonov* t) {
    if (!t) throw std::invalid_argument("vsr_tikhonov_solve_f32: null operator");
    if (!tik_fp32_ok(t))
        throw std::invalid_argument(
            "tikhonov_fast: fp32 mode needs the spatial path (separable compact PSF, lattice prior, "
            "rates (2, 2, 2|4), tile-aligned LR grid)");
}

int vsr_tikhonov_solve_f32(vsr_tikhonov* t, const float* y_r, float* x_r) {
    return guarded([&] {
        tik_require_fp32(t);
        vsr_ctx::Guard g(t->ctx->device);
        if (!t->yf.p) t->yf.alloc(t->sp.lr.count());
        if (!t->xf.p) t->xf.alloc(t->sp.hr.count());
        h2d(t->ctx, t->yf.p, y_r, t->yf.bytes());
        tik_run(t, nullptr, nullptr, t->yf.p, t->xf.p);
        d2h(t->ctx, x_r, t->xf.p, t->xf.bytes());
        tik_check(t);
    });
}

int vsr_tikhonov_solve_f32_d(vsr_tikhonov* t, const float* y_dev, float* x_dev) {
    return guarded([&] {
        tik_require_fp32(t);
        vsr_ctx::Guard g(t->ctx->device);
        tik_run(t, nullptr, nullptr, y_dev, x_dev);
    });
}

int vsr_tikhonov_fp32_ok(vsr_tikhonov* t) { return t && tik_fp32_ok(t) ? 1 : 0; }

int vsr_tikhonov_check(vsr_tikhonov* t) {
    return guarded([&] {
        vsr_ctx::Guard g(t->ctx->device);
        tik_check(t);
    });
}

int vsr_tikhonov_fast(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3],
                      const double* y_r, const double* lambda_c, double reg, const double* xbar_r,
                      double* x_r) {
    vsr_tikhonov* t = nullptr;
    int rc = vsr_tikhonov_create(ctx, hr_dims, rates, lambda_c, reg, xbar_r, &t);
    if (rc != VSR_OK) return rc;
    rc = vsr_tikhonov_solve(t, y_r, x_r);
    std::string msg = g_last_error;
    vsr_tikhonov_destroy(t);
    g_last_error = msg;
    return rc;
}

double vsr_tikhonov_algorithmic_bytes(const size_t hr_dims[3], const size_t rates[3]) {
    const double N = (double)hr_dims[0] * hr_dims[1] * hr_dims[2];
    const double d = (double)rates[0] * rates[1] * rates[2];
    return (72.0 + 40.0 / d) * N;
}

// ============================================================ TV pieces
int vsr_make_gamma(vsr_ctx* ctx, const size_t hr_dims[3], double tau, double* gamma_r) {
    return guarded([&] {
        require_ctx(ctx);
        const Dims d = to_dims(hr_dims);
        validate_tau(tau);
        vsr_ctx::Guard g(ctx->device);
        const auto nr = diff_norm_table(d.m), nc = diff_norm_table(d.n), ns = diff_norm_table(d.s);
        DevBuf<double> dr(d.m), dc(d.n), ds(d.s), out(d.count());
        h2d(ctx, dr.p, nr.data(), dr.bytes());
        h2d(ctx, dc.p, nc.data(), dc.bytes());
        h2d(ctx, ds.p, ns.data(), ds.bytes());
        launch_gamma(d, dr.p, dc.p, ds.p, tau, out.p, ctx->stream);
        d2h(ctx, gamma_r, out.p, out.bytes());
        sync(ctx);
    });
}

int vsr_tv_x_update(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3],
                    const double* y_r, const double* lambda_c, double mu,
                    const double* theta_hat_c, const double* gamma_r, double* x_r) {
    return guarded([&] {
        require_ctx(ctx);
        const Spec sp = make_spec(hr_dims, rates);
        require_positive(mu, "mu");  // solvers.cpp:248
        const size_t N = sp.hr.count(), Nl = sp.lr.count();
        // require_gamma_valid (solvers.cpp:209-216)
        for (size_t p = 0; p < N; ++p)
            if (!(gamma_r[p] > 0.0) || !std::isfinite(gamma_r[p]))
                throw numeric_error(
                    "tv_x_update: gamma must be strictly positive and finite everywhere; entry " +
                    std::to_string(p) +
                    " is not (unfloored DC singularity of the difference gram?)");
        vsr_ctx::Guard g(ctx->device);
        const FoldGeom G = make_geom(sp.hr, sp.rates);
        DevBuf<double> dy(Nl), gam(N), x(N);
        DevBuf<double2> Yl(Nl), lam(N), W(N);
        h2d(ctx, dy.p, y_r, dy.bytes());
        h2d(ctx, lam.p, lambda_c, lam.bytes());
        h2d(ctx, W.p, theta_hat_c, W.bytes());
        h2d(ctx, gam.p, gamma_r, gam.bytes());
        fft_engine().forward3(sp.lr, dy.p, IN_REAL, Yl.p, inv_sqrt_count(sp.lr), ctx->stream);
        ++g_fwd;
        GammaTables tabs{nullptr, nullptr, nullptr, 0.0};
        launch_tv_fold(G, Yl.p, lam.p, W.p, W.p, gam.p, tabs, mu, nullptr, ctx->stream);
        ResidueCheck rc(ctx, sp.hr);
        fft_engine().inverse3(sp.hr, W.p, x.p, OUT_REAL, inv_sqrt_count(sp.hr), &rc.red, ctx->stream);
        ++g_inv;
        double status[4];
        unsigned long long bad;
        rc.finish(ctx, 1e-8, status, &bad);
        if (status[0] != 0.0) throw numeric_error(residue_message(status[1], 1e-8));
        d2h(ctx, x_r, x.p, x.bytes());
        sync(ctx);
    });
}

int vsr_tv_shrink(vsr_ctx* ctx, size_t count, const double* nu1, const double* nu2,
                  const double* nu3, double threshold, double* out1, double* out2, double* out3) {
    return guarded([&] {
        require_ctx(ctx);
        if (threshold < 0.0) throw std::invalid_argument("tv_shrink: threshold must be >= 0");
        if (count == 0) return;
        vsr_ctx::Guard g(ctx->device);
        DevBuf<double> a(count), b(count), c(count), o1(count), o2(count), o3(count);
        h2d(ctx, a.p, nu1, a.bytes());
        h2d(ctx, b.p, nu2, b.bytes());
        h2d(ctx, c.p, nu3, c.bytes());
        launch_shrink(count, a.p, b.p, c.p, threshold, o1.p, o2.p, o3.p, ctx->stream);
        d2h(ctx, out1, o1.p, o1.bytes());
        d2h(ctx, out2, o2.p, o2.bytes());
        d2h(ctx, out3, o3.p, o3.bytes());
        sync(ctx);
    });
}

int vsr_objective_tv(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3],
                     const double* x_r, const double* y_r, const double* lambda_c,
                     double tv_weight, double* out) {
    return guarded([&] {
        require_ctx(ctx);
        const Spec sp = make_spec(hr_dims, rates);
        require_nonempty(sp.hr, "fft3");
        vsr_ctx::Guard g(ctx->device);
        const FoldGeom G = make_geom(sp.hr, sp.rates);
        const size_t N = sp.hr.count(), Nl = sp.lr.count();
        DevBuf<double> dx(N), dy(Nl);
        DevBuf<double2> lam(N), W(N), Yl(Nl);
        h2d(ctx, dx.p, x_r, dx.bytes());
        h2d(ctx, dy.p, y_r, dy.bytes());
        h2d(ctx, lam.p, lambda_c, lam.bytes());
        cudaStream_t st = ctx->stream;
        // data term by LR Parseval: ||y - D H x||^2 = ||F_l y - (1/sqrt d) fold(Lambda x̂)||^2
        fft_engine().forward3(sp.lr, dy.p, IN_REAL, Yl.p, inv_sqrt_count(sp.lr), st);
        fft_engine().forward3(sp.hr, dx.p, IN_REAL, W.p, inv_sqrt_count(sp.hr), st);
        g_fwd += 2;
        const size_t fb = fit_blocks(G), tb = tv_norm_blocks(sp.hr);
        DevBuf<double> fitp(fb), tvp(tb), res(2);
        launch_fit_partials(G, Yl.p, lam.p, W.p, fitp.p, st);
        launch_tv_norm(sp.hr, dx.p, tvp.p, st);
        launch_finalize_sum(fitp.p, 1, 1, fb, res.p, st);
        launch_finalize_sum(tvp.p, 1, 1, tb, res.p + 1, st);
        double h[2];
        d2h(ctx, h, res.p, sizeof(h));
        sync(ctx);
        *out = 0.5 * h[0] + tv_weight * h[1];  // solvers.cpp:318
    });
}

// ============================================================ ADMM-TV
// admm_tv (src/solvers.cpp:321-411).  State per iteration: theta (8N),
// dual (24N, ping-pong), x (8N), spectral work (16N), Lambda (16N).
struct vsr_tv {
    vsr_ctx* ctx = nullptr;
    Spec sp;
    FoldGeom G;
    double lambda = 0, mu = 0, rel_tol = 0, tau = 0;
    size_t max_iters = 0;
    DevBuf<double2> lam, Yl, W;
    DevBuf<double> x, xprev, theta, dualA, dualB;
    DevBuf<double> tnr, tnc, tns;
    DevBuf<double> fitp, stp, resp;
    DevBuf<unsigned long long> bad;
    DevBuf<double> obj, res, rel, status, init_obj;
    size_t fit_blocks = 0, st_blocks = 0, res_blocks = 0;
    SepState sep;
    DevBuf<double> gw;  // LR table sum_b Gamma_b |Lambda_b|^2 (axis-1 sandwich)
    DevBuf<double2> W2;  // sandwich output on the half-spectrum path (m x n x (s/2+1))
    // fp32 mode (cfg->precision): fp32 iteration state; x stays fp64 for the
    // initial objective and the widened result
    bool f32 = false;
    DevBuf<float> xf, xprevf, thetaf, dualAf, dualBf;
    DevBuf<float2> Wf, W2f;
    DevBuf<int2> tiles;  // half-spectrum sandwich: the tiles that do work (one per conjugate pair)
    int ntiles = 0;
    DevBuf<int> iter_dev;  // iteration index read by the finalize kernel (graph replay)
    cudaGraphExec_t gexec = nullptr;  // kGraphIters consecutive iterations (dual ping-pong period 2)
    uint64_t g_kernels = 0;
    // fixed-count iterations: the scalar finalize runs on a side stream and
    // overlaps the next iteration's forward passes; the next fold (which
    // rewrites the partials) waits for it
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    bool fin_pending = false;
    ~vsr_tv() {
        if (gexec) cudaGraphExecDestroy(gexec);
        if (side) cudaStreamDestroy(side);
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
    }
    size_t iters_done = 0;
    bool dual_in_a = true;
    bool stopped = false;
    std::chrono::steady_clock::time_point t0;
};

static void tv_validate(const vsr_tv_config* cfg) {
    if (!cfg) throw std::invalid_argument("admm_tv: null config");
    require_positive(cfg->lambda, "lambda");  // solvers.cpp:323-326
    require_positive(cfg->mu, "mu");
    if (cfg->max_iters < 1) throw std::invalid_argument("admm_tv: max_iters must be >= 1");
}

// TV transforms on the Hermitian half spectrum along axis 3 (VSR_TV_FULL=1: full).
static bool tv_half(const Dims& hr) {
    static const bool off = [] {
        const char* e = std::getenv("VSR_TV_FULL");
        return e && e[0] == '1';
    }();
    return !off && fft_engine().half3_ok(hr);
}

static vsr_tv* tv_build(vsr_ctx* ctx, const Spec& sp, const double* y_dev, const double* psf_dev,
                        const vsr_tv_config* cfg, const double* init_dev) {
    auto t0 = std::chrono::steady_clock::now();
    auto* h = new vsr_tv();
    try {
        h->ctx = ctx;
        h->sp = sp;
        h->t0 = t0;
        h->G = make_geom(sp.hr, sp.rates);
        h->lambda = cfg->lambda;
        h->mu = cfg->mu;
        h->rel_tol = cfg->rel_tol;
        h->max_iters = cfg->max_iters;
        h->tau = cfg->has_tau ? cfg->tau : 1e-8 * cfg->mu;  // solvers.cpp:332
        validate_tau(h->tau);
        const Dims& hr = sp.hr;
        const size_t N = hr.count(), Nl = sp.lr.count();
        cudaStream_t st = ctx->stream;
        h->f32 = cfg->precision == VSR_PRECISION_F32;
        if (cfg->precision != VSR_PRECISION_F64 && !h->f32)
            throw std::invalid_argument("admm_tv: unknown precision");
        h->lam.alloc(N);
        h->Yl.alloc(Nl);
        h->W.alloc(N);  // fp32 mode: the initial objective's full spectrum only (freed after setup)
        h->x.alloc(N);
        if (!h->f32) {
            if (h->rel_tol > 0.0) h->xprev.alloc(N);
            h->theta.alloc(N);
            h->dualA.alloc(3 * N);
            h->dualB.alloc(3 * N);
        }
        const auto nr = diff_norm_table(hr.m), nc = diff_norm_table(hr.n), ns = diff_norm_table(hr.s);
        h->tnr.alloc(hr.m);
        h->tnc.alloc(hr.n);
        h->tns.alloc(hr.s);
        h2d(ctx, h->tnr.p, nr.data(), h->tnr.bytes());
        h2d(ctx, h->tnc.p, nc.data(), h->tnc.bytes());
        h2d(ctx, h->tns.p, ns.data(), h->tns.bytes());
        h->fit_blocks = tv_fold_blocks(h->G);
        h->st_blocks = stencil_geom(hr).blocks();
        h->res_blocks = fft_engine().inverse_final_blocks(hr);
        h->fitp.alloc(std::max<size_t>(
            std::max(std::max(std::max(h->fit_blocks, fit_blocks(h->G)), tv_sandwich_blocks(h->G)),
                     tv_sandwich1_blocks(h->G)),
            1));
        h->stp.alloc(kStencilVals * h->st_blocks);
        h->resp.alloc(2 * std::max<size_t>(std::max(std::max(h->res_blocks, fft_engine().pass_blocks(hr, 2)),
                                                    fft_engine().half3_blocks(hr)),
                                           1));
        h->bad.alloc(1);
        h->obj.alloc(h->max_iters);
        h->res.alloc(h->max_iters);
        h->rel.alloc(h->max_iters);
        h->status.alloc(4);
        h->init_obj.alloc(1);
        h->iter_dev.alloc(1);
        VSR_CUDA(cudaMemsetAsync(h->iter_dev.p, 0, sizeof(int), st));
        const double st_init[4] = {-1.0, 0.0, 0.0, 0.0};
        h2d(ctx, h->status.p, st_init, sizeof(st_init));
        VSR_CUDA(cudaMemsetAsync(h->bad.p, 0xff, sizeof(unsigned long long), st));

        // precompute (solvers.cpp:336-344): Lambda = DFT(psf); LR spectrum of y
        fft_engine().forward3(hr, psf_dev, IN_REAL, h->lam.p, 1.0, st);
        fft_engine().forward3(sp.lr, y_dev, IN_REAL, h->Yl.p, inv_sqrt_count(sp.lr), st);
        g_fwd += 2;
        h->sep.detect(hr, h->lam.p, st);
        if (h->f32) {
            if (!(fuse_axis(h->G, 1) == 1 && tv_half(hr) && h->sep.t.a && hr.m % 2 == 0 &&
                  tv_sandwich_pipe_ok(h->G)))
                throw std::invalid_argument(
                    "admm_tv: fp32 mode needs a separable PSF spectrum and a half-spectrum geometry "
                    "(power-of-two axis 3, even axis 1, a pipelined axis-1 sandwich shape)");
            const size_t Nh = hr.m * hr.n * (hr.s / 2 + 1);
            h->xf.alloc(N);
            if (h->rel_tol > 0.0) h->xprevf.alloc(N);
            h->thetaf.alloc(N);
            h->dualAf.alloc(3 * N);
            h->dualBf.alloc(3 * N);
            h->Wf.alloc(Nh);
            h->W2f.alloc(Nh);
        }
        if (fuse_axis(h->G, 1) == 1) {
            if (tv_half(hr)) {
                if (!h->f32) h->W2.alloc(hr.m * hr.n * (hr.s / 2 + 1));
                if (tv_sandwich1_tile_g2(h->G) == 1) {
                    const std::vector<int2> tl = tv_sandwich1_active_tiles(h->G);
                    h->ntiles = (int)tl.size();
                    h->tiles.alloc(tl.size());
                    h2d(ctx, h->tiles.p, tl.data(), h->tiles.bytes());
                }
            }
            h->gw.alloc(Nl);
            GammaTables tabs{h->tnr.p, h->tnc.p, h->tns.p, h->tau};
            launch_tv_gram(h->G, h->lam.p, h->sep.t, tabs, h->gw.p, st);
        }
        // init (solvers.cpp:346-354)
        if (cfg->init == VSR_INIT_ZERO) {
            VSR_CUDA(cudaMemsetAsync(h->x.p, 0, h->x.bytes(), st));
        } else if (cfg->init == VSR_INIT_UPSAMPLED) {
            launch_nn_upsample(hr, sp.rates, y_dev, h->x.p, st);
        } else if (cfg->init == VSR_INIT_PROVIDED) {
            if (!init_dev) throw shape_error("admm_tv: init volume: dims mismatch");
            VSR_CUDA(cudaMemcpyAsync(h->x.p, init_dev, h->x.bytes(), cudaMemcpyDeviceToDevice, st));
        } else {
            throw std::invalid_argument("admm_tv: unknown init mode");
        }
        // u0 = L x0, dual0 = 0 (:356-358) -> theta for iteration 1; TV(x0)
        if (h->f32) {
            launch_narrow(h->x.p, h->xf.p, N, st);
            launch_tv_stencil_f32(hr, true, h->xf.p, nullptr, h->dualAf.p, h->thetaf.p, h->lambda / h->mu, nullptr,
                                  h->stp.p, st);
        } else {
            launch_tv_stencil(hr, true, h->x.p, nullptr, h->dualA.p, h->theta.p, h->lambda / h->mu,
                              nullptr, h->stp.p, st);
        }
        // initial objective (:361): data term by LR Parseval from fft3(x0)
        fft_engine().forward3(hr, h->x.p, IN_REAL, h->W.p, inv_sqrt_count(hr), st);
        ++g_fwd;
        launch_fit_partials(h->G, h->Yl.p, h->lam.p, h->W.p, h->fitp.p, st);
        TvIterScalars sc{h->obj.p, h->res.p, h->rel.p, h->status.p};
        launch_tv_finalize(0, h->fitp.p, fit_blocks(h->G), h->stp.p, h->st_blocks, nullptr, 0,
                           h->lambda, 1e-8, sc, h->init_obj.p, st);
        if (h->f32) {  // the fp64 spectra served the setup only
            sync(ctx);
            h->W.release();
            h->lam.release();
        }
    } catch (...) {
        delete h;
        throw;
    }
    return h;
}

// iterations per captured TV graph: a multiple of the dual ping-pong period 2
#ifndef VSR_TV_GRAPH_ITERS
#define VSR_TV_GRAPH_ITERS 4
#endif
constexpr size_t kTvGraphIters = VSR_TV_GRAPH_ITERS;

// the previous iteration's side-stream finalize must be done before the
// partial buffers are rewritten (and before anything reads the report)
static void tv_join(vsr_tv* h) {
    if (h->fin_pending) {
        VSR_CUDA(cudaStreamWaitEvent(h->ctx->stream, h->ev_join, 0));
        h->fin_pending = false;
    }
}

static void tv_finalize_step(vsr_tv* h, Profiler* prof, bool a1, bool half, cudaStream_t st);

static void tv_step(vsr_tv* h) {
    cudaStream_t st = h->ctx->stream;
    const Dims& hr = h->sp.hr;
    const double s = inv_sqrt_count(hr);
    // theta_hat = fft3(theta); k_hat = data_hat + mu theta_hat (:374-375), folded x-update (:376)
    Profiler* prof = h->ctx->prof();
    GammaTables tabs{h->tnr.p, h->tnc.p, h->tns.p, h->tau, h->gw.p};
    const bool fused = use_fused(h->G);
    const bool a1 = fuse_axis(h->G, 1) == 1;
    // Hermitian half spectrum along axis 3 (theta is real): planes 0..s/2 only
    const bool half = a1 && tv_half(hr);
    const Dims hrh{hr.m, hr.n, hr.s / 2 + 1};
    if (h->f32) {  // fp32 mode: the half-spectrum route on fp32 state (tv_build checked the geometry)
        tabs.half3 = 1;
        tabs.tiles = h->tiles.p;
        tabs.ntiles = h->ntiles;
        {
            ProfScope ps(prof, "fft_fwd_axis3_r2c_half", st);
            fft_engine().r2c_axis3_half_f(hr, h->thetaf.p, h->Wf.p, st);
        }
        {
            ProfScope ps(prof, "fft_fwd_axis2_half", st);
            fft_engine().axis_pass_cf(hrh, 1, false, h->Wf.p, st);
        }
        tv_join(h);
        {
            ProfScope ps(prof, "tv_fft1_fold_ifft1_half", st);
            if (!tv_sandwich_pipe_f32(h->G, h->Yl.p, h->sep.t, h->Wf.p, h->W2f.p, tabs, h->mu, h->mu * (double)h->G.d,
                                      1.0 / h->mu, s, h->fitp.p, st))
                throw std::logic_error("admm_tv fp32: sandwich geometry");
        }
        if (h->rel_tol > 0.0) std::swap(h->xf, h->xprevf);  // x_prev = x (:364)
        PassReduce red{h->resp.p, h->bad.p};
        {
            ProfScope ps(prof, "fft_inv_axis2_half", st);
            fft_engine().axis_pass_cf(hrh, 1, true, h->W2f.p, st);
        }
        {
            ProfScope ps(prof, "fft_inv_axis3_c2r_half", st);
            fft_engine().c2r_axis3_half_f(hr, h->W2f.p, h->xf.p, s, &red, st);
        }
        g_fwd += 1;
        g_inv += 1;
        float* din = h->dual_in_a ? h->dualAf.p : h->dualBf.p;
        float* dout = h->dual_in_a ? h->dualBf.p : h->dualAf.p;
        {
            ProfScope ps(prof, "tv_stencil", st);
            launch_tv_stencil_f32(hr, false, h->xf.p, din, dout, h->thetaf.p, h->lambda / h->mu,
                                  h->rel_tol > 0.0 ? h->xprevf.p : nullptr, h->stp.p, st);
        }
        h->dual_in_a = !h->dual_in_a;
        tv_finalize_step(h, prof, true, true, st);
        return;
    }
    if (half) {
        tabs.half3 = 1;
        tabs.tiles = h->ntiles ? h->tiles.p : nullptr;
        tabs.ntiles = h->ntiles;
        {
            ProfScope ps(prof, "fft_fwd_axis3_r2c_half", st);
            fft_engine().r2c_axis3_half(hr, h->theta.p, h->W.p, st);
        }
        {
            ProfScope ps(prof, "fft_fwd_axis2_half", st);
            fft_engine().axis_pass(hrh, 1, false, h->W.p, IN_COMPLEX, h->W.p, OUT_COMPLEX, 1.0, nullptr, st);
        }
        tv_join(h);
        ProfScope ps(prof, "tv_fft1_fold_ifft1_half", st);
        launch_tv_sandwich1(h->G, h->Yl.p, h->lam.p, h->W.p, tabs, h->mu, s, h->fitp.p, st, h->sep.t, h->W2.p);
    } else if (a1) {
        {
            ProfScope ps(prof, "fft_fwd_axis3_r2c", st);
            fft_engine().axis_pass(hr, 2, false, h->theta.p, IN_REAL, h->W.p, OUT_COMPLEX, 1.0, nullptr, st);
        }
        {
            ProfScope ps(prof, "fft_fwd_axis2", st);
            fft_engine().axis_pass(hr, 1, false, h->W.p, IN_COMPLEX, h->W.p, OUT_COMPLEX, 1.0, nullptr, st);
        }
        tv_join(h);
        ProfScope ps(prof, "tv_fft1_fold_ifft1", st);
        launch_tv_sandwich1(h->G, h->Yl.p, h->lam.p, h->W.p, tabs, h->mu, s, h->fitp.p, st, h->sep.t);
    } else if (fused) {
        fft_engine().forward12(hr, h->theta.p, IN_REAL, h->W.p, st, prof);
        tv_join(h);
        ProfScope ps(prof, "tv_fft3_fold_ifft3", st);
        launch_tv_sandwich(h->G, h->Yl.p, h->lam.p, h->W.p, tabs, h->mu, s, h->fitp.p, st, h->sep.t);
    } else {
        fft_engine().forward3(hr, h->theta.p, IN_REAL, h->W.p, s, st, prof);
        tv_join(h);
        ProfScope ps(prof, "tv_fold", st);
        launch_tv_fold(h->G, h->Yl.p, h->lam.p, h->W.p, h->W.p, nullptr, tabs, h->mu, h->fitp.p, st);
    }
    if (h->rel_tol > 0.0) std::swap(h->x, h->xprev);  // x_prev = x (:364)
    PassReduce red{h->resp.p, h->bad.p};
    if (half) {
        {
            ProfScope ps(prof, "fft_inv_axis2_half", st);
            fft_engine().axis_pass(hrh, 1, true, h->W2.p, IN_COMPLEX, h->W2.p, OUT_COMPLEX, 1.0, nullptr, st);
        }
        ProfScope ps(prof, "fft_inv_axis3_c2r_half", st);
        fft_engine().c2r_axis3_half(hr, h->W2.p, h->x.p, s, &red, st);
    } else if (a1) {
        {
            ProfScope ps(prof, "fft_inv_axis2", st);
            fft_engine().axis_pass(hr, 1, true, h->W.p, IN_COMPLEX, h->W.p, OUT_COMPLEX, 1.0, nullptr, st);
        }
        ProfScope ps(prof, "fft_inv_axis3_c2r", st);
        fft_engine().axis_pass(hr, 2, true, h->W.p, IN_COMPLEX, h->x.p, OUT_REAL, s, &red, st);
    } else if (fused)
        fft_engine().inverse21(hr, h->W.p, h->x.p, OUT_REAL, s, &red, st, prof);
    else
        fft_engine().inverse3(hr, h->W.p, h->x.p, OUT_REAL, s, &red, st, prof);
    g_fwd += 1;
    g_inv += 1;
    double* din = h->dual_in_a ? h->dualA.p : h->dualB.p;
    double* dout = h->dual_in_a ? h->dualB.p : h->dualA.p;
    // shrink / dual / residual (:379-393) and theta for the next iteration (:367-373)
    {
        ProfScope ps(prof, "tv_stencil", st);
        launch_tv_stencil(hr, false, h->x.p, din, dout, h->theta.p, h->lambda / h->mu,
                          h->rel_tol > 0.0 ? h->xprev.p : nullptr, h->stp.p, st);
    }
    h->dual_in_a = !h->dual_in_a;
    tv_finalize_step(h, prof, a1, half, st);
}

// the iteration's scalar finalize (objective, residual, rel change, residue
// status), on a side stream for fixed-count runs
static void tv_finalize_step(vsr_tv* h, Profiler* prof, bool a1, bool half, cudaStream_t st) {
    const Dims& hr = h->sp.hr;
    const bool fused = use_fused(h->G);
    TvIterScalars sc{h->obj.p, h->res.p, h->rel.p, h->status.p, h->iter_dev.p};
    const bool side = h->rel_tol <= 0.0 && prof == nullptr;
    if (side) {
        if (!h->side) {
            VSR_CUDA(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
            VSR_CUDA(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
            VSR_CUDA(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
        }
        VSR_CUDA(cudaEventRecord(h->ev_fork, st));
        VSR_CUDA(cudaStreamWaitEvent(h->side, h->ev_fork, 0));
    }
    {
        ProfScope ps(prof, "tv_finalize", st);
        launch_tv_finalize((int)h->iters_done, h->fitp.p,
                           half && h->ntiles ? (size_t)h->ntiles
                                             : (a1 ? tv_sandwich1_blocks(h->G)
                                                   : (fused ? tv_sandwich_blocks(h->G) : h->fit_blocks)),
                           h->stp.p, h->st_blocks, h->resp.p,
                           half ? fft_engine().half3_blocks(hr)
                                : (a1 ? fft_engine().pass_blocks(hr, 2) : h->res_blocks),
                           h->lambda, 1e-8, sc, nullptr,
                           side ? h->side : st);
    }
    if (side) {
        VSR_CUDA(cudaEventRecord(h->ev_join, h->side));
        h->fin_pending = true;
    }
    ++h->iters_done;
}

// Fixed-count iterations (rel_tol = 0, profiler off) replay a CUDA graph of
// kTvGraphIters consecutive iterations (a multiple of the ping-pong period 2) (the dual buffers ping-pong with period 2; the
// iteration index lives on the device).  VSR_NO_GRAPH=1 keeps eager launches.
static void tv_iterate(vsr_tv* h, size_t iters) {
    static const bool no_graph = [] {
        const char* e = std::getenv("VSR_NO_GRAPH");
        return e && e[0] == '1';
    }();
    size_t k = 0;
    const bool graphs = !no_graph && h->rel_tol <= 0.0 && h->ctx->prof() == nullptr;
    if (graphs) {
        cudaStream_t st = h->ctx->stream;
        constexpr size_t G = kTvGraphIters;
        while (k + G <= iters && h->iters_done + G <= h->max_iters) {
            if (!h->dual_in_a || h->iters_done == 0) {  // align to the captured parity / warm up
                tv_step(h);
                ++k;
                continue;
            }
            if (!h->gexec) {
                const uint64_t l0 = g_launches.load(), f0 = g_fwd.load(), i0 = g_inv.load();
                const size_t it0 = h->iters_done;
                cudaGraph_t graph = nullptr;
                tv_join(h);  // no cross-capture event waits
                VSR_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
                try {
                    for (size_t q = 0; q < G; ++q) tv_step(h);
                    tv_join(h);  // the side stream rejoins before the capture ends
                } catch (...) {
                    cudaStreamEndCapture(st, &graph);
                    if (graph) cudaGraphDestroy(graph);
                    throw;
                }
                VSR_CUDA(cudaStreamEndCapture(st, &graph));
                const cudaError_t e = cudaGraphInstantiate(&h->gexec, graph, 0);
                cudaGraphDestroy(graph);
                VSR_CUDA(e);
                h->g_kernels = g_launches.load() - l0;
                g_launches.fetch_sub(h->g_kernels);  // counted when the graph runs
                g_fwd.fetch_sub(g_fwd.load() - f0);
                g_inv.fetch_sub(g_inv.load() - i0);
                h->iters_done = it0;  // the captured steps have not run yet
            }
            tv_join(h);  // an eager step's side-stream finalize precedes the graph's fold
            VSR_CUDA(cudaGraphLaunch(h->gexec, st));
            g_launches.fetch_add(h->g_kernels);
            g_fwd += G;
            g_inv += G;
            h->iters_done += G;
            k += G;
        }
    }
    for (; k < iters && !h->stopped && h->iters_done < h->max_iters; ++k) {
        tv_step(h);
        if (h->rel_tol > 0.0) {  // stop test (:405) needs the scalar now
            double rc = 0.0;
            d2h(h->ctx, &rc, h->rel.p + (h->iters_done - 1), sizeof(double));
            sync(h->ctx);
            if (rc < h->rel_tol) h->stopped = true;
        }
    }
    tv_join(h);  // report readers on the main stream see the last iteration's scalars
}

// the iterate as fp64 (fp32 mode: widened on the stream into the fp64 x buffer)
static const double* tv_x_fp64(vsr_tv* h) {
    if (h->f32) launch_widen(h->xf.p, h->x.p, h->x.n, h->ctx->stream);
    return h->x.p;
}

static void tv_fill_report(vsr_tv* h, vsr_report* rep, const char* where) {
    double status[4];
    unsigned long long bad = 0;
    d2h(h->ctx, status, h->status.p, sizeof(status));
    d2h(h->ctx, &bad, h->bad.p, sizeof(bad));
    double init_obj = 0.0;
    d2h(h->ctx, &init_obj, h->init_obj.p, sizeof(double));
    sync(h->ctx);
    if (status[0] >= 0.0) throw numeric_error(residue_message(status[1], 1e-8));
    if (bad != ULLONG_MAX)
        throw numeric_error(std::string(where) + ": non-finite value at flat index " + std::to_string(bad));
    if (rep) {
        rep->iterations = h->iters_done;
        rep->initial_objective = init_obj;
        if (rep->objective) d2h(h->ctx, rep->objective, h->obj.p, h->iters_done * sizeof(double));
        if (rep->primal_residual)
            d2h(h->ctx, rep->primal_residual, h->res.p, h->iters_done * sizeof(double));
        sync(h->ctx);
        rep->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - h->t0).count();
    }
}

// ============================================================ admm_l2l2
// solvers.cpp:95-189, device loop: per iteration t = v - dual, fft3(t),
// x_hat / L x_hat pointwise, two inverse transforms (x, Hx) with the residue
// reductions, the v / dual update with the objective, residual and
// rel-change partials, then a fixed-order finalize.  With rel_tol > 0 the host
// reads rel_change after each iteration (the reference's stop rule, :182).
int vsr_admm_l2l2(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3], const double* y_r,
                  const double* lambda_c, double reg, const double* xbar_r, size_t max_iters,
                  const vsr_l2_config* cfg, double* x_r, vsr_report* report) {
    return guarded([&] {
        require_ctx(ctx);
        const vsr_l2_config def{0.1, 1e-10, nullptr, nullptr, nullptr};
        const vsr_l2_config& c = cfg ? *cfg : def;
        const Spec sp = make_spec(hr_dims, rates);
        require_positive(reg, "lambda");  // solvers.cpp:98-99
        require_positive(c.mu, "mu");
        if (max_iters < 1) throw std::invalid_argument("admm_l2l2: max_iters must be >= 1");
        const bool warm = c.warm_x || c.warm_v || c.warm_dual;
        if (warm && !(c.warm_x && c.warm_v && c.warm_dual))
            throw shape_error("admm_l2l2: warm start: dims mismatch");
        vsr_ctx::Guard g(ctx->device);
        const auto t0 = std::chrono::steady_clock::now();
        cudaStream_t st = ctx->stream;
        const Dims& hr = sp.hr;
        const size_t N = hr.count(), Nl = sp.lr.count();
        DevBuf<double2> lam(N), xbh(N), W(N), W2(N);
        DevBuf<double> y(Nl), xbar(N), x(N), v(N), dual(N), t(N), hx(N), xprev;
        if (c.rel_tol > 0.0) xprev.alloc(N);
        h2d(ctx, lam.p, lambda_c, lam.bytes());
        h2d(ctx, y.p, y_r, y.bytes());
        h2d(ctx, xbar.p, xbar_r, xbar.bytes());
        if (warm) {
            h2d(ctx, x.p, c.warm_x, x.bytes());
            h2d(ctx, v.p, c.warm_v, v.bytes());
            h2d(ctx, dual.p, c.warm_dual, dual.bytes());
        } else {
            VSR_CUDA(cudaMemsetAsync(x.p, 0, x.bytes(), st));
            VSR_CUDA(cudaMemsetAsync(v.p, 0, v.bytes(), st));
            VSR_CUDA(cudaMemsetAsync(dual.p, 0, dual.bytes(), st));
        }
        const double s = inv_sqrt_count(hr);
        fft_engine().forward3(hr, xbar.p, IN_REAL, xbh.p, s, st);  // xbar_hat (:105)
        ++g_fwd;
        const size_t nres = fft_engine().inverse_final_blocks(hr);
        DevBuf<double> up(5 * l2_partial_blocks()), px(2 * nres), ph(2 * nres);
        DevBuf<unsigned long long> bad(1), badh(1);
        DevBuf<double> obj(max_iters), res(max_iters), rel(max_iters), status(2), init_obj(1);
        VSR_CUDA(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), st));
        VSR_CUDA(cudaMemsetAsync(badh.p, 0xff, sizeof(unsigned long long), st));
        VSR_CUDA(cudaMemsetAsync(status.p, 0, 2 * sizeof(double), st));
        const L2Dims D{(long long)hr.m, (long long)hr.n, (long long)hr.s, (long long)N, (long long)sp.lr.m,
                       (long long)sp.lr.n, sp.rates[0], sp.rates[1], sp.rates[2]};
        const L2Scalars sc{obj.p, res.p, rel.p, status.p, init_obj.p};
        PassReduce rx{px.p, bad.p}, rh{ph.p, badh.p};
        // initial objective (:117-129): Hx via fft3 / L / ifft3_real
        fft_engine().forward3(hr, x.p, IN_REAL, W.p, s, st);
        launch_l2_mul(W.p, lam.p, (long long)N, st);
        fft_engine().inverse3(hr, W.p, hx.p, OUT_REAL, s, &rh, st);
        ++g_fwd;
        ++g_inv;
        launch_l2_update(D, false, hx.p, x.p, xbar.p, y.p, v.p, dual.p, nullptr, c.mu, up.p, st);
        launch_l2_finalize(-1, up.p, nullptr, ph.p, (long long)nres, reg, 1e-8, sc, st);
        size_t iters = 0;
        for (size_t it = 0; it < max_iters; ++it) {
            if (xprev.p) VSR_CUDA(cudaMemcpyAsync(xprev.p, x.p, x.bytes(), cudaMemcpyDeviceToDevice, st));
            launch_l2_sub(v.p, dual.p, t.p, (long long)N, st);                 // :139
            fft_engine().forward3(hr, t.p, IN_REAL, W.p, s, st);               // :140
            launch_l2_xhat(W.p, W2.p, lam.p, xbh.p, c.mu, reg, (long long)N, st);  // :141-150
            fft_engine().inverse3(hr, W.p, x.p, OUT_REAL, s, &rx, st);         // :146
            fft_engine().inverse3(hr, W2.p, hx.p, OUT_REAL, s, &rh, st);       // :151
            g_fwd += 1;
            g_inv += 2;
            launch_l2_update(D, true, hx.p, x.p, xbar.p, y.p, v.p, dual.p, xprev.p, c.mu, up.p, st);
            launch_l2_finalize((int)it, up.p, px.p, ph.p, (long long)nres, reg, 1e-8, sc, st);
            iters = it + 1;
            if (c.rel_tol > 0.0) {  // :182
                double rc = 0.0;
                d2h(ctx, &rc, rel.p + it, sizeof(double));
                sync(ctx);
                if (rc < c.rel_tol) break;
            }
        }
        double stv[2];
        unsigned long long b0 = 0, b1 = 0;
        d2h(ctx, stv, status.p, sizeof(stv));
        d2h(ctx, &b0, bad.p, sizeof(b0));
        d2h(ctx, &b1, badh.p, sizeof(b1));
        sync(ctx);
        if (stv[0] != 0.0) throw numeric_error(residue_message(stv[1], 1e-8));
        if (b0 != ULLONG_MAX)  // require_finite(x, "admm_l2l2") (:185)
            throw numeric_error("admm_l2l2: non-finite value at flat index " + std::to_string(b0));
        d2h(ctx, x_r, x.p, x.bytes());
        if (report) {
            report->iterations = iters;
            d2h(ctx, &report->initial_objective, init_obj.p, sizeof(double));
            if (report->objective) d2h(ctx, report->objective, obj.p, iters * sizeof(double));
            if (report->primal_residual) d2h(ctx, report->primal_residual, res.p, iters * sizeof(double));
        }
        sync(ctx);
        if (report) report->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

int vsr_admm_tv(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3], const double* y_r,
                const double* psf_r, const vsr_tv_config* cfg, double* x_r, vsr_report* report) {
    return guarded([&] {
        require_ctx(ctx);
        const Spec sp = make_spec(hr_dims, rates);
        tv_validate(cfg);
        require_nonempty(sp.hr, "fft3");
        vsr_ctx::Guard g(ctx->device);
        const size_t N = sp.hr.count(), Nl = sp.lr.count();
        DevBuf<double> dy(Nl), dpsf(N), dinit;
        h2d(ctx, dy.p, y_r, dy.bytes());
        h2d(ctx, dpsf.p, psf_r, dpsf.bytes());
        if (cfg->init == VSR_INIT_PROVIDED) {
            if (!cfg->init_volume) throw shape_error("admm_tv: init volume: dims mismatch");
            dinit.alloc(N);
            h2d(ctx, dinit.p, cfg->init_volume, dinit.bytes());
        }
        vsr_tv* h = tv_build(ctx, sp, dy.p, dpsf.p, cfg, dinit.p);
        try {
            tv_iterate(h, h->max_iters);
            tv_fill_report(h, report, "admm_tv");
            d2h(ctx, x_r, tv_x_fp64(h), h->x.bytes());
            sync(ctx);
            if (report) report->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - h->t0).count();
        } catch (...) {
            delete h;
            throw;
        }
        delete h;
    });
}

int vsr_tv_create_d(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3],
                    const double* y_r_dev, const double* psf_r_dev, const vsr_tv_config* cfg,
                    vsr_tv** out) {
    return guarded([&] {
        require_ctx(ctx);
        const Spec sp = make_spec(hr_dims, rates);
        tv_validate(cfg);
        require_nonempty(sp.hr, "fft3");
        vsr_ctx::Guard g(ctx->device);
        *out = tv_build(ctx, sp, y_r_dev, psf_r_dev, cfg, cfg->init_volume);
    });
}

int vsr_tv_iterate_d(vsr_tv* h, size_t iters) {
    return guarded([&] {
        vsr_ctx::Guard g(h->ctx->device);
        tv_iterate(h, iters);
    });
}

int vsr_tv_x_d(vsr_tv* h, const double** x_dev) {
    return guarded([&] {
        vsr_ctx::Guard g(h->ctx->device);
        *x_dev = tv_x_fp64(h);
    });
}

int vsr_tv_x_f32_d(vsr_tv* h, const float** x_dev) {
    return guarded([&] {
        if (!h->f32) throw std::invalid_argument("admm_tv: not an fp32-mode handle");
        *x_dev = h->xf.p;
    });
}

int vsr_tv_report(vsr_tv* h, vsr_report* report) {
    return guarded([&] {
        vsr_ctx::Guard g(h->ctx->device);
        tv_fill_report(h, report, "admm_tv");
    });
}

int vsr_tv_destroy(vsr_tv* h) {
    return guarded([&] {
        if (!h) return;
        vsr_ctx::Guard g(h->ctx->device);
        cudaStreamSynchronize(h->ctx->stream);
        delete h;
    });
}

int vsr_tikhonov_separable(vsr_tikhonov* t) { return t && t->sep.t.a ? 1 : 0; }
int vsr_tikhonov_lattice_prior(vsr_tikhonov* t) { return t && t->Zl.p ? 1 : 0; }
int vsr_tikhonov_spatial(vsr_tikhonov* t) { return t && t->spl.ok ? 1 : 0; }
int vsr_tv_separable(vsr_tv* h) { return h && h->sep.t.a ? 1 : 0; }

int vsr_launch_count(uint64_t* out) {
    if (out) *out = g_launches.load(std::memory_order_relaxed);
    return VSR_OK;
}

int vsr_profile_enable(vsr_ctx* ctx, int enable) {
    return guarded([&] {
        require_ctx(ctx);
        ctx->profiling = enable != 0;
    });
}

int vsr_profile_read(vsr_ctx* ctx, int max_stages, char* names, size_t name_len, double* total_ms,
                     uint64_t* launches, int* n_stages) {
    return guarded([&] {
        require_ctx(ctx);
        vsr_ctx::Guard g(ctx->device);
        auto agg = ctx->profiler.drain();
        int n = 0;
        for (auto& a : agg) {
            if (n >= max_stages) break;
            std::strncpy(names + (size_t)n * name_len, a.first.c_str(), name_len - 1);
            names[(size_t)n * name_len + name_len - 1] = 0;
            total_ms[n] = a.second.first;
            launches[n] = a.second.second;
            ++n;
        }
        *n_stages = n;
    });
}

double vsr_tv_algorithmic_bytes(const size_t hr_dims[3], const size_t rates[3]) {
    const double N = (double)hr_dims[0] * hr_dims[1] * hr_dims[2];
    const double d = (double)rates[0] * rates[1] * rates[2];
    return (160.0 + 16.0 / d) * N;
}

}  // extern "C"
