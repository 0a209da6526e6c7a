// Common device/host utilities for the volsr B200 path.
// Layout contract (reference include/volsr/volume.hpp:26-45): a volume with
// dims (m, n, s) is stored lexicographically, axis 1 (m) fastest; complex
// values are interleaved (re, im) doubles, i.e. double2.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstddef>
#include <stdexcept>
#include <string>

namespace vsr {

// Error taxonomy mirrored from the reference (volume.hpp:12-24) plus a device
// failure class.  The C ABI maps each to a status code (include/vsr.h).
struct shape_error : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct numeric_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct io_error : std::runtime_error {  // volume.hpp:22 (volume files)
    using std::runtime_error::runtime_error;
};

#define VSR_CUDA(call)                                                                   \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            throw ::vsr::cuda_error(std::string("CUDA error ") + cudaGetErrorString(e_) + \
                                    " at " __FILE__ ":" + std::to_string(__LINE__));     \
    } while (0)

// Every kernel launch site is followed by VSR_LAUNCH_CHECK(), which also
// counts the launch (reported through vsr_launch_count for the bench).
void note_launch();
#define VSR_LAUNCH_CHECK()               \
    do {                                 \
        VSR_CUDA(cudaGetLastError());    \
        ::vsr::note_launch();            \
    } while (0)

// Optional per-stage CUDA-event profiler (bench roofline): stages record an
// event pair on the launching stream; durations are read after a sync.
struct Profiler {
    virtual ~Profiler() = default;
    virtual void begin(const char* name, cudaStream_t st) = 0;
    virtual void end(cudaStream_t st) = 0;
};
struct ProfScope {
    Profiler* p;
    cudaStream_t st;
    ProfScope(Profiler* prof, const char* name, cudaStream_t s) : p(prof), st(s) {
        if (p) p->begin(name, st);
    }
    ~ProfScope() {
        if (p) p->end(st);
    }
};

struct Dims {
    size_t m = 0, n = 0, s = 0;
    size_t count() const { return m * n * s; }
    bool operator==(const Dims& o) const { return m == o.m && n == o.n && s == o.s; }
    size_t len(int axis) const { return axis == 0 ? m : (axis == 1 ? n : s); }
};

inline std::string to_string(const Dims& d) {
    return std::to_string(d.m) + "x" + std::to_string(d.n) + "x" + std::to_string(d.s);
}

inline bool is_pow2(size_t v) { return v && !(v & (v - 1)); }

// ---------------------------------------------------------------- complex ops
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// conj(a) * b
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
    return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double cnorm(double2 a) { return a.x * a.x + a.y * a.y; }

// fp32 (float2) overloads for the optional fp32 mode
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
    return make_float2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__device__ __forceinline__ float cnorm(float2 a) { return a.x * a.x + a.y * a.y; }

// complex-type traits: the FFT core and the fp32-capable kernels are
// templated on C = double2 (reference precision) or float2 (fp32 mode)
template <class C>
struct CplxT;
template <>
struct CplxT<double2> {
    using real = double;
    __host__ __device__ static __forceinline__ double2 make(double x, double y) { return make_double2(x, y); }
};
template <>
struct CplxT<float2> {
    using real = float;
    __host__ __device__ static __forceinline__ float2 make(float x, float y) { return make_float2(x, y); }
};
template <class C>
__device__ __forceinline__ C cmake(typename CplxT<C>::real x, typename CplxT<C>::real y) {
    return CplxT<C>::make(x, y);
}
__device__ __forceinline__ double2 to_d2(double2 a) { return a; }
__device__ __forceinline__ double2 to_d2(float2 a) { return make_double2(a.x, a.y); }
template <class C>
__device__ __forceinline__ C from_d2(double2 a) {
    return cmake<C>((typename CplxT<C>::real)a.x, (typename CplxT<C>::real)a.y);
}

// ------------------------------------------------- deterministic block reduce
// Fixed-order tree: warp shuffle tree, then warp 0 reduces the per-warp sums in
// warp order.  Same launch geometry => bit-identical result run to run.
template <int NV>
__device__ __forceinline__ void block_reduce_sum(double (&v)[NV], double* smem /* >= 32*NV */) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], off);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = (blockDim.x + 31) >> 5;
    __syncthreads();
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) smem[warp * NV + k] = v[k];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            double t = lane < nwarps ? smem[lane * NV + k] : 0.0;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) t += __shfl_down_sync(0xffffffffu, t, off);
            v[k] = t;
        }
    }
}

// ------------------------------------------------- reciprocal of a positive
// 1/x for x > 0: MUFU.RCP64H seed and two Newton steps (~1 ulp), cheaper than
// the IEEE division sequence.  The seed flushes subnormal x to 0 (-> inf), so
// x below DBL_MIN (a denominator |Lambda|^2 + 2 reg d with a subnormal reg)
// takes the IEEE division instead.
__device__ __forceinline__ double rcp_pos(double x) {
    if (x < 2.2250738585072014e-308) return 1.0 / x;
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = y * fma(-x, y, 2.0);
    y = y * fma(-x, y, 2.0);
    return y;
}
// The same for x known to be normal (>= DBL_MIN, checked by the caller on the
// host): no slow-path branch, so independent reciprocals interleave.
__device__ __forceinline__ double rcp_pos_normal(double x) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    y = y * fma(-x, y, 2.0);
    y = y * fma(-x, y, 2.0);
    return y;
}

}  // namespace vsr
