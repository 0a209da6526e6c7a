// Hand-written fp64 3D FFT engine for sm_100a (replaces FFTW3 in the
// reference: proj/src/fft.cpp:21-101).
//
// A 3D transform is three axis passes.  Each pass is one kernel that moves a
// tile of whole lines HBM -> registers, runs a Stockham radix-16/8/4/2
// decomposition with warp-local register butterflies and shared-memory
// exchanges between stages, and writes the tile back (in place or out of
// place).  Axis 1 is contiguous (lines laid out back to back); axes 2 and 3
// are strided and tiled T consecutive inner indices wide, so every HBM row
// segment is T*16 bytes (128 B for T = 8).
#pragma once

#include <map>
#include <mutex>
#include <vector>

#include "vsr_common.cuh"

namespace vsr {

// IN_HALF / OUT_HALF (strided axes only): the line is Hermitian (the other two
// axes are in the spatial domain of a real volume), so only positions
// q <= L/2 are stored; the rest are conj(X[L - q]).
enum InKind { IN_COMPLEX = 0, IN_REAL = 1, IN_HALF = 2 };
enum OutKind { OUT_COMPLEX = 0, OUT_REAL = 1, OUT_HALF = 2 };

// Deterministic reduction slots written by a pass with OUT_REAL: per-block
// partial sums of (imag^2, |z|^2) and the minimum flat index of a non-finite
// real output (reference ifft3_real src/fft.cpp:84-93 and require_finite
// src/volume.cpp:31-36).
struct PassReduce {
    double* partials = nullptr;               // 2 doubles per block
    unsigned long long* bad_index = nullptr;  // atomicMin target (init ULLONG_MAX)
};

// Slab-sharded half-spectrum planes (slab.cu): plane k of an axis-3 r2c lives
// at peer[owner[k]] + off[k] (complex elements; the rank's rows of that plane
// are contiguous there).  peer == nullptr: the local (m, n, s/2+1) layout.
struct RemotePlanes {
    double2* const* peer = nullptr;
    const int* owner = nullptr;
    const long long* off = nullptr;
};

class FftEngine {
public:
    // Device twiddle table exp(-2*pi*i*j/L), j in [0, L), cached per L.
    const double2* twiddles(size_t L);

    // Number of thread blocks a pass launches (for sizing PassReduce partials).
    size_t pass_blocks(const Dims& d, int axis) const;

    // One pass along `axis` (0 = m, 1 = n, 2 = s).  in/out may alias (in-place).
    // The result of the pass is multiplied by `scale`.
    void axis_pass(const Dims& d, int axis, bool inverse, const void* in, InKind ik, void* out,
                   OutKind ok, double scale, const PassReduce* red, cudaStream_t st);

    // Forward 3D: pass order 1,2,3; first pass in -> out, then in place on out.
    void forward3(const Dims& d, const void* in, InKind ik, double2* out, double scale,
                  cudaStream_t st, Profiler* prof = nullptr);
    // Inverse 3D: pass order 3,2,1; passes 3,2 run IN PLACE on `in` (clobbered),
    // pass 1 writes `out` (complex or real + reduction).
    void inverse3(const Dims& d, double2* in, void* out, OutKind ok, double scale,
                  const PassReduce* red, cudaStream_t st, Profiler* prof = nullptr);

    // Inverse passes 2 then 1 only (axis 3 already done, e.g. by a fused
    // fold kernel): axis 2 in place on `in`, axis 1 writes `out`.
    void inverse21(const Dims& d, double2* in, void* out, OutKind ok, double scale,
                   const PassReduce* red, cudaStream_t st, Profiler* prof = nullptr);
    // Forward passes 1 then 2 only (axis 3 left to a fused kernel).
    void forward12(const Dims& d, const void* in, InKind ik, double2* out, cudaStream_t st,
                   Profiler* prof = nullptr);

    // Real <-> Hermitian half spectrum along axis 3 (planes 0..s/2 of an
    // (m, n, s/2+1) array): forward r2c of a real volume, and the inverse c2r
    // (+ residue reduction) once axes 1 and 2 are back in the spatial domain.
    bool half3_ok(const Dims& d) const;
    size_t half3_blocks(const Dims& d) const;  // blocks (residue partials) of c2r_axis3_half
    void r2c_axis3_half(const Dims& d, const double* in, double2* out, cudaStream_t st);
    void c2r_axis3_half(const Dims& d, const double2* in, double* out, double scale, const PassReduce* red,
                        cudaStream_t st);
    // the same passes with the half-spectrum planes on their owner ranks: the
    // r2c stores each plane into its owner's buffer (peer stores over NVLink),
    // the c2r pulls each plane from its owner (peer loads)
    void r2c_axis3_half_remote(const Dims& d, const double* in, const RemotePlanes& rp, cudaStream_t st);
    void c2r_axis3_half_remote(const Dims& d, const RemotePlanes& rp, double* out, double scale,
                               const PassReduce* red, cudaStream_t st);

    // Blocks of the final (axis-1) pass of inverse3.
    size_t inverse_final_blocks(const Dims& d) const { return pass_blocks(d, 0); }

    // ---- fp32 mode: float2 twiddles, the strided complex pass in place, and
    // the half-spectrum r2c / c2r along axis 3 (fp32 arithmetic)
    const float2* twiddles_f(size_t L);
    void axis_pass_cf(const Dims& d, int axis, bool inverse, float2* inout, cudaStream_t st);
    void r2c_axis3_half_f(const Dims& d, const float* in, float2* out, cudaStream_t st);
    void c2r_axis3_half_f(const Dims& d, const float2* in, float* out, double scale, const PassReduce* red,
                          cudaStream_t st);

private:
    std::mutex mu_;
    std::map<size_t, double2*> tw_;
    std::map<size_t, float2*> twf_;
};

FftEngine& fft_engine();

}  // namespace vsr
