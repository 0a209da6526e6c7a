/* FFTW3-API shim for compiling the reference (oracle/_ref) — TEST INFRASTRUCTURE.
 *
 * The reference links FFTW3 (unpinned version; proj/CMakeLists.txt:16-17),
 * which is absent from this image.  This header declares exactly the subset
 * the reference calls (proj/src/fft.cpp:3,34-38,56): fftw_complex, fftw_plan,
 * fftw_plan_dft_3d, fftw_execute_dft and the FFTW_* flags, with FFTW's
 * published semantics: an UNNORMALISED multidimensional DFT
 *     out[k] = sum_j in[j] * exp(sign * 2*pi*i * sum_a j_a k_a / n_a),
 * row-major with the LAST dimension contiguous.  Backed by a CPU fp64
 * row-column FFT (fftw_shim.cpp).  Not FFTW; results agree with any exact
 * DFT to ~1e-16 relative, which the reference's own FFT tests pin
 * (test_volume.cpp:44-87).
 */
#ifndef VSR_FFTW3_SHIM_H
#define VSR_FFTW3_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct vsr_fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_ESTIMATE (1U << 6)
#define FFTW_UNALIGNED (1U << 1)

fftw_plan fftw_plan_dft_3d(int n0, int n1, int n2, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags);
void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif

#endif
