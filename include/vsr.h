/* vsr.h — C ABI of the B200-native volsr reconstruction hot path.
 *
 * Drop-in boundary for the reference's solver path (arxiv 2010.15491, `volsr`
 * C++ library under /root/reference/proj).  Every entry point below names the
 * reference interface it replaces (file:line).  The C++ mirror of the
 * reference API (include/volsr_b200/volsr.hpp) and the Python mirror
 * (paper_2010_15491_b200/volsr.py) are thin layers over these calls.
 *
 * Conventions
 *   - dims[3] = {m, n, s}: axis 1 (m) fastest, flat index i + m*j + m*n*k
 *     (reference include/volsr/volume.hpp:26-45).
 *   - rates[3] = {dr, dc, ds} (reference include/volsr/operators.hpp:12-27).
 *   - Real volumes: double[count]; complex volumes: interleaved (re, im)
 *     double[2*count] (std::complex<double> layout).
 *   - Functions without a `_d` suffix take HOST pointers (pageable or pinned);
 *     `_d` variants take DEVICE pointers on the context's device and are
 *     ordered on the context's stream.
 *   - No exception crosses this boundary: every function returns a status code
 *     and vsr_last_error_message() holds the thread's last message.  The C++
 *     mirror rethrows the reference's exception types by code.
 */
#ifndef VSR_H
#define VSR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (reference error taxonomy, include/volsr/volume.hpp:12-24) */
#define VSR_OK 0
#define VSR_ERR_SHAPE 1        /* volsr::shape_error (std::invalid_argument) */
#define VSR_ERR_INVALID 2      /* std::invalid_argument (lambda <= 0, mu <= 0, ...) */
#define VSR_ERR_NUMERIC 3      /* volsr::numeric_error */
#define VSR_ERR_OUT_OF_RANGE 4 /* std::out_of_range */
#define VSR_ERR_CUDA 5         /* device / runtime failure (no reference analogue) */
#define VSR_ERR_INTERNAL 6
#define VSR_ERR_IO 7           /* volsr::io_error (volume files) */

typedef struct vsr_ctx vsr_ctx;
typedef struct vsr_tikhonov vsr_tikhonov;
typedef struct vsr_folded vsr_folded;
typedef struct vsr_tv vsr_tv;

const char* vsr_last_error_message(void);
int vsr_version(void);

/* ---- context: one device, one stream, cached FFT twiddles and scratch */
int vsr_ctx_create(int device, vsr_ctx** out);
int vsr_ctx_destroy(vsr_ctx* ctx);
int vsr_ctx_synchronize(vsr_ctx* ctx);
void* vsr_ctx_stream(vsr_ctx* ctx); /* cudaStream_t */
int vsr_ctx_device(vsr_ctx* ctx);

/* ---- degrade: replaces volsr::degrade (src/sim.cpp:106-127) and its
 *      gaussian_noise (:88-104).  y = decimate(blur(x, Lambda(psf))) + sigma n
 *      with sigma^2 = var(y) / 10^(bsnr_db / 10) (only when has_bsnr), n the
 *      reference's mt19937_64 + Box-Muller stream for `seed`.  x, psf: HR host
 *      volumes (psf as make_gaussian_psf lays it out); y_out: LR host volume;
 *      sigma_out: the noise sigma (0 without bsnr).  Errors as the reference:
 *      numeric_error for a non-finite y, the ifft3_real residue check. */
int vsr_degrade(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3], const double* x, const double* psf,
                int has_bsnr, double bsnr_db, uint64_t seed, double* y_out, double* sigma_out);

/* ---- volume files: replaces volsr::load_volume / save_volume /
 *      strip_volume_extension (src/volume_io.cpp:27-131, include/volsr/volume_io.hpp).
 *      <base>.volhdr (dims=m,n,s / dtype=f32|f64 / order=lex) + <base>.vol (raw
 *      little-endian scalars, lexicographic).  `path` may carry either extension.
 *      Errors: VSR_ERR_IO (io_error text of the reference), VSR_ERR_SHAPE (buffer
 *      size), VSR_ERR_NUMERIC (save of a non-finite value).  The _d variants
 *      stream the payload between the file and device memory in 32 MB chunks
 *      through two pinned buffers (f32 crosses PCIe narrow and is converted on
 *      the device; the non-finite check runs on the device). */
#define VSR_DTYPE_F64 0
#define VSR_DTYPE_F32 1
int vsr_volume_header(const char* path, size_t dims_out[3], int* dtype_out);
int vsr_load_volume(const char* path, double* out, size_t count);
int vsr_save_volume(const char* path, const size_t dims[3], const double* v, int dtype);
int vsr_load_volume_d(vsr_ctx* ctx, const char* path, double* dev_out, size_t count);
int vsr_save_volume_d(vsr_ctx* ctx, const char* path, const size_t dims[3], const double* dev_in, int dtype);

/* pinned host / device memory helpers (for end-to-end staging) */
int vsr_host_alloc(size_t bytes, void** out);
int vsr_host_free(void* p);
int vsr_device_alloc(vsr_ctx* ctx, size_t bytes, void** out);
int vsr_device_free(vsr_ctx* ctx, void* p);
int vsr_memcpy_h2d(vsr_ctx* ctx, void* dst_dev, const void* src_host, size_t bytes);
int vsr_memcpy_d2h(vsr_ctx* ctx, void* dst_host, const void* src_dev, size_t bytes);

/* ---- FFT contract: replaces volsr::fft3 / ifft3 / ifft3_real /
 *      dft3_unnormalized / fft_counters (include/volsr/fft.hpp:12-31,
 *      src/fft.cpp:50-111).  Unitary 1/sqrt(N), sign -1 forward. */
int vsr_fft3(vsr_ctx* ctx, const size_t dims[3], const double* in_c, double* out_c);
int vsr_fft3_real(vsr_ctx* ctx, const size_t dims[3], const double* in_r, double* out_c);
int vsr_ifft3(vsr_ctx* ctx, const size_t dims[3], const double* in_c, double* out_c);
int vsr_ifft3_real(vsr_ctx* ctx, const size_t dims[3], const double* in_c, double* out_r,
                   double max_rel_imag);
int vsr_dft3_unnormalized(vsr_ctx* ctx, const size_t dims[3], const double* in_r, double* out_c);
int vsr_fft_counters(uint64_t* forward, uint64_t* inverse);
int vsr_reset_fft_counters(void);

/* ---- forward-model operators (include/volsr/operators.hpp:53-87) */
/* psf_to_spectrum == dft3_unnormalized of the padded PSF (src/operators.cpp:121-123) */
int vsr_psf_to_spectrum(vsr_ctx* ctx, const size_t dims[3], const double* psf_r, double* lambda_c);
int vsr_decimate(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3], const double* x,
                 double* y);                                      /* operators.cpp:133-142 */
int vsr_decimate_adjoint(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3],
                         const double* y, double* x);             /* operators.cpp:144-153 */
int vsr_nn_upsample(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3], const double* y,
                    double* x);                                   /* operators.cpp:155-164 */
/* DiffSpectra finite_diff_spectra(hr) (operators.hpp:79-87, operators.cpp:225-243):
 * three complex HR volumes (rows, cols, slices), exactly 0 at DC */
int vsr_finite_diff_spectra(vsr_ctx* ctx, const size_t hr_dims[3], double* rows_c, double* cols_c,
                            double* slices_c);
int vsr_diff_forward(vsr_ctx* ctx, const size_t dims[3], int axis, const double* x,
                     double* out);                                /* operators.cpp:191-206 */
int vsr_diff_adjoint(vsr_ctx* ctx, const size_t dims[3], int axis, const double* x,
                     double* out);                                /* operators.cpp:208-223 */
int vsr_blur_apply(vsr_ctx* ctx, const size_t dims[3], const double* x, const double* lambda_c,
                   int conjugate, double* out);                  /* operators.cpp:125-131 */

/* ---- spectral fold: replaces volsr::FoldedSpectrum / alias_fold / alias_expand /
 *      gram_diag(_weighted) (include/volsr/spectral.hpp:12-68, src/spectral.cpp:7-142) */
int vsr_alias_fold(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3],
                   const double* hr_c, double* lr_c);
int vsr_alias_expand(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3],
                     const double* lr_c, double* hr_c);
int vsr_folded_create(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3],
                      const double* lambda_c, vsr_folded** out);
int vsr_folded_destroy(vsr_folded* f);
/* independent copy of a FoldedSpectrum (the reference type is copyable) */
int vsr_folded_clone(const vsr_folded* src, vsr_folded** out);
int vsr_folded_block_value(vsr_folded* f, size_t br, size_t bc, size_t bs, size_t g,
                           double out_c[2]);
int vsr_folded_apply(vsr_folded* f, const double* hr_c, double* lr_c);
int vsr_folded_apply_adjoint(vsr_folded* f, const double* lr_c, double* hr_c);
int vsr_folded_apply_weighted(vsr_folded* f, const double* hr_c, const double* hr_w, double* lr_c);
int vsr_folded_apply_adjoint_weighted(vsr_folded* f, const double* lr_c, const double* hr_w,
                                      double* hr_c);
int vsr_folded_gram_diag(vsr_folded* f, double* lr_r);
int vsr_folded_gram_diag_weighted(vsr_folded* f, const double* hr_w, double* lr_r);
int vsr_folded_swap_blocks_for_fault_injection(vsr_folded* f);

/* ---- Tikhonov: replaces volsr::TikhonovOperator / tikhonov_fast
 *      (include/volsr/solvers.hpp:27-47, src/solvers.cpp:36-72).
 *      ctor: lambda_c = SpectrumDiag (complex HR), reg = TikhonovConfig::lambda,
 *      xbar = TikhonovConfig::xbar (real HR). */
int vsr_tikhonov_create(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3],
                        const double* lambda_c, double reg, const double* xbar_r,
                        vsr_tikhonov** out);
int vsr_tikhonov_create_d(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3],
                          const double* lambda_c_dev, double reg, const double* xbar_r_dev,
                          vsr_tikhonov** out);
int vsr_tikhonov_destroy(vsr_tikhonov* t);
/* solve(): y = LR real (host) -> x = HR real (host).  Exactly one forward and
 * one inverse 3D transform are counted (test_solvers.cpp:141-157). */
int vsr_tikhonov_solve(vsr_tikhonov* t, const double* y_r, double* x_r);
/* device-resident: enqueue on the context stream; errors are sticky and
 * reported by the next vsr_tikhonov_check (which synchronizes). */
int vsr_tikhonov_solve_d(vsr_tikhonov* t, const double* y_r_dev, double* x_r_dev);
int vsr_tikhonov_check(vsr_tikhonov* t);
/* fp32 mode (no reference analogue; BASELINE north_star's optional fp32 mode):
 * y and x in fp32, the LR stage in fp64, the expansion in fp32 arithmetic.
 * Only on the spatial path (vsr_tikhonov_fp32_ok); VSR_ERR_INVALID otherwise. */
int vsr_tikhonov_solve_f32(vsr_tikhonov* t, const float* y_r, float* x_r);
int vsr_tikhonov_solve_f32_d(vsr_tikhonov* t, const float* y_dev, float* x_dev);
int vsr_tikhonov_fp32_ok(vsr_tikhonov* t);
int vsr_tikhonov_fast(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3],
                      const double* y_r, const double* lambda_c, double reg, const double* xbar_r,
                      double* x_r);
/* bytes the Tikhonov solve moves per call under the compulsory-traffic model
 * (SURVEY §8(d)): (72 + 40/d) * N. */
double vsr_tikhonov_algorithmic_bytes(const size_t hr_dims[3], const size_t rates[3]);

/* ---- TV pieces: replace make_gamma (solvers.hpp:117, solvers.cpp:191-205),
 *      tv_x_update (:89-91, :245-259), tv_shrink (:100-101, :286-301),
 *      objective_tv (:111-112, :303-319). */
int vsr_make_gamma(vsr_ctx* ctx, const size_t hr_dims[3], double tau, double* gamma_r);
/* make_gamma(const DiffSpectra&, tau) (solvers.hpp:117) from explicit spectra;
 * VSR_ERR_NUMERIC with the reference text when a denominator is not positive */
int vsr_make_gamma_spectra(vsr_ctx* ctx, const size_t hr_dims[3], const double* rows_c, const double* cols_c,
                           const double* slices_c, double tau, double* gamma_r);
int vsr_tv_x_update(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3],
                    const double* y_r, const double* lambda_c, double mu,
                    const double* theta_hat_c, const double* gamma_r, double* x_r);
int vsr_tv_shrink(vsr_ctx* ctx, size_t count, const double* nu1, const double* nu2,
                  const double* nu3, double threshold, double* out1, double* out2, double* out3);
int vsr_objective_tv(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3],
                     const double* x_r, const double* y_r, const double* lambda_c,
                     double tv_weight, double* out);

/* ---- ADMM-TV: replaces volsr::admm_tv with TvAdmmConfig / SolveReport
 *      (include/volsr/solvers.hpp:15-21,72-83,106-107; src/solvers.cpp:321-411). */
#define VSR_INIT_ZERO 0
#define VSR_INIT_UPSAMPLED 1
#define VSR_INIT_PROVIDED 2
typedef struct vsr_tv_config {
    double lambda;       /* TV weight (default 0.06) */
    double mu;           /* ADMM penalty (default 0.1) */
    size_t max_iters;    /* default 30 */
    double rel_tol;      /* default 1e-6; 0 = fixed iteration count */
    int has_tau;         /* 0 -> tau = 1e-8 * mu (solvers.cpp:332) */
    double tau;
    int init;            /* VSR_INIT_* */
    const double* init_volume; /* HR real, when init == VSR_INIT_PROVIDED */
    int precision;       /* VSR_PRECISION_F64 (reference, default) or VSR_PRECISION_F32: the
                            iteration state (x, dual, theta, spectra) in fp32 and the transforms
                            and fold in fp32 arithmetic, LR frequency 0 in fp64; needs a
                            separable PSF spectrum and a half-spectrum geometry (no reference
                            analogue: BASELINE north_star's optional fp32 mode) */
} vsr_tv_config;

#define VSR_PRECISION_F64 0
#define VSR_PRECISION_F32 1

typedef struct vsr_report {
    size_t iterations;
    double initial_objective;
    double seconds;
    double* objective;       /* caller-owned, capacity >= max_iters */
    double* primal_residual; /* caller-owned, capacity >= max_iters */
} vsr_report;

int vsr_admm_tv(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3], const double* y_r,
                const double* psf_r, const vsr_tv_config* cfg, double* x_r, vsr_report* report);

/* admm_l2l2 (solvers.hpp:54-70, solvers.cpp:95-189): the iterative l2-l2
 * comparator with the split v = Hx.  Same arithmetic as the reference (one
 * forward and two inverse transforms per iteration); warm start optional (all
 * three of x, v, dual, or none). */
typedef struct vsr_l2_config {
    double mu;                /* default 0.1 */
    double rel_tol;           /* default 1e-10; 0 = fixed iteration count */
    const double* warm_x;     /* HR real, optional */
    const double* warm_v;
    const double* warm_dual;
} vsr_l2_config;

int vsr_admm_l2l2(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3], const double* y_r,
                  const double* lambda_c, double reg, const double* xbar_r, size_t max_iters,
                  const vsr_l2_config* cfg, double* x_r, vsr_report* report);

/* Stepwise ADMM-TV solver over device-resident state (bench / streaming use).
 * create: precompute (psf -> Lambda, y -> LR spectrum, Gamma tables) and the
 * iteration-0 state; iterate(k): k iterations enqueued on the stream. */
int vsr_tv_create_d(vsr_ctx* ctx, const size_t hr_dims[3], const size_t rates[3],
                    const double* y_r_dev, const double* psf_r_dev, const vsr_tv_config* cfg,
                    vsr_tv** out);
int vsr_tv_iterate_d(vsr_tv* h, size_t iters);
int vsr_tv_x_d(vsr_tv* h, const double** x_dev);  /* fp32 mode: x widened into a handle-owned fp64 buffer */
int vsr_tv_x_f32_d(vsr_tv* h, const float** x_dev); /* fp32 mode only: the fp32 iterate itself */
int vsr_tv_report(vsr_tv* h, vsr_report* report); /* synchronizes */
int vsr_tv_destroy(vsr_tv* h);
double vsr_tv_algorithmic_bytes(const size_t hr_dims[3], const size_t rates[3]);

/* unitary-scaled forward 3D FFT of device data (the engine alone; bench/tests) */
int vsr_fft3_d(vsr_ctx* ctx, const size_t dims[3], const double* in, int in_real, double* out_c,
               double scale);

/* ---- slab-sharded solvers over P ranks, one GPU per rank.
 *      Rank p owns HR rows y in [p n/P, (p+1) n/P) of every plane: a slab is
 *      an (m, n/P, s) array.  Spectrally the axis-3 half spectrum is split by
 *      plane over conjugate LR class pairs, so every fold alias set is local;
 *      the exchanges are the kernels' own NVLink peer loads/stores (CUDA IPC)
 *      between stream-ordered barriers.  y (LR) and the PSF / Lambda are
 *      passed in full on every rank; slab arguments are arrays with one entry
 *      per LOCAL rank (1 for NCCL / host comms, P for a local comm).  Every
 *      call is collective over the comm.  Host buffers unless marked _d. */
typedef struct vsr_comm vsr_comm;
typedef struct vsr_slab_tv vsr_slab_tv;
typedef struct vsr_slab_tikhonov vsr_slab_tikhonov;
/* caller-provided exchange (e.g. a gloo process group): both return 0 on success */
typedef struct vsr_host_exchange {
    int (*barrier)(void* user);                                          /* all ranks reached it */
    int (*all_gather)(void* user, const void* send, void* recv, size_t bytes); /* rank order */
} vsr_host_exchange;
/* P virtual ranks in this process on the context's device (stage by stage, stream order) */
int vsr_comm_local(vsr_ctx* ctx, int nranks, vsr_comm** out);
/* one process per GPU over NCCL (libnccl.so.2 loaded at run time); rank 0's id to all */
int vsr_nccl_unique_id(unsigned char out[128]);
int vsr_comm_nccl(vsr_ctx* ctx, int nranks, int rank, const unsigned char id[128], vsr_comm** out);
int vsr_comm_host(vsr_ctx* ctx, int nranks, int rank, const vsr_host_exchange* ops, void* user, vsr_comm** out);
int vsr_comm_destroy(vsr_comm* comm);
int vsr_comm_info(vsr_comm* comm, int* nranks, int* rank /* -1: local comm */, int* local_ranks);
/* plane ownership: owner_half[f3] for f3 = 0..s/2 (may be NULL), planes owned by `rank` */
int vsr_slab_plan(const size_t hr_dims[3], const size_t rates[3], int nranks, int rank, int* owner_half,
                  int* nplanes);
/* admm_tv (solvers.hpp:106-107, solvers.cpp:321-411): cfg->init_volume is
 * ignored, init_slabs carries the Provided init; x_slabs receive x. */
int vsr_slab_admm_tv(vsr_comm* comm, const size_t hr_dims[3], const size_t rates[3], const double* y_r,
                     const double* psf_r, const vsr_tv_config* cfg, const double* const* init_slabs,
                     double* const* x_slabs, vsr_report* report);
int vsr_slab_tv_create(vsr_comm* comm, const size_t hr_dims[3], const size_t rates[3], const double* y_r,
                       const double* psf_r, const vsr_tv_config* cfg, const double* const* init_slabs,
                       vsr_slab_tv** out);
int vsr_slab_tv_iterate(vsr_slab_tv* h, size_t iters);
int vsr_slab_tv_local_ranks(vsr_slab_tv* h, int* count);
int vsr_slab_tv_x_d(vsr_slab_tv* h, int local, const double** x_dev);
/* require_finite + x slabs (may be NULL) + report (may be NULL); synchronizes */
int vsr_slab_tv_finish(vsr_slab_tv* h, double* const* x_slabs, vsr_report* report);
int vsr_slab_tv_destroy(vsr_slab_tv* h);
/* TikhonovOperator (solvers.hpp:27-43): full Lambda (complex HR) on every rank */
int vsr_slab_tikhonov_create(vsr_comm* comm, const size_t hr_dims[3], const size_t rates[3],
                             const double* lambda_c, double reg, const double* const* xbar_slabs,
                             vsr_slab_tikhonov** out);
int vsr_slab_tikhonov_solve(vsr_slab_tikhonov* h, const double* y_r, double* const* x_slabs);
int vsr_slab_tikhonov_solve_d(vsr_slab_tikhonov* h, const double* y_dev);
int vsr_slab_tikhonov_check(vsr_slab_tikhonov* h);
int vsr_slab_tikhonov_x_d(vsr_slab_tikhonov* h, int local, const double** x_dev);
int vsr_slab_tikhonov_destroy(vsr_slab_tikhonov* h);

/* 1 when the operator's blur spectrum was detected separable, Lambda(f) =
 * a[f1] b[f2] c[f3] (any Gaussian PSF): the fused folds then rebuild Lambda
 * from three 1-D tables instead of streaming the 16N-byte HR spectrum. */
int vsr_tikhonov_separable(vsr_tikhonov* t);
/* 1 when the Tikhonov prior xbar lives on the decimation lattice (e.g. the
 * reference CLI default xbar = zero_fill_upsample(y)): fft3(xbar) is then kept
 * as an LR spectrum (16N/d bytes) instead of the HR one (16N). */
int vsr_tikhonov_lattice_prior(vsr_tikhonov* t);
/* 1 when the solve runs as the spatial expansion: separable Lambda with a
 * compact real 1-D PSF factor per axis and a lattice prior.  The alias fold
 * then factors per axis and x = xbar + sqrt(d) H^T D^H F_l^-1(U) is formed in
 * one HBM pass (two LR transforms, no HR transform).  VSR_NO_SPATIAL=1 off. */
int vsr_tikhonov_spatial(vsr_tikhonov* t);
int vsr_tv_separable(vsr_tv* h);

/* ---- instrumentation (bench): kernels launched by this library so far, and
 *      per-stage CUDA-event durations on the context stream when enabled. */
int vsr_launch_count(uint64_t* out);
int vsr_profile_enable(vsr_ctx* ctx, int enable);
/* Drains the recorded stages (synchronizes on their events).  names is a
 * max_stages x name_len char array; total_ms / launches per stage name. */
int vsr_profile_read(vsr_ctx* ctx, int max_stages, char* names, size_t name_len, double* total_ms,
                     uint64_t* launches, int* n_stages);

#ifdef __cplusplus
}
#endif

#endif /* VSR_H */
