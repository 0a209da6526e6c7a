// extern "C" driver over the REFERENCE volsr API, linked into
// oracle/_ref/libvolsr_ref.so together with the reference's own sources
// (compiled where they lie under /root/reference/proj/src by oracle/Makefile).
// TEST INFRASTRUCTURE: used by tests/ (golden vectors, oracle pinning) and by
// bench.py's CPU-baseline / reference arm only.
#include <complex>
#include <cstring>
#include <string>
#include <vector>

#include "volsr/fft.hpp"
#include "volsr/operators.hpp"
#include "volsr/solvers.hpp"
#include "volsr/spectral.hpp"
#include "volsr/volume_io.hpp"
#include "volsr/sim.hpp"

using namespace volsr;

namespace {
thread_local std::string g_err;

template <class F>
int wrap(F&& f) {
    try {
        f();
        return 0;
    } catch (const shape_error& e) {
        g_err = e.what();
        return 1;
    } catch (const numeric_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 4;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 6;
    }
}

Dims3 D(const size_t d[3]) { return Dims3{d[0], d[1], d[2]}; }

Volume3D vol(const size_t d[3], const double* p) {
    const Dims3 dd = D(d);
    return Volume3D(dd, std::vector<double>(p, p + dd.count()));
}

ComplexVolume3D cvol(const size_t d[3], const double* p) {
    const Dims3 dd = D(d);
    const auto* c = reinterpret_cast<const std::complex<double>*>(p);
    return ComplexVolume3D(dd, std::vector<std::complex<double>>(c, c + dd.count()));
}

void put(const Volume3D& v, double* out) { std::memcpy(out, v.data().data(), v.size() * sizeof(double)); }
void put(const ComplexVolume3D& v, double* out) {
    std::memcpy(out, v.data().data(), v.size() * sizeof(std::complex<double>));
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_fft3(const size_t d[3], const double* in_c, double* out_c) {
    return wrap([&] { put(fft3(cvol(d, in_c)), out_c); });
}
int ref_fft3_real(const size_t d[3], const double* in_r, double* out_c) {
    return wrap([&] { put(fft3(vol(d, in_r)), out_c); });
}
int ref_ifft3(const size_t d[3], const double* in_c, double* out_c) {
    return wrap([&] { put(ifft3(cvol(d, in_c)), out_c); });
}
int ref_ifft3_real(const size_t d[3], const double* in_c, double* out_r, double tol) {
    return wrap([&] { put(ifft3_real(cvol(d, in_c), tol), out_r); });
}
int ref_psf_to_spectrum(const size_t d[3], const double* psf, double* out_c) {
    return wrap([&] { put(psf_to_spectrum(vol(d, psf)).values, out_c); });
}
int ref_make_gaussian_psf(const size_t size[3], const double sigma[3], const size_t hr[3], double* out) {
    return wrap([&] {
        put(make_gaussian_psf(PsfSpec::gaussian({size[0], size[1], size[2]}, {sigma[0], sigma[1], sigma[2]}),
                              D(hr)),
            out);
    });
}
int ref_fft_counters(unsigned long long* f, unsigned long long* i) {
    const FftCounters c = fft_counters();
    *f = c.forward;
    *i = c.inverse;
    return 0;
}
void ref_reset_fft_counters() { reset_fft_counters(); }

void* ref_tikhonov_create(const size_t hr[3], const size_t rates[3], const double* lambda_c, double reg,
                          const double* xbar) {
    TikhonovOperator* op = nullptr;
    int rc = wrap([&] {
        DecimationSpec spec(D(hr), {rates[0], rates[1], rates[2]});
        TikhonovConfig cfg;
        cfg.lambda = reg;
        cfg.xbar = vol(hr, xbar);
        op = new TikhonovOperator(SpectrumDiag{cvol(hr, lambda_c)}, spec, cfg);
    });
    return rc == 0 ? op : nullptr;
}
int ref_tikhonov_solve(void* h, const double* y, double* x) {
    return wrap([&] {
        auto* op = static_cast<TikhonovOperator*>(h);
        const Dims3 lr = op->spec().lr();
        const size_t d[3] = {lr.m, lr.n, lr.s};
        put(op->solve(vol(d, y)), x);
    });
}
void ref_tikhonov_destroy(void* h) { delete static_cast<TikhonovOperator*>(h); }

int ref_make_gamma(const size_t hr[3], double tau, double* out) {
    return wrap([&] { put(make_gamma(finite_diff_spectra(D(hr)), tau), out); });
}

int ref_tv_x_update(const size_t hr[3], const size_t rates[3], const double* y, const double* lambda_c,
                    double mu, const double* theta_hat_c, const double* gamma, double* x) {
    return wrap([&] {
        DecimationSpec spec(D(hr), {rates[0], rates[1], rates[2]});
        const SpectrumDiag lam{cvol(hr, lambda_c)};
        const FoldedSpectrum folded(lam, spec);
        const Dims3 lr = spec.lr();
        const size_t dl[3] = {lr.m, lr.n, lr.s};
        put(tv_x_update(vol(dl, y), folded, lam, spec, mu, cvol(hr, theta_hat_c), vol(hr, gamma)), x);
    });
}

int ref_objective_tv(const size_t hr[3], const size_t rates[3], const double* x, const double* y,
                     const double* lambda_c, double w, double* out) {
    return wrap([&] {
        DecimationSpec spec(D(hr), {rates[0], rates[1], rates[2]});
        const Dims3 lr = spec.lr();
        const size_t dl[3] = {lr.m, lr.n, lr.s};
        *out = objective_tv(vol(hr, x), vol(dl, y), SpectrumDiag{cvol(hr, lambda_c)}, spec, w);
    });
}

int ref_admm_tv(const size_t hr[3], const size_t rates[3], const double* y, const double* psf, double lambda,
                double mu, size_t max_iters, double rel_tol, int has_tau, double tau, int init,
                const double* init_vol, double* x_out, double* obj_out, double* res_out, size_t* iters,
                double* init_obj, double* seconds) {
    return wrap([&] {
        DecimationSpec spec(D(hr), {rates[0], rates[1], rates[2]});
        TvAdmmConfig cfg;
        cfg.lambda = lambda;
        cfg.mu = mu;
        cfg.max_iters = max_iters;
        cfg.rel_tol = rel_tol;
        if (has_tau) cfg.tau = tau;
        cfg.init = init == 0 ? TvAdmmConfig::Init::Zero
                             : (init == 1 ? TvAdmmConfig::Init::UpsampledObservation
                                          : TvAdmmConfig::Init::Provided);
        if (init == 2) cfg.init_volume = vol(hr, init_vol);
        const Dims3 lr = spec.lr();
        const size_t dl[3] = {lr.m, lr.n, lr.s};
        auto [x, rep] = admm_tv(vol(dl, y), vol(hr, psf), spec, cfg);
        put(x, x_out);
        for (size_t i = 0; i < rep.iterations; ++i) {
            obj_out[i] = rep.objective[i];
            res_out[i] = rep.primal_residual[i];
        }
        *iters = rep.iterations;
        *init_obj = rep.initial_objective;
        *seconds = rep.seconds;
    });
}

int ref_admm_l2l2(const size_t hr[3], const size_t rates[3], const double* y, const double* lambda_c, double reg,
                  const double* xbar, size_t max_iters, double mu, double rel_tol, double* x_out, double* obj_out,
                  double* res_out, size_t* iters, double* init_obj) {
    return wrap([&] {
        DecimationSpec spec(D(hr), {rates[0], rates[1], rates[2]});
        TikhonovConfig cfg;
        cfg.lambda = reg;
        cfg.xbar = vol(hr, xbar);
        AdmmL2Options opts;
        opts.mu = mu;
        opts.rel_tol = rel_tol;
        const Dims3 lr = spec.lr();
        const size_t dl[3] = {lr.m, lr.n, lr.s};
        auto [x, rep] = admm_l2l2(vol(dl, y), SpectrumDiag{cvol(hr, lambda_c)}, spec, cfg, max_iters, opts);
        put(x, x_out);
        for (size_t i = 0; i < rep.iterations; ++i) {
            obj_out[i] = rep.objective[i];
            res_out[i] = rep.primal_residual[i];
        }
        *iters = rep.iterations;
        *init_obj = rep.initial_objective;
    });
}

// sim.cpp:106-127 (degrade with a Gaussian PsfSpec) for the degrade golden
int ref_degrade(const size_t hr[3], const size_t rates[3], const double* x, const size_t psf_size[3],
                const double psf_sigma[3], int has_bsnr, double bsnr_db, unsigned long long seed, double* y_out,
                double* sigma_out) {
    return wrap([&] {
        DegradationRecipe r{PsfSpec::gaussian({psf_size[0], psf_size[1], psf_size[2]},
                                              {psf_sigma[0], psf_sigma[1], psf_sigma[2]}),
                            DecimationSpec(D(hr), {rates[0], rates[1], rates[2]}),
                            has_bsnr ? std::optional<double>(bsnr_db) : std::nullopt, seed};
        const DegradeResult res = degrade(vol(hr, x), r);
        put(res.y, y_out);
        *sigma_out = res.noise_sigma;
    });
}

// volume_io.cpp:34-131 (save_volume / load_volume) for the file-format goldens
int ref_save_volume(const char* base, const size_t d[3], const double* v, int f32) {
    return wrap([&] {
        Volume3D vol(Dims3{d[0], d[1], d[2]}, std::vector<double>(v, v + d[0] * d[1] * d[2]));
        save_volume(vol, base, f32 ? VolumeDType::f32 : VolumeDType::f64);
    });
}
int ref_load_volume(const char* base, size_t d_out[3], double* out, size_t cap) {
    return wrap([&] {
        const Volume3D v = load_volume(base);
        d_out[0] = v.dims().m, d_out[1] = v.dims().n, d_out[2] = v.dims().s;
        if (v.size() > cap) throw std::invalid_argument("ref_load_volume: buffer too small");
        put(v, out);
    });
}

// sim.cpp:23-73 (make_phantom) and metrics.cpp (psnr) for the acceptance
// criterion-3 test (acceptance_main.cpp:118-153)
int ref_make_phantom(const size_t d[3], int kind, unsigned long long seed, double* out) {
    return wrap([&] {
        const PhantomKind k = kind == 0 ? PhantomKind::NestedEllipsoids
                                        : (kind == 1 ? PhantomKind::RandomSmooth : PhantomKind::Constant);
        put(make_phantom(D(d), k, seed), out);
    });
}

}  // extern "C"
