// C++ callers' view of the B200 path: the reference's own solver tests
// (proj/tests/test_solvers.cpp, test_volume.cpp) restated against the
// header-only mirror include/volsr_b200/volsr.hpp, i.e. the reference API
// backed by libvsr_b200.so.  Run by tests/test_cpp_mirror.py on a GPU.
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "volsr_b200/volsr.hpp"

using namespace volsr;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                          \
    do {                                                                  \
        ++g_checks;                                                       \
        if (!(c)) {                                                       \
            ++g_fail;                                                     \
            std::fprintf(stderr, "%s:%d: CHECK FAILED: %s\n", __FILE__, __LINE__, #c); \
        }                                                                 \
    } while (0)
template <class E, class F>
bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
    }
    return false;
}

static Volume3D random_volume(const Dims3& d, std::mt19937_64& rng, double lo = -1.0, double hi = 1.0) {
    std::uniform_real_distribution<double> u(lo, hi);
    Volume3D v(d);
    for (auto& x : v.data()) x = u(rng);
    return v;
}
static double rel_err(const Volume3D& a, const Volume3D& b) {
    double n = 0, d = 0;
    for (std::size_t p = 0; p < a.size(); ++p) n += (a[p] - b[p]) * (a[p] - b[p]), d += b[p] * b[p];
    return std::sqrt(n) / std::max(std::sqrt(d), 1e-300);
}
static Volume3D random_psf(const Dims3& hr, std::size_t k, std::mt19937_64& rng) {
    std::uniform_real_distribution<double> u(0.0, 1.0);
    std::vector<double> w(k * k * k);
    for (auto& v : w) v = u(rng);
    return make_gaussian_psf(PsfSpec::explicit_kernel({k, k, k}, std::move(w)), hr);
}

int main() {
    {  // test_volume.cpp:44-50
        const Dims3 d{4, 3, 5};
        const ComplexVolume3D sp = fft3(Volume3D(d, 0.75));
        CHECK(std::abs(sp[0] - 0.75 * std::sqrt(60.0)) < 1e-12);
        for (std::size_t p = 1; p < sp.size(); ++p) CHECK(std::abs(sp[p]) < 1e-12);
    }
    {  // test_volume.cpp:52-69 round trip + Parseval
        std::mt19937_64 rng(7);
        for (const Dims3& d : {Dims3{5, 3, 7}, Dims3{4, 6, 2}, Dims3{8, 8, 8}, Dims3{1, 9, 4}}) {
            const Volume3D x = random_volume(d, rng);
            const ComplexVolume3D xh = fft3(x);
            const ComplexVolume3D back = ifft3(xh);
            double num = 0, den = 0, ef = 0;
            for (std::size_t p = 0; p < x.size(); ++p) {
                num += std::norm(back[p] - std::complex<double>(x[p]));
                den += x[p] * x[p];
                ef += std::norm(xh[p]);
            }
            CHECK(std::sqrt(num / den) < 1e-12);
            CHECK(std::abs(ef - den) / den < 1e-12);
        }
    }
    {  // test_volume.cpp:83-87
        std::mt19937_64 rng(3);
        std::uniform_real_distribution<double> u(-1, 1);
        ComplexVolume3D bogus(Dims3{4, 4, 4});
        for (auto& z : bogus.data()) z = {u(rng), u(rng)};
        CHECK(throws<numeric_error>([&] { (void)ifft3_real(bogus, 1e-8); }));
    }
    {  // test_solvers.cpp:55-69
        std::mt19937_64 rng(1);
        const Dims3 d{4, 4, 4};
        const DecimationSpec spec(d, {1, 1, 1});
        SpectrumDiag ones{ComplexVolume3D(d, 1.0)};
        TikhonovConfig cfg;
        cfg.lambda = 0.35;
        cfg.xbar = random_volume(d, rng);
        const Volume3D y = random_volume(d, rng);
        const Volume3D x = tikhonov_fast(y, ones, spec, cfg);
        for (std::size_t p = 0; p < x.size(); ++p) {
            const double want = (y[p] + 2 * 0.35 * cfg.xbar[p]) / (1 + 2 * 0.35);
            CHECK(std::abs(x[p] - want) <= 1e-12 * (1 + std::abs(want)));
        }
    }
    {  // test_solvers.cpp:71-82
        std::mt19937_64 rng(2);
        const Dims3 d{8, 8, 8};
        const DecimationSpec spec(d, {2, 2, 2});
        TikhonovConfig cfg;
        cfg.lambda = 1e6;
        cfg.xbar = random_volume(d, rng);
        const Volume3D y = random_volume(spec.lr(), rng);
        CHECK(rel_err(tikhonov_fast(y, psf_to_spectrum(random_psf(d, 3, rng)), spec, cfg), cfg.xbar) < 1e-4);
    }
    {  // test_solvers.cpp:84-92 bad lambda
        const Dims3 d{4, 4, 4};
        TikhonovConfig cfg;
        cfg.lambda = 0.0;
        cfg.xbar = Volume3D(d);
        CHECK(throws<std::invalid_argument>(
            [&] { tikhonov_fast(Volume3D(d), SpectrumDiag{ComplexVolume3D(d, 1.0)}, DecimationSpec(d, {1, 1, 1}), cfg); }));
        CHECK(throws<shape_error>([&] { DecimationSpec(Dims3{4, 5, 4}, {2, 2, 2}); }));
    }
    {  // test_solvers.cpp:113-139 normal equations
        std::mt19937_64 rng(4);
        const Dims3 d{12, 10, 8};
        const DecimationSpec spec(d, {2, 2, 2});
        const SpectrumDiag lam = psf_to_spectrum(make_gaussian_psf(PsfSpec::gaussian({5, 5, 5}, {1.5, 1.2, 1.0}), d));
        TikhonovConfig cfg;
        cfg.lambda = 0.05;
        cfg.xbar = random_volume(d, rng);
        const Volume3D y = random_volume(spec.lr(), rng);
        const Volume3D x = tikhonov_fast(y, lam, spec, cfg);
        const Volume3D lhs_b = blur_apply(decimate_adjoint(decimate(blur_apply(x, lam), spec), spec), lam, true);
        const Volume3D rhs_b = blur_apply(decimate_adjoint(y, spec), lam, true);
        double res = 0, rn = 0;
        for (std::size_t p = 0; p < x.size(); ++p) {
            const double l = lhs_b[p] + 0.1 * x[p], r = rhs_b[p] + 0.1 * cfg.xbar[p];
            res += (l - r) * (l - r);
            rn += r * r;
        }
        CHECK(std::sqrt(res / rn) < 1e-8);
    }
    {  // test_solvers.cpp:141-157 FFT budget
        std::mt19937_64 rng(5);
        const Dims3 d{8, 8, 8};
        const DecimationSpec spec(d, {2, 2, 2});
        TikhonovConfig cfg;
        cfg.lambda = 0.1;
        cfg.xbar = random_volume(d, rng);
        const TikhonovOperator op(psf_to_spectrum(random_psf(d, 3, rng)), spec, cfg);
        const Volume3D y = random_volume(spec.lr(), rng);
        reset_fft_counters();
        (void)op.solve(y);
        CHECK(fft_counters().forward == 1);
        CHECK(fft_counters().inverse == 1);
    }
    {  // test_solvers.cpp:261-287 shrink closed forms
        const Dims3 d{1, 1, 1};
        auto one = [&](double v) { return Volume3D(d, v); };
        auto o = tv_shrink(one(3.0), one(0.0), one(0.0), 1.0);
        CHECK(std::abs(o[0][0] - 2.0) < 1e-12 && o[1][0] == 0.0 && o[2][0] == 0.0);
        o = tv_shrink(one(0.3), one(0.2), one(0.1), 1.0);
        CHECK(o[0][0] == 0.0 && o[1][0] == 0.0 && o[2][0] == 0.0);
        CHECK(throws<std::invalid_argument>([&] { tv_shrink(one(1.0), one(0.0), one(0.0), -0.5); }));
    }
    {  // test_solvers.cpp:369-384 DC-singular gamma
        CHECK(throws<numeric_error>([&] { make_gamma(finite_diff_spectra(Dims3{4, 4, 4}), 0.0); }));
    }
    {  // test_solvers.cpp:386-401 near-identity ADMM-TV
        std::mt19937_64 rng(12);
        const Dims3 d{12, 12, 12};
        const DecimationSpec spec(d, {1, 1, 1});
        const Volume3D psf = make_gaussian_psf(PsfSpec::gaussian({1, 1, 1}, {0, 0, 0}), d);
        const Volume3D y = random_volume(d, rng, 0.0, 1.0);
        TvAdmmConfig cfg;
        cfg.lambda = 1e-6;
        cfg.mu = 0.1;
        cfg.max_iters = 60;
        cfg.rel_tol = 1e-9;
        auto [x, rep] = admm_tv(y, psf, spec, cfg);
        CHECK(rel_err(x, y) < 1e-3);
        CHECK(rep.objective.back() <= rep.initial_objective);
    }
    {  // test_solvers.cpp:426-452 config validation
        const Dims3 d{8, 8, 8};
        const DecimationSpec spec(d, {2, 2, 2});
        const Volume3D psf = make_gaussian_psf(PsfSpec::gaussian({3, 3, 3}, {1, 1, 1}), d);
        const Volume3D y(spec.lr(), 0.5);
        TvAdmmConfig cfg;
        cfg.max_iters = 2;
        cfg.init = TvAdmmConfig::Init::Provided;
        cfg.init_volume = Volume3D(Dims3{4, 4, 4});
        CHECK(throws<shape_error>([&] { admm_tv(y, psf, spec, cfg); }));
        cfg.init = TvAdmmConfig::Init::Zero;
        cfg.lambda = -1.0;
        CHECK(throws<std::invalid_argument>([&] { admm_tv(y, psf, spec, cfg); }));
    }
    {  // byte-identical outputs across runs (test_cli.cpp:237-268)
        std::mt19937_64 rng(6);
        const Dims3 d{32, 32, 32};
        const DecimationSpec spec(d, {2, 2, 2});
        const Volume3D psf = make_gaussian_psf(PsfSpec::gaussian({5, 5, 5}, {1.5, 1.5, 1.5}), d);
        const Volume3D y = random_volume(spec.lr(), rng, 0.0, 1.0);
        TvAdmmConfig cfg;
        cfg.lambda = 2e-3;
        cfg.mu = 0.05;
        cfg.max_iters = 5;
        cfg.rel_tol = 0.0;
        const auto a = admm_tv(y, psf, spec, cfg), b = admm_tv(y, psf, spec, cfg);
        CHECK(a.first.data() == b.first.data());
        CHECK(a.second.objective == b.second.objective);
    }
    {  // test_solvers.cpp:194-222 admm_l2l2 stays at the exact fixed point
        std::mt19937_64 rng(7);
        const Dims3 d{8, 8, 8};
        const DecimationSpec spec(d, {2, 2, 2});
        const Volume3D psf = make_gaussian_psf(PsfSpec::gaussian({3, 3, 3}, {1, 1, 1}), d);
        const SpectrumDiag lam = psf_to_spectrum(psf);
        TikhonovConfig cfg;
        cfg.lambda = 0.05;
        cfg.xbar = random_volume(d, rng, -1.0, 1.0);
        const Volume3D y = random_volume(spec.lr(), rng, -1.0, 1.0);
        const Volume3D xstar = tikhonov_fast(y, lam, spec, cfg);
        AdmmL2Options opts;
        opts.mu = 0.3;
        opts.rel_tol = 0.0;
        AdmmL2State state;
        state.x = xstar;
        state.v = blur_apply(xstar, lam);
        Volume3D r = decimate(state.v, spec);
        for (std::size_t g = 0; g < r.size(); ++g) r[g] -= y[g];
        state.dual = decimate_adjoint(r, spec);
        for (std::size_t p = 0; p < state.dual.size(); ++p) state.dual[p] /= opts.mu;
        opts.warm_start = state;
        auto [x1, report] = admm_l2l2(y, lam, spec, cfg, 1, opts);
        CHECK(report.iterations == 1);
        CHECK(rel_err(x1, xstar) < 1e-10);
        CHECK(throws<std::invalid_argument>([&] { admm_l2l2(y, lam, spec, cfg, 0); }));
    }
    {  // B200 extensions: the fp32 mode and the slab-sharded solvers through the mirror
        std::mt19937_64 rng(11);
        const Dims3 d{256, 32, 32};
        const DecimationSpec spec(d, {4, 4, 4});
        const Volume3D psf = make_gaussian_psf(PsfSpec::gaussian({5, 5, 5}, {1.5, 1.5, 1.5}), d);
        const Volume3D y = random_volume(spec.lr(), rng, 0.0, 1.0);
        TvAdmmConfig cfg;
        cfg.lambda = 2e-3;
        cfg.mu = 0.05;
        cfg.max_iters = 5;
        cfg.rel_tol = 0.0;
        cfg.tau = 5e-5;
        auto [x64, r64] = admm_tv(y, psf, spec, cfg);
        cfg.precision = TvAdmmConfig::Precision::F32;
        auto [x32, r32] = admm_tv(y, psf, spec, cfg);
        CHECK(r32.iterations == 5);
        CHECK(rel_err(x32, x64) < 1e-5);
        cfg.precision = TvAdmmConfig::Precision::F64;
        // two virtual ranks: the y-slabs joined back are the single-GPU result, bit for bit
        const b200::SlabComm comm = b200::SlabComm::local(2);
        auto [slabs, rs] = b200::admm_tv_sharded(comm, y, psf, spec, cfg);
        CHECK(slabs.size() == 2);
        double maxdiff = 0.0;
        for (int p = 0; p < 2; ++p)
            for (std::size_t k = 0; k < d.s; ++k)
                for (std::size_t j = 0; j < d.n / 2; ++j)
                    for (std::size_t i = 0; i < d.m; ++i)
                        maxdiff = std::max(maxdiff, std::abs(slabs[p].at(i, j, k) - x64.at(i, j + p * d.n / 2, k)));
        CHECK(maxdiff == 0.0);
        CHECK(rs.iterations == 5);
        // Tikhonov: slabs and the fp32 solve on the spatial path
        const Dims3 d2{64, 64, 64};
        const DecimationSpec s2(d2, {2, 2, 2});
        const Volume3D psf2 = make_gaussian_psf(PsfSpec::gaussian({5, 5, 5}, {1.2, 1.2, 1.2}), d2);
        const SpectrumDiag lam = psf_to_spectrum(psf2);
        const Volume3D y2 = random_volume(s2.lr(), rng, 0.0, 1.0);
        TikhonovConfig tc;
        tc.lambda = 1e-3;
        tc.xbar = zero_fill_upsample(y2, s2);
        const TikhonovOperator op(lam, s2, tc);
        const Volume3D xt = op.solve(y2);
        CHECK(op.fp32_ok());
        std::vector<float> yf(y2.data().begin(), y2.data().end());
        const std::vector<float> xf = op.solve_f32(yf);
        double num = 0.0, den = 0.0;
        for (std::size_t q = 0; q < xf.size(); ++q) {
            num += (xf[q] - xt[q]) * (xf[q] - xt[q]);
            den += xt[q] * xt[q];
        }
        CHECK(std::sqrt(num / den) < 1e-5);
        std::vector<Volume3D> xb;
        for (int p = 0; p < 2; ++p) {
            Volume3D v(Dims3{d2.m, d2.n / 2, d2.s});
            for (std::size_t k = 0; k < d2.s; ++k)
                for (std::size_t j = 0; j < d2.n / 2; ++j)
                    for (std::size_t i = 0; i < d2.m; ++i) v.at(i, j, k) = tc.xbar.at(i, j + p * d2.n / 2, k);
            xb.push_back(std::move(v));
        }
        const b200::SlabTikhonovOperator sop(comm, lam, s2, tc.lambda, xb);
        const std::vector<Volume3D> xs = sop.solve(y2);
        double md = 0.0;
        for (int p = 0; p < 2; ++p)
            for (std::size_t k = 0; k < d2.s; ++k)
                for (std::size_t j = 0; j < d2.n / 2; ++j)
                    for (std::size_t i = 0; i < d2.m; ++i)
                        md = std::max(md, std::abs(xs[p].at(i, j, k) - xt.at(i, j + p * d2.n / 2, k)));
        CHECK(md < 1e-12);
    }
    std::printf("checks: %d failed: %d\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
