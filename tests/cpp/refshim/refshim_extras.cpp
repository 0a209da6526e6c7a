// TEST INFRASTRUCTURE for the reference's own doctest suites compiled
// unchanged against the B200 mirror (tests/test_cpp_mirror.py).  The hot path
// (fft3, folds, tikhonov_fast, tv_x_update, admm_tv, ...) comes from
// include/volsr_b200/volsr.hpp over libvsr_b200.so; this file supplies the
// pieces of the reference API the suites also call that are NOT the hot path:
//   * the dense normal-equation and Eq.-8 oracles (reference solvers.cpp:74-93,
//     :261-284, spectral.cpp:163-178), written over the reference's own dense
//     builders (src/dense.cpp, compiled against this shim);
//   * PSNR / MSE (metrics.cpp:9-29);
//   * the phantom and noise generators used to synthesise test inputs
//     (sim.cpp:23-104).
#include <algorithm>
#include <cmath>
#include <limits>
#include <random>

#include "volsr/dense.hpp"
#include "volsr/metrics.hpp"
#include "volsr/sim.hpp"
#include "volsr/solvers.hpp"

namespace volsr {

namespace {
void require_pos(double v, const char* name) {
    if (!(v > 0.0)) throw std::invalid_argument(std::string(name) + " must be positive, got " + std::to_string(v));
}

Volume3D solve_spd(const Eigen::MatrixXd& A, const Eigen::VectorXd& b, const Dims3& dims, const char* what) {
    Eigen::LLT<Eigen::MatrixXd> llt(A);
    if (llt.info() != Eigen::Success) throw numeric_error(std::string(what) + ": system matrix not positive definite");
    return from_eigen(llt.solve(b), dims);
}
}  // namespace

// (DH)^T (DH) x + 2 lambda x = (DH)^T y + 2 lambda xbar
Volume3D dense_tikhonov(const Volume3D& y, const Volume3D& psf, const DecimationSpec& spec,
                        const TikhonovConfig& cfg) {
    require_pos(cfg.lambda, "lambda");
    require_dense_size(spec.hr().count(), "dense_tikhonov");
    require_same_dims(y.dims(), spec.lr(), "dense_tikhonov");
    require_same_dims(cfg.xbar.dims(), spec.hr(), "dense_tikhonov: xbar");
    const Eigen::MatrixXd DH = build_dense_decimation(spec) * build_dense_blur(psf);
    const auto N = static_cast<Eigen::Index>(spec.hr().count());
    const Eigen::MatrixXd A = DH.transpose() * DH + 2.0 * cfg.lambda * Eigen::MatrixXd::Identity(N, N);
    const Eigen::VectorXd b = DH.transpose() * to_eigen(y) + 2.0 * cfg.lambda * to_eigen(cfg.xbar);
    return solve_spd(A, b, spec.hr(), "dense_tikhonov");
}

// (DH)^T (DH) x + mu sum_a L_a^T L_a x + mu tau x = (DH)^T y + mu theta
Volume3D dense_tv_x_update(const Volume3D& y, const Volume3D& psf, const DecimationSpec& spec, double mu,
                           const Volume3D& theta, double tau) {
    require_pos(mu, "mu");
    require_dense_size(spec.hr().count(), "dense_tv_x_update");
    const Eigen::MatrixXd DH = build_dense_decimation(spec) * build_dense_blur(psf);
    const auto N = static_cast<Eigen::Index>(spec.hr().count());
    Eigen::MatrixXd A = DH.transpose() * DH + mu * tau * Eigen::MatrixXd::Identity(N, N);
    for (Axis a : {Axis::Rows, Axis::Cols, Axis::Slices}) {
        const Eigen::MatrixXd L = build_dense_diff(spec.hr(), a);
        A += mu * (L.transpose() * L);
    }
    const Eigen::VectorXd b = DH.transpose() * to_eigen(y) + mu * to_eigen(theta);
    return solve_spd(A, b, spec.hr(), "dense_tv_x_update");
}

// max |F D^T D F^H - K| with K[p, q] = prod_a [f_a(p) = f_a(q) mod l_a] / d_a
// (contiguous frequency blocks)
double verify_eq8(const DecimationSpec& spec) {
    const Dims3& hr = spec.hr();
    require_dense_size(hr.count(), "verify_eq8");
    const Eigen::MatrixXd D = build_dense_decimation(spec);
    const Eigen::MatrixXcd F = build_dense_dft(hr);
    const Eigen::MatrixXd mask = D.transpose() * D;
    const Eigen::MatrixXcd lhs = F * mask * F.adjoint();
    const Dims3& lr = spec.lr();
    const std::size_t rate[3] = {spec.dr(), spec.dc(), spec.ds()};
    const std::size_t len[3] = {lr.m, lr.n, lr.s};
    auto coord = [&](std::size_t p, int a) {
        const std::size_t c[3] = {p % hr.m, (p / hr.m) % hr.n, p / (hr.m * hr.n)};
        return c[a] % len[a];
    };
    double dev = 0.0;
    const std::size_t N = hr.count();
    for (std::size_t p = 0; p < N; ++p)
        for (std::size_t q = 0; q < N; ++q) {
            double k = 1.0;
            for (int a = 0; a < 3; ++a) k *= coord(p, a) == coord(q, a) ? 1.0 / static_cast<double>(rate[a]) : 0.0;
            dev = std::max(dev, std::abs(lhs(static_cast<Eigen::Index>(p), static_cast<Eigen::Index>(q)) - k));
        }
    return dev;
}

double mse(const Volume3D& a, const Volume3D& b) {
    require_same_dims(a.dims(), b.dims(), "mse");
    double acc = 0.0;
    for (std::size_t p = 0; p < a.size(); ++p) acc += (a[p] - b[p]) * (a[p] - b[p]);
    return acc / static_cast<double>(a.size());
}

double psnr(const Volume3D& reference, const Volume3D& estimate, std::optional<double> peak) {
    require_same_dims(reference.dims(), estimate.dims(), "psnr");
    const double p = peak ? *peak : *std::max_element(reference.data().begin(), reference.data().end());
    if (p <= 0.0) throw std::invalid_argument("psnr: peak must be positive");
    const double e = mse(reference, estimate);
    if (e == 0.0) return std::numeric_limits<double>::infinity();
    return 10.0 * std::log10(p * p / e);
}

Volume3D gaussian_noise(const Dims3& dims, std::uint64_t seed) {
    std::mt19937_64 gen(seed);
    auto u = [&gen]() { return (static_cast<double>(gen() >> 11) + 1.0) * 0x1p-53; };  // (0, 1]
    const double two_pi = 2.0 * 3.14159265358979323846;
    Volume3D out(dims);
    for (std::size_t p = 0; p < out.size(); p += 2) {
        const double u1 = u(), u2 = u();
        const double r = std::sqrt(-2.0 * std::log(u1));
        out[p] = r * std::cos(two_pi * u2);
        if (p + 1 < out.size()) out[p + 1] = r * std::sin(two_pi * u2);
    }
    return out;
}

namespace {
double centred(std::size_t i, std::size_t len) { return 2.0 * (static_cast<double>(i) + 0.5) / static_cast<double>(len) - 1.0; }

// three nested bodies on [-1, 1]^3; later ones overwrite earlier ones
Volume3D ellipsoid_stack(const Dims3& d) {
    if (d.m < 8 || d.n < 8 || d.s < 8) throw std::invalid_argument("make_phantom: nested-ellipsoids needs dims >= 8 per axis");
    struct Body {
        double c[3], r[3], v;
    };
    static const Body bodies[3] = {{{0.0, 0.0, 0.0}, {0.88, 0.82, 0.92}, 1.00},
                                   {{0.1, -0.08, 0.0}, {0.40, 0.36, 0.50}, 0.45},
                                   {{0.0, 0.0, 0.05}, {0.14, 0.14, 0.80}, 0.05}};
    Volume3D v(d, 0.0);
    for (std::size_t k = 0; k < d.s; ++k)
        for (std::size_t j = 0; j < d.n; ++j)
            for (std::size_t i = 0; i < d.m; ++i) {
                const double x[3] = {centred(i, d.m), centred(j, d.n), centred(k, d.s)};
                double val = 0.0;
                for (const Body& b : bodies) {
                    double r2 = 0.0;
                    for (int a = 0; a < 3; ++a) {
                        const double t = (x[a] - b.c[a]) / b.r[a];
                        r2 += t * t;
                    }
                    if (r2 <= 1.0) val = b.v;
                }
                v.at(i, j, k) = val;
            }
    return v;
}

// seeded Gaussian noise blurred by a Gaussian of sigma max(1, min_axis / 16), rescaled to [0, 1]
Volume3D smooth_noise(const Dims3& d, std::uint64_t seed) {
    const Volume3D noise = gaussian_noise(d, seed);
    const double sigma = std::max(1.0, static_cast<double>(std::min({d.m, d.n, d.s})) / 16.0);
    std::size_t k = static_cast<std::size_t>(std::lround(4.0 * sigma)) | 1;
    k = std::min({k, d.m, d.n, d.s});
    if (k % 2 == 0) --k;
    const Volume3D psf = make_gaussian_psf(PsfSpec::gaussian({k, k, k}, {sigma, sigma, sigma}), d);
    Volume3D v = blur_apply(noise, psf_to_spectrum(psf));
    const auto [lo, hi] = std::minmax_element(v.data().begin(), v.data().end());
    const double a = *lo, range = *hi > *lo ? *hi - *lo : 1.0;
    for (auto& x : v.data()) x = (x - a) / range;
    return v;
}
}  // namespace

Volume3D make_phantom(const Dims3& dims, PhantomKind kind, std::uint64_t seed, double constant_value) {
    if (dims.count() == 0) throw std::invalid_argument("make_phantom: empty dims");
    switch (kind) {
        case PhantomKind::Constant: return Volume3D(dims, constant_value);
        case PhantomKind::NestedEllipsoids: return ellipsoid_stack(dims);
        case PhantomKind::RandomSmooth: return smooth_noise(dims, seed);
    }
    throw std::invalid_argument("make_phantom: unknown kind");
}

}  // namespace volsr
