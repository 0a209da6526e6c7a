// volsr_b200/volsr.hpp — header-only C++ mirror of the reference `volsr`
// solver API (include/volsr/{volume,fft,operators,spectral,solvers}.hpp under
// /root/reference/proj) over the C ABI in vsr.h.  Same namespace, type and
// function names, argument meaning and exception types, so callers written
// against the reference compile unchanged against this header and link
// libvsr_b200.so instead of the CPU library.
//
// Every numeric step runs on the GPU (one process-wide context on device
// VSR_DEVICE, default 0); there is no CPU fallback.
#pragma once

#include <array>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdlib>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../vsr.h"

namespace volsr {

// ------------------------------------------------------------- volume.hpp:12-104
struct shape_error : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct numeric_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct io_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct Dims3 {
    std::size_t m = 0, n = 0, s = 0;
    std::size_t count() const { return m * n * s; }
    bool operator==(const Dims3&) const = default;
};

inline std::string to_string(const Dims3& d) {
    return std::to_string(d.m) + "x" + std::to_string(d.n) + "x" + std::to_string(d.s);
}

inline std::size_t lex_index(std::size_t i, std::size_t j, std::size_t k, const Dims3& d) {
    if (i >= d.m || j >= d.n || k >= d.s)
        throw std::out_of_range("lex_index: voxel (" + std::to_string(i) + "," + std::to_string(j) + "," +
                                std::to_string(k) + ") outside grid " + to_string(d));
    return i + d.m * j + d.m * d.n * k;
}

class Volume3D {
public:
    Volume3D() = default;
    explicit Volume3D(const Dims3& dims, double fill = 0.0) : dims_(dims), data_(dims.count(), fill) {}
    Volume3D(const Dims3& dims, std::vector<double> data) : dims_(dims), data_(std::move(data)) {
        if (data_.size() != dims_.count())
            throw shape_error("Volume3D: data length " + std::to_string(data_.size()) +
                              " does not match dims " + to_string(dims_));
    }
    const Dims3& dims() const { return dims_; }
    std::size_t size() const { return data_.size(); }
    double operator[](std::size_t p) const { return data_[p]; }
    double& operator[](std::size_t p) { return data_[p]; }
    double at(std::size_t i, std::size_t j, std::size_t k) const { return data_[lex_index(i, j, k, dims_)]; }
    double& at(std::size_t i, std::size_t j, std::size_t k) { return data_[lex_index(i, j, k, dims_)]; }
    const std::vector<double>& data() const { return data_; }
    std::vector<double>& data() { return data_; }

private:
    Dims3 dims_;
    std::vector<double> data_;
};

class ComplexVolume3D {
public:
    using value_type = std::complex<double>;
    ComplexVolume3D() = default;
    explicit ComplexVolume3D(const Dims3& dims, value_type fill = {}) : dims_(dims), data_(dims.count(), fill) {}
    ComplexVolume3D(const Dims3& dims, std::vector<value_type> data) : dims_(dims), data_(std::move(data)) {
        if (data_.size() != dims_.count())
            throw shape_error("ComplexVolume3D: data length " + std::to_string(data_.size()) +
                              " does not match dims " + to_string(dims_));
    }
    const Dims3& dims() const { return dims_; }
    std::size_t size() const { return data_.size(); }
    value_type operator[](std::size_t p) const { return data_[p]; }
    value_type& operator[](std::size_t p) { return data_[p]; }
    value_type at(std::size_t i, std::size_t j, std::size_t k) const { return data_[lex_index(i, j, k, dims_)]; }
    value_type& at(std::size_t i, std::size_t j, std::size_t k) { return data_[lex_index(i, j, k, dims_)]; }
    const std::vector<value_type>& data() const { return data_; }
    std::vector<value_type>& data() { return data_; }

private:
    Dims3 dims_;
    std::vector<value_type> data_;
};

inline void require_same_dims(const Dims3& a, const Dims3& b, const char* where) {
    if (!(a == b)) throw shape_error(std::string(where) + ": dims mismatch, " + to_string(a) + " vs " + to_string(b));
}

// volume.hpp:106-116: value-type helpers on host containers (caller-side
// checks and norms of returned volumes; the solvers never route through them)
inline void require_finite(const Volume3D& v, const char* where) {
    for (std::size_t p = 0; p < v.size(); ++p)
        if (!std::isfinite(v[p]))
            throw numeric_error(std::string(where) + ": non-finite value at flat index " + std::to_string(p));
}
inline double dot(const Volume3D& a, const Volume3D& b) {
    require_same_dims(a.dims(), b.dims(), "dot");
    double acc = 0.0;
    for (std::size_t p = 0; p < a.size(); ++p) acc += a[p] * b[p];
    return acc;
}
inline double norm2(const Volume3D& a) { return std::sqrt(dot(a, a)); }
inline std::complex<double> dot(const ComplexVolume3D& a, const ComplexVolume3D& b) {  // conj(a) . b
    require_same_dims(a.dims(), b.dims(), "dot");
    std::complex<double> acc = 0.0;
    for (std::size_t p = 0; p < a.size(); ++p) acc += std::conj(a[p]) * b[p];
    return acc;
}
inline double norm2(const ComplexVolume3D& a) {
    double acc = 0.0;
    for (std::size_t p = 0; p < a.size(); ++p) acc += std::norm(a[p]);
    return std::sqrt(acc);
}
inline ComplexVolume3D to_complex(const Volume3D& v) {
    ComplexVolume3D out(v.dims());
    for (std::size_t p = 0; p < v.size(); ++p) out[p] = v[p];
    return out;
}

// ------------------------------------------------------------- C ABI plumbing
namespace detail {
inline vsr_ctx* ctx() {
    static vsr_ctx* c = [] {
        vsr_ctx* p = nullptr;
        const char* e = std::getenv("VSR_DEVICE");
        const int rc = vsr_ctx_create(e ? std::atoi(e) : 0, &p);
        if (rc != VSR_OK) throw std::runtime_error(vsr_last_error_message());
        return p;
    }();
    return c;
}
inline void check(int rc) {
    if (rc == VSR_OK) return;
    const std::string m = vsr_last_error_message();
    switch (rc) {
        case VSR_ERR_SHAPE: throw shape_error(m);
        case VSR_ERR_INVALID: throw std::invalid_argument(m);
        case VSR_ERR_NUMERIC: throw numeric_error(m);
        case VSR_ERR_OUT_OF_RANGE: throw std::out_of_range(m);
        case VSR_ERR_IO: throw io_error(m);
        default: throw std::runtime_error(m);
    }
}
struct D3 {
    std::size_t v[3];
    explicit D3(const Dims3& d) : v{d.m, d.n, d.s} {}
};
inline const double* cp(const ComplexVolume3D& v) { return reinterpret_cast<const double*>(v.data().data()); }
inline double* cp(ComplexVolume3D& v) { return reinterpret_cast<double*>(v.data().data()); }
}  // namespace detail

// ------------------------------------------------------------- fft.hpp:12-31
inline ComplexVolume3D fft3(const Volume3D& v) {
    ComplexVolume3D out(v.dims());
    detail::check(vsr_fft3_real(detail::ctx(), detail::D3(v.dims()).v, v.data().data(), detail::cp(out)));
    return out;
}
inline ComplexVolume3D fft3(const ComplexVolume3D& v) {
    ComplexVolume3D out(v.dims());
    detail::check(vsr_fft3(detail::ctx(), detail::D3(v.dims()).v, detail::cp(v), detail::cp(out)));
    return out;
}
inline ComplexVolume3D ifft3(const ComplexVolume3D& v) {
    ComplexVolume3D out(v.dims());
    detail::check(vsr_ifft3(detail::ctx(), detail::D3(v.dims()).v, detail::cp(v), detail::cp(out)));
    return out;
}
inline Volume3D ifft3_real(const ComplexVolume3D& v, double max_rel_imag = 1e-8) {
    Volume3D out(v.dims());
    detail::check(vsr_ifft3_real(detail::ctx(), detail::D3(v.dims()).v, detail::cp(v), out.data().data(),
                                 max_rel_imag));
    return out;
}
inline ComplexVolume3D dft3_unnormalized(const Volume3D& v) {
    ComplexVolume3D out(v.dims());
    detail::check(vsr_dft3_unnormalized(detail::ctx(), detail::D3(v.dims()).v, v.data().data(), detail::cp(out)));
    return out;
}
struct FftCounters {
    std::uint64_t forward = 0, inverse = 0;
};
inline FftCounters fft_counters() {
    FftCounters c;
    uint64_t f = 0, i = 0;
    vsr_fft_counters(&f, &i);
    c.forward = f;
    c.inverse = i;
    return c;
}
inline void reset_fft_counters() { vsr_reset_fft_counters(); }

// ------------------------------------------------------------- operators.hpp:12-87
class DecimationSpec {
public:
    DecimationSpec(const Dims3& hr, std::array<std::size_t, 3> rates) : hr_(hr), rates_(rates) {
        const char* names[3] = {"1 (rows)", "2 (cols)", "3 (slices)"};
        const std::size_t ext[3] = {hr.m, hr.n, hr.s};
        for (int a = 0; a < 3; ++a) {
            if (rates[a] == 0) throw shape_error(std::string("DecimationSpec: zero rate on axis ") + names[a]);
            if (ext[a] % rates[a] != 0)
                throw shape_error("DecimationSpec: rate " + std::to_string(rates[a]) + " does not divide axis " +
                                  names[a] + " of length " + std::to_string(ext[a]));
        }
        lr_ = {hr.m / rates[0], hr.n / rates[1], hr.s / rates[2]};
    }
    const Dims3& hr() const { return hr_; }
    const Dims3& lr() const { return lr_; }
    std::size_t dr() const { return rates_[0]; }
    std::size_t dc() const { return rates_[1]; }
    std::size_t ds() const { return rates_[2]; }
    std::size_t rate() const { return rates_[0] * rates_[1] * rates_[2]; }
    const std::size_t* rates_ptr() const { return rates_.data(); }

private:
    Dims3 hr_, lr_;
    std::array<std::size_t, 3> rates_;
};

struct SpectrumDiag {
    ComplexVolume3D values;
    const Dims3& dims() const { return values.dims(); }
};

// PSF description and host-side construction (operators.cpp:23-119; setup, not hot path)
struct PsfSpec {
    std::array<std::size_t, 3> size{1, 1, 1};
    std::array<double, 3> sigma{0.0, 0.0, 0.0};
    std::vector<double> weights;
    static PsfSpec gaussian(std::array<std::size_t, 3> size, std::array<double, 3> sigma) {
        PsfSpec s;
        s.size = size;
        s.sigma = sigma;
        return s;
    }
    static PsfSpec explicit_kernel(std::array<std::size_t, 3> size, std::vector<double> w) {
        if (w.size() != size[0] * size[1] * size[2])
            throw std::invalid_argument("PsfSpec: weight count does not match kernel size");
        double sum = 0.0;
        for (double v : w) {
            if (!(v >= 0.0)) throw std::invalid_argument("PsfSpec: weights must be nonnegative");
            sum += v;
        }
        if (sum <= 0.0) throw std::invalid_argument("PsfSpec: weights must not all be zero");
        for (double& v : w) v /= sum;
        PsfSpec s;
        s.size = size;
        s.weights = std::move(w);
        return s;
    }
};

inline Volume3D make_gaussian_psf(const PsfSpec& spec, const Dims3& hr) {
    const std::size_t ext[3] = {hr.m, hr.n, hr.s};
    for (int a = 0; a < 3; ++a) {
        if (spec.size[a] % 2 == 0)
            throw std::invalid_argument("make_gaussian_psf: kernel size must be odd on axis " + std::to_string(a + 1));
        if (spec.size[a] > ext[a])
            throw std::invalid_argument("make_gaussian_psf: kernel size " + std::to_string(spec.size[a]) +
                                        " exceeds volume axis " + std::to_string(a + 1) + " of length " +
                                        std::to_string(ext[a]));
    }
    const std::size_t kr = spec.size[0], kc = spec.size[1], ks = spec.size[2];
    std::vector<double> k(kr * kc * ks);
    if (!spec.weights.empty()) {
        k = spec.weights;
    } else {
        auto g1 = [](std::size_t n, double sg) {
            std::vector<double> w(n);
            const long h = (long)(n / 2);
            for (long t = -h; t <= h; ++t)
                w[(std::size_t)(t + h)] = sg <= 0.0 ? (t == 0 ? 1.0 : 0.0) : std::exp(-0.5 * (t / sg) * (t / sg));
            return w;
        };
        const auto wr = g1(kr, spec.sigma[0]), wc = g1(kc, spec.sigma[1]), ws = g1(ks, spec.sigma[2]);
        double sum = 0.0;
        for (std::size_t c = 0; c < ks; ++c)
            for (std::size_t b = 0; b < kc; ++b)
                for (std::size_t a = 0; a < kr; ++a) sum += (k[a + kr * b + kr * kc * c] = wr[a] * wc[b] * ws[c]);
        for (double& v : k) v /= sum;
    }
    Volume3D psf(hr);
    for (std::size_t c = 0; c < ks; ++c)
        for (std::size_t b = 0; b < kc; ++b)
            for (std::size_t a = 0; a < kr; ++a) {
                const std::size_t i = (std::size_t)(((long)a - (long)(kr / 2) + (long)hr.m) % (long)hr.m);
                const std::size_t j = (std::size_t)(((long)b - (long)(kc / 2) + (long)hr.n) % (long)hr.n);
                const std::size_t l = (std::size_t)(((long)c - (long)(ks / 2) + (long)hr.s) % (long)hr.s);
                psf.at(i, j, l) += k[a + kr * b + kr * kc * c];
            }
    return psf;
}

// ------------------------------------------------------------- sim.hpp:26-41
struct DegradationRecipe {
    PsfSpec psf;
    DecimationSpec spec;
    std::optional<double> bsnr_db;
    std::uint64_t rng_seed = 0;
};
struct DegradeResult {
    Volume3D y;
    double noise_sigma = 0.0;
};
inline DegradeResult degrade(const Volume3D& x, const DegradationRecipe& recipe) {
    require_same_dims(x.dims(), recipe.spec.hr(), "degrade");
    const Volume3D psf = make_gaussian_psf(recipe.psf, recipe.spec.hr());
    const detail::D3 hr(recipe.spec.hr());
    const std::size_t r[3] = {recipe.spec.dr(), recipe.spec.dc(), recipe.spec.ds()};
    DegradeResult out;
    out.y = Volume3D(recipe.spec.lr());
    detail::check(vsr_degrade(detail::ctx(), hr.v, r, x.data().data(), psf.data().data(), recipe.bsnr_db.has_value(),
                              recipe.bsnr_db.value_or(0.0), recipe.rng_seed, out.y.data().data(), &out.noise_sigma));
    return out;
}

// ------------------------------------------------------------- volume_io.hpp
enum class VolumeDType { f32, f64 };

inline std::string strip_volume_extension(const std::string& path) {
    auto ends = [&](const char* e) {
        const std::string x(e);
        return path.size() >= x.size() && path.compare(path.size() - x.size(), x.size(), x) == 0;
    };
    if (ends(".volhdr")) return path.substr(0, path.size() - 7);
    if (ends(".vol")) return path.substr(0, path.size() - 4);
    return path;
}

inline void save_volume(const Volume3D& v, const std::string& base, VolumeDType dtype = VolumeDType::f64) {
    const detail::D3 d(v.dims());
    detail::check(vsr_save_volume(base.c_str(), d.v, v.data().data(),
                                  dtype == VolumeDType::f32 ? VSR_DTYPE_F32 : VSR_DTYPE_F64));
}

inline Volume3D load_volume(const std::string& base) {
    std::size_t d[3];
    int t = 0;
    detail::check(vsr_volume_header(base.c_str(), d, &t));
    Volume3D v(Dims3{d[0], d[1], d[2]});
    detail::check(vsr_load_volume(base.c_str(), v.data().data(), v.size()));
    return v;
}

inline SpectrumDiag psf_to_spectrum(const Volume3D& psf) { return SpectrumDiag{dft3_unnormalized(psf)}; }

inline Volume3D blur_apply(const Volume3D& x, const SpectrumDiag& lambda, bool conjugate = false) {
    require_same_dims(x.dims(), lambda.dims(), "blur_apply");
    Volume3D out(x.dims());
    detail::check(vsr_blur_apply(detail::ctx(), detail::D3(x.dims()).v, x.data().data(), detail::cp(lambda.values),
                                 conjugate ? 1 : 0, out.data().data()));
    return out;
}
inline Volume3D decimate(const Volume3D& x, const DecimationSpec& spec) {
    require_same_dims(x.dims(), spec.hr(), "decimate");
    Volume3D y(spec.lr());
    detail::check(vsr_decimate(detail::ctx(), detail::D3(spec.hr()).v, spec.rates_ptr(), x.data().data(),
                               y.data().data()));
    return y;
}
inline Volume3D decimate_adjoint(const Volume3D& y, const DecimationSpec& spec) {
    require_same_dims(y.dims(), spec.lr(), "decimate_adjoint");
    Volume3D x(spec.hr());
    detail::check(vsr_decimate_adjoint(detail::ctx(), detail::D3(spec.hr()).v, spec.rates_ptr(), y.data().data(),
                                       x.data().data()));
    return x;
}
inline Volume3D nn_upsample(const Volume3D& y, const DecimationSpec& spec) {
    require_same_dims(y.dims(), spec.lr(), "nn_upsample");
    Volume3D x(spec.hr());
    detail::check(vsr_nn_upsample(detail::ctx(), detail::D3(spec.hr()).v, spec.rates_ptr(), y.data().data(),
                                  x.data().data()));
    return x;
}
inline Volume3D zero_fill_upsample(const Volume3D& y, const DecimationSpec& spec) {
    Volume3D x = decimate_adjoint(y, spec);
    const double d = static_cast<double>(spec.rate());
    for (auto& v : x.data()) v *= d;
    return x;
}

enum class Axis { Rows = 0, Cols = 1, Slices = 2 };
inline Volume3D diff_forward(const Volume3D& x, Axis a) {
    Volume3D out(x.dims());
    detail::check(vsr_diff_forward(detail::ctx(), detail::D3(x.dims()).v, (int)a, x.data().data(), out.data().data()));
    return out;
}
inline Volume3D diff_adjoint(const Volume3D& x, Axis a) {
    Volume3D out(x.dims());
    detail::check(vsr_diff_adjoint(detail::ctx(), detail::D3(x.dims()).v, (int)a, x.data().data(), out.data().data()));
    return out;
}

// operators.hpp:79-87
struct DiffSpectra {
    SpectrumDiag rows, cols, slices;
    const SpectrumDiag& along(Axis a) const { return a == Axis::Rows ? rows : (a == Axis::Cols ? cols : slices); }
};
inline DiffSpectra finite_diff_spectra(const Dims3& hr) {
    DiffSpectra d{SpectrumDiag{ComplexVolume3D(hr)}, SpectrumDiag{ComplexVolume3D(hr)},
                  SpectrumDiag{ComplexVolume3D(hr)}};
    detail::check(vsr_finite_diff_spectra(detail::ctx(), detail::D3(hr).v, detail::cp(d.rows.values),
                                          detail::cp(d.cols.values), detail::cp(d.slices.values)));
    return d;
}

// ------------------------------------------------------------- spectral.hpp:12-19
inline ComplexVolume3D alias_fold(const ComplexVolume3D& hr, const DecimationSpec& spec) {
    require_same_dims(hr.dims(), spec.hr(), "alias_fold");
    ComplexVolume3D out(spec.lr());
    detail::check(vsr_alias_fold(detail::ctx(), detail::D3(spec.hr()).v, spec.rates_ptr(), detail::cp(hr),
                                 detail::cp(out)));
    return out;
}
inline ComplexVolume3D alias_expand(const ComplexVolume3D& lr, const DecimationSpec& spec) {
    require_same_dims(lr.dims(), spec.lr(), "alias_expand");
    ComplexVolume3D out(spec.hr());
    detail::check(vsr_alias_expand(detail::ctx(), detail::D3(spec.hr()).v, spec.rates_ptr(), detail::cp(lr),
                                   detail::cp(out)));
    return out;
}

// ------------------------------------------------------------- spectral.hpp:21-68
class FoldedSpectrum {
public:
    FoldedSpectrum(const SpectrumDiag& lambda, const DecimationSpec& spec) : spec_(spec) {
        require_same_dims(lambda.dims(), spec.hr(), "FoldedSpectrum");
        detail::check(vsr_folded_create(detail::ctx(), detail::D3(spec.hr()).v, spec.rates_ptr(),
                                        detail::cp(lambda.values), &h_));
    }
    // a value type, as in the reference: copies own an independent device copy of Lambda
    FoldedSpectrum(const FoldedSpectrum& o) : spec_(o.spec_) { detail::check(vsr_folded_clone(o.h_, &h_)); }
    FoldedSpectrum(FoldedSpectrum&& o) noexcept : spec_(o.spec_), h_(o.h_) { o.h_ = nullptr; }
    FoldedSpectrum& operator=(const FoldedSpectrum& o) {
        if (this != &o) {
            vsr_folded* h = nullptr;
            detail::check(vsr_folded_clone(o.h_, &h));
            vsr_folded_destroy(h_);
            h_ = h;
            spec_ = o.spec_;
        }
        return *this;
    }
    FoldedSpectrum& operator=(FoldedSpectrum&& o) noexcept {
        std::swap(h_, o.h_);
        spec_ = o.spec_;
        return *this;
    }
    ~FoldedSpectrum() {
        if (h_) vsr_folded_destroy(h_);
    }
    const DecimationSpec& spec() const { return spec_; }
    std::complex<double> block_value(std::size_t br, std::size_t bc, std::size_t bs, std::size_t g) const {
        double v[2];
        detail::check(vsr_folded_block_value(h_, br, bc, bs, g, v));
        return {v[0], v[1]};
    }
    ComplexVolume3D apply(const ComplexVolume3D& hr) const {
        require_same_dims(hr.dims(), spec_.hr(), "FoldedSpectrum::apply");
        ComplexVolume3D out(spec_.lr());
        detail::check(vsr_folded_apply(h_, detail::cp(hr), detail::cp(out)));
        return out;
    }
    ComplexVolume3D apply_adjoint(const ComplexVolume3D& lr) const {
        require_same_dims(lr.dims(), spec_.lr(), "FoldedSpectrum::apply_adjoint");
        ComplexVolume3D out(spec_.hr());
        detail::check(vsr_folded_apply_adjoint(h_, detail::cp(lr), detail::cp(out)));
        return out;
    }
    ComplexVolume3D apply_weighted(const ComplexVolume3D& hr, const Volume3D& w) const {
        require_same_dims(hr.dims(), spec_.hr(), "FoldedSpectrum::apply_weighted");
        require_same_dims(w.dims(), spec_.hr(), "FoldedSpectrum::apply_weighted: weights");
        ComplexVolume3D out(spec_.lr());
        detail::check(vsr_folded_apply_weighted(h_, detail::cp(hr), w.data().data(), detail::cp(out)));
        return out;
    }
    ComplexVolume3D apply_adjoint_weighted(const ComplexVolume3D& lr, const Volume3D& w) const {
        require_same_dims(lr.dims(), spec_.lr(), "FoldedSpectrum::apply_adjoint_weighted");
        require_same_dims(w.dims(), spec_.hr(), "FoldedSpectrum::apply_adjoint_weighted: weights");
        ComplexVolume3D out(spec_.hr());
        detail::check(vsr_folded_apply_adjoint_weighted(h_, detail::cp(lr), w.data().data(), detail::cp(out)));
        return out;
    }
    void swap_blocks_for_fault_injection() { detail::check(vsr_folded_swap_blocks_for_fault_injection(h_)); }
    vsr_folded* handle() const { return h_; }

private:
    DecimationSpec spec_;
    vsr_folded* h_ = nullptr;
};

inline FoldedSpectrum fold_lambda(const SpectrumDiag& lambda, const DecimationSpec& spec) {  // spectral.hpp:54
    return FoldedSpectrum(lambda, spec);
}

inline Volume3D gram_diag(const FoldedSpectrum& f) {
    Volume3D out(f.spec().lr());
    detail::check(vsr_folded_gram_diag(f.handle(), out.data().data()));
    return out;
}
inline Volume3D gram_diag_weighted(const FoldedSpectrum& f, const Volume3D& w) {
    require_same_dims(w.dims(), f.spec().hr(), "gram_diag_weighted");
    Volume3D out(f.spec().lr());
    detail::check(vsr_folded_gram_diag_weighted(f.handle(), w.data().data(), out.data().data()));
    return out;
}

// ------------------------------------------------------------- solvers.hpp:10-117
struct TikhonovConfig {
    double lambda = 0.01;
    Volume3D xbar;
};

struct SolveReport {
    std::size_t iterations = 0;
    double initial_objective = 0.0;
    std::vector<double> objective;
    std::vector<double> primal_residual;
    double seconds = 0.0;
};

class TikhonovOperator {
public:
    TikhonovOperator(const SpectrumDiag& lambda, const DecimationSpec& spec, const TikhonovConfig& cfg)
        : spec_(spec) {
        if (!(cfg.lambda > 0.0))
            throw std::invalid_argument("lambda must be positive, got " + std::to_string(cfg.lambda));
        require_same_dims(lambda.dims(), spec.hr(), "TikhonovOperator");
        require_same_dims(cfg.xbar.dims(), spec.hr(), "TikhonovOperator: xbar");
        detail::check(vsr_tikhonov_create(detail::ctx(), detail::D3(spec.hr()).v, spec.rates_ptr(),
                                          detail::cp(lambda.values), cfg.lambda, cfg.xbar.data().data(), &h_));
    }
    TikhonovOperator(const TikhonovOperator&) = delete;
    TikhonovOperator& operator=(const TikhonovOperator&) = delete;
    ~TikhonovOperator() { vsr_tikhonov_destroy(h_); }
    Volume3D solve(const Volume3D& y) const {
        require_same_dims(y.dims(), spec_.lr(), "TikhonovOperator::solve");
        Volume3D x(spec_.hr());
        detail::check(vsr_tikhonov_solve(h_, y.data().data(), x.data().data()));
        return x;
    }
    const DecimationSpec& spec() const { return spec_; }
    // B200 extension: the fp32 mode on the spatial path (fp32 y / x, lexicographic);
    // fp32_ok() tells whether this operator's path allows it
    bool fp32_ok() const { return vsr_tikhonov_fp32_ok(h_) != 0; }
    std::vector<float> solve_f32(const std::vector<float>& y) const {
        if (y.size() != spec_.lr().count()) throw shape_error("TikhonovOperator::solve_f32: dims mismatch");
        std::vector<float> x(spec_.hr().count());
        detail::check(vsr_tikhonov_solve_f32(h_, y.data(), x.data()));
        return x;
    }

private:
    DecimationSpec spec_;
    vsr_tikhonov* h_ = nullptr;
};

inline Volume3D tikhonov_fast(const Volume3D& y, const SpectrumDiag& lambda, const DecimationSpec& spec,
                              const TikhonovConfig& cfg) {
    return TikhonovOperator(lambda, spec, cfg).solve(y);
}

// solvers.hpp:54-70: iterative l2-l2 comparator (split v = Hx)
struct AdmmL2State {
    Volume3D x, v, dual;  // all HR dims
};

struct AdmmL2Options {
    double mu = 0.1;
    double rel_tol = 1e-10;
    std::optional<AdmmL2State> warm_start;
};

inline std::pair<Volume3D, SolveReport> admm_l2l2(const Volume3D& y, const SpectrumDiag& lambda,
                                                  const DecimationSpec& spec, const TikhonovConfig& cfg,
                                                  std::size_t max_iters, const AdmmL2Options& opts = {}) {
    if (!(cfg.lambda > 0.0)) throw std::invalid_argument("lambda must be positive, got " + std::to_string(cfg.lambda));
    if (!(opts.mu > 0.0)) throw std::invalid_argument("mu must be positive, got " + std::to_string(opts.mu));
    require_same_dims(y.dims(), spec.lr(), "admm_l2l2");
    require_same_dims(cfg.xbar.dims(), spec.hr(), "admm_l2l2: xbar");
    if (max_iters < 1) throw std::invalid_argument("admm_l2l2: max_iters must be >= 1");
    vsr_l2_config c{opts.mu, opts.rel_tol, nullptr, nullptr, nullptr};
    if (opts.warm_start) {
        require_same_dims(opts.warm_start->x.dims(), spec.hr(), "admm_l2l2: warm start");
        require_same_dims(opts.warm_start->v.dims(), spec.hr(), "admm_l2l2: warm start");
        require_same_dims(opts.warm_start->dual.dims(), spec.hr(), "admm_l2l2: warm start");
        c.warm_x = opts.warm_start->x.data().data();
        c.warm_v = opts.warm_start->v.data().data();
        c.warm_dual = opts.warm_start->dual.data().data();
    }
    SolveReport rep;
    rep.objective.resize(max_iters);
    rep.primal_residual.resize(max_iters);
    vsr_report vr{0, 0.0, 0.0, rep.objective.data(), rep.primal_residual.data()};
    Volume3D x(spec.hr());
    detail::check(vsr_admm_l2l2(detail::ctx(), detail::D3(spec.hr()).v, spec.rates_ptr(), y.data().data(),
                                detail::cp(lambda.values), cfg.lambda, cfg.xbar.data().data(), max_iters, &c,
                                x.data().data(), &vr));
    rep.iterations = vr.iterations;
    rep.initial_objective = vr.initial_objective;
    rep.seconds = vr.seconds;
    rep.objective.resize(vr.iterations);
    rep.primal_residual.resize(vr.iterations);
    return {std::move(x), std::move(rep)};
}

struct TvAdmmConfig {
    double lambda = 0.06;
    double mu = 0.1;
    std::size_t max_iters = 30;
    double rel_tol = 1e-6;
    std::optional<double> tau;
    enum class Init { Zero, UpsampledObservation, Provided };
    Init init = Init::Zero;
    Volume3D init_volume;
    // B200 extension (not in the reference): the optional fp32 mode
    // (include/vsr.h VSR_PRECISION_F32); the default keeps the reference precision
    enum class Precision { F64, F32 };
    Precision precision = Precision::F64;
};

// solvers.hpp:117 make_gamma(const DiffSpectra&, double)
inline Volume3D make_gamma(const DiffSpectra& diffs, double tau) {
    const Dims3& hr = diffs.rows.dims();
    require_same_dims(diffs.cols.dims(), hr, "make_gamma");
    require_same_dims(diffs.slices.dims(), hr, "make_gamma");
    Volume3D g(hr);
    detail::check(vsr_make_gamma_spectra(detail::ctx(), detail::D3(hr).v, detail::cp(diffs.rows.values),
                                         detail::cp(diffs.cols.values), detail::cp(diffs.slices.values), tau,
                                         g.data().data()));
    return g;
}

inline Volume3D tv_x_update(const Volume3D& y, const FoldedSpectrum&, const SpectrumDiag& lambda,
                            const DecimationSpec& spec, double mu, const ComplexVolume3D& theta_hat,
                            const Volume3D& gamma) {
    if (!(mu > 0.0)) throw std::invalid_argument("mu must be positive, got " + std::to_string(mu));
    require_same_dims(y.dims(), spec.lr(), "tv_x_update");
    require_same_dims(theta_hat.dims(), spec.hr(), "tv_x_update: theta_hat");
    require_same_dims(gamma.dims(), spec.hr(), "tv_x_update: gamma");
    Volume3D x(spec.hr());
    detail::check(vsr_tv_x_update(detail::ctx(), detail::D3(spec.hr()).v, spec.rates_ptr(), y.data().data(),
                                  detail::cp(lambda.values), mu, detail::cp(theta_hat), gamma.data().data(),
                                  x.data().data()));
    return x;
}

inline std::array<Volume3D, 3> tv_shrink(const Volume3D& a, const Volume3D& b, const Volume3D& c, double t) {
    require_same_dims(a.dims(), b.dims(), "tv_shrink");
    require_same_dims(a.dims(), c.dims(), "tv_shrink");
    std::array<Volume3D, 3> o{Volume3D(a.dims()), Volume3D(a.dims()), Volume3D(a.dims())};
    detail::check(vsr_tv_shrink(detail::ctx(), a.size(), a.data().data(), b.data().data(), c.data().data(), t,
                                o[0].data().data(), o[1].data().data(), o[2].data().data()));
    return o;
}

inline double objective_tv(const Volume3D& x, const Volume3D& y, const SpectrumDiag& lambda,
                           const DecimationSpec& spec, double w) {
    require_same_dims(x.dims(), spec.hr(), "objective_tv");
    require_same_dims(y.dims(), spec.lr(), "objective_tv");
    double out = 0.0;
    detail::check(vsr_objective_tv(detail::ctx(), detail::D3(spec.hr()).v, spec.rates_ptr(), x.data().data(),
                                   y.data().data(), detail::cp(lambda.values), w, &out));
    return out;
}

inline std::pair<Volume3D, SolveReport> admm_tv(const Volume3D& y, const Volume3D& psf, const DecimationSpec& spec,
                                                const TvAdmmConfig& cfg) {
    if (!(cfg.lambda > 0.0)) throw std::invalid_argument("lambda must be positive, got " + std::to_string(cfg.lambda));
    if (!(cfg.mu > 0.0)) throw std::invalid_argument("mu must be positive, got " + std::to_string(cfg.mu));
    if (cfg.max_iters < 1) throw std::invalid_argument("admm_tv: max_iters must be >= 1");
    require_same_dims(y.dims(), spec.lr(), "admm_tv");
    require_same_dims(psf.dims(), spec.hr(), "admm_tv: psf");
    if (cfg.init == TvAdmmConfig::Init::Provided)
        require_same_dims(cfg.init_volume.dims(), spec.hr(), "admm_tv: init volume");
    vsr_tv_config c{cfg.lambda, cfg.mu, cfg.max_iters, cfg.rel_tol, cfg.tau.has_value() ? 1 : 0,
                    cfg.tau.value_or(0.0), static_cast<int>(cfg.init),
                    cfg.init == TvAdmmConfig::Init::Provided ? cfg.init_volume.data().data() : nullptr,
                    cfg.precision == TvAdmmConfig::Precision::F32 ? VSR_PRECISION_F32 : VSR_PRECISION_F64};
    SolveReport rep;
    rep.objective.resize(cfg.max_iters);
    rep.primal_residual.resize(cfg.max_iters);
    vsr_report vr{0, 0.0, 0.0, rep.objective.data(), rep.primal_residual.data()};
    Volume3D x(spec.hr());
    detail::check(vsr_admm_tv(detail::ctx(), detail::D3(spec.hr()).v, spec.rates_ptr(), y.data().data(),
                              psf.data().data(), &c, x.data().data(), &vr));
    rep.iterations = vr.iterations;
    rep.initial_objective = vr.initial_objective;
    rep.seconds = vr.seconds;
    rep.objective.resize(vr.iterations);
    rep.primal_residual.resize(vr.iterations);
    return {std::move(x), std::move(rep)};
}

// ---------------------------------------------------------------- B200 extensions
// Slab-sharded solvers over P ranks (include/vsr.h vsr_comm_* / vsr_slab_*,
// SURVEY §8(e)): rank p owns the HR rows y in [p n/P, (p+1) n/P) of every
// plane; y and the PSF / Lambda are full volumes on every rank.  Slab results
// come back as one (m, n/P, s) Volume3D per LOCAL rank (P for a local comm,
// 1 for an NCCL comm).  Not part of the reference API.
namespace b200 {

class SlabComm {
public:
    // P virtual ranks in this process on the context's device
    static SlabComm local(int nranks) {
        vsr_comm* c = nullptr;
        detail::check(vsr_comm_local(detail::ctx(), nranks, &c));
        return SlabComm(c);
    }
    // one process per GPU over NCCL; rank 0's id (vsr_nccl_unique_id) on every rank
    static SlabComm nccl(int nranks, int rank, const unsigned char id[128]) {
        vsr_comm* c = nullptr;
        detail::check(vsr_comm_nccl(detail::ctx(), nranks, rank, id, &c));
        return SlabComm(c);
    }
    SlabComm(SlabComm&& o) noexcept : c_(o.c_) { o.c_ = nullptr; }
    SlabComm(const SlabComm&) = delete;
    SlabComm& operator=(const SlabComm&) = delete;
    ~SlabComm() {
        if (c_) vsr_comm_destroy(c_);
    }
    int nranks() const { int n = 0, r = 0, l = 0; vsr_comm_info(c_, &n, &r, &l); return n; }
    int local_ranks() const { int n = 0, r = 0, l = 0; vsr_comm_info(c_, &n, &r, &l); return l; }
    vsr_comm* handle() const { return c_; }

private:
    explicit SlabComm(vsr_comm* c) : c_(c) {}
    vsr_comm* c_ = nullptr;
};

inline Dims3 slab_dims(const DecimationSpec& spec, const SlabComm& comm) {
    const Dims3 hr = spec.hr();
    return Dims3{hr.m, hr.n / static_cast<std::size_t>(comm.nranks()), hr.s};
}

// admm_tv (solvers.hpp:106-107) over the ranks; cfg.init == Provided takes
// init_slabs (one per local rank) instead of cfg.init_volume
inline std::pair<std::vector<Volume3D>, SolveReport> admm_tv_sharded(
    const SlabComm& comm, const Volume3D& y, const Volume3D& psf, const DecimationSpec& spec,
    const TvAdmmConfig& cfg, const std::vector<Volume3D>& init_slabs = {}) {
    require_same_dims(y.dims(), spec.lr(), "admm_tv");
    require_same_dims(psf.dims(), spec.hr(), "admm_tv: psf");
    const int L = comm.local_ranks();
    std::vector<Volume3D> xs(L, Volume3D(slab_dims(spec, comm)));
    std::vector<double*> xp(L);
    for (int i = 0; i < L; ++i) xp[i] = xs[i].data().data();
    std::vector<const double*> ip;
    if (cfg.init == TvAdmmConfig::Init::Provided) {
        if ((int)init_slabs.size() != L) throw shape_error("admm_tv: init volume: one slab per local rank");
        for (const auto& v : init_slabs) ip.push_back(v.data().data());
    }
    vsr_tv_config c{cfg.lambda, cfg.mu, cfg.max_iters, cfg.rel_tol, cfg.tau.has_value() ? 1 : 0,
                    cfg.tau.value_or(0.0), static_cast<int>(cfg.init), nullptr, VSR_PRECISION_F64};
    SolveReport rep;
    rep.objective.resize(cfg.max_iters);
    rep.primal_residual.resize(cfg.max_iters);
    vsr_report vr{0, 0.0, 0.0, rep.objective.data(), rep.primal_residual.data()};
    detail::check(vsr_slab_admm_tv(comm.handle(), detail::D3(spec.hr()).v, spec.rates_ptr(), y.data().data(),
                                   psf.data().data(), &c, ip.empty() ? nullptr : ip.data(), xp.data(), &vr));
    rep.iterations = vr.iterations;
    rep.initial_objective = vr.initial_objective;
    rep.seconds = vr.seconds;
    rep.objective.resize(vr.iterations);
    rep.primal_residual.resize(vr.iterations);
    return {std::move(xs), std::move(rep)};
}

// TikhonovOperator (solvers.hpp:27-43) over the ranks; xbar as slabs
class SlabTikhonovOperator {
public:
    SlabTikhonovOperator(const SlabComm& comm, const SpectrumDiag& lambda, const DecimationSpec& spec,
                         double reg, const std::vector<Volume3D>& xbar_slabs)
        : spec_(spec), comm_(&comm) {
        require_same_dims(lambda.dims(), spec.hr(), "TikhonovOperator");
        if ((int)xbar_slabs.size() != comm.local_ranks())
            throw shape_error("TikhonovOperator: xbar: one slab per local rank");
        std::vector<const double*> xb;
        for (const auto& v : xbar_slabs) xb.push_back(v.data().data());
        detail::check(vsr_slab_tikhonov_create(comm.handle(), detail::D3(spec.hr()).v, spec.rates_ptr(),
                                               detail::cp(lambda.values), reg, xb.data(), &h_));
    }
    SlabTikhonovOperator(const SlabTikhonovOperator&) = delete;
    SlabTikhonovOperator& operator=(const SlabTikhonovOperator&) = delete;
    ~SlabTikhonovOperator() { vsr_slab_tikhonov_destroy(h_); }
    std::vector<Volume3D> solve(const Volume3D& y) const {
        require_same_dims(y.dims(), spec_.lr(), "TikhonovOperator::solve");
        const int L = comm_->local_ranks();
        std::vector<Volume3D> xs(L, Volume3D(slab_dims(spec_, *comm_)));
        std::vector<double*> xp(L);
        for (int i = 0; i < L; ++i) xp[i] = xs[i].data().data();
        detail::check(vsr_slab_tikhonov_solve(h_, y.data().data(), xp.data()));
        return xs;
    }

private:
    DecimationSpec spec_;
    const SlabComm* comm_;
    vsr_slab_tikhonov* h_ = nullptr;
};

}  // namespace b200
}  // namespace volsr
