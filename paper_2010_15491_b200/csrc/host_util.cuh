// Host-side helpers shared by the C-ABI translation units (capi.cu, slab.cu):
// an owning device buffer, the DecimationSpec validation (reference
// src/operators.cpp:8-21) and the argument checks of src/solvers.cpp.
#pragma once

#include <cmath>
#include <string>
#include <vector>

#include "vsr_common.cuh"

namespace vsr_host {
using vsr::Dims;
using vsr::numeric_error;
using vsr::shape_error;

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) VSR_CUDA(cudaMalloc(&p, count * sizeof(T)));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~DevBuf() { release(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        release();
        p = o.p;
        n = o.n;
        o.p = nullptr;
        o.n = 0;
        return *this;
    }
    size_t bytes() const { return n * sizeof(T); }
};

inline Dims to_dims(const size_t d[3]) {
    if (!d) throw std::invalid_argument("dims pointer is null");
    Dims r;
    r.m = d[0];
    r.n = d[1];
    r.s = d[2];
    return r;
}

// DecimationSpec ctor (src/operators.cpp:8-21).
struct Spec {
    Dims hr, lr;
    int rates[3];
    size_t rate() const { return (size_t)rates[0] * rates[1] * rates[2]; }
};

inline Spec make_spec(const size_t hr_dims[3], const size_t rates[3]) {
    if (!rates) throw std::invalid_argument("rates pointer is null");
    const Dims hr = to_dims(hr_dims);
    static const char* names[3] = {"1 (rows)", "2 (cols)", "3 (slices)"};
    const size_t ext[3] = {hr.m, hr.n, hr.s};
    for (int a = 0; a < 3; ++a) {
        if (rates[a] == 0) throw shape_error(std::string("DecimationSpec: zero rate on axis ") + names[a]);
        if (ext[a] % rates[a] != 0)
            throw shape_error("DecimationSpec: rate " + std::to_string(rates[a]) +
                              " does not divide axis " + names[a] + " of length " +
                              std::to_string(ext[a]));
    }
    Spec s;
    s.hr = hr;
    s.lr = Dims{hr.m / rates[0], hr.n / rates[1], hr.s / rates[2]};
    for (int a = 0; a < 3; ++a) s.rates[a] = (int)rates[a];
    return s;
}

inline void require_nonempty(const Dims& d, const char* where) {
    if (d.count() == 0) throw shape_error(std::string(where) + ": empty volume");
}

inline void require_positive(double v, const char* name) {  // src/solvers.cpp:18-22
    if (!(v > 0.0))
        throw std::invalid_argument(std::string(name) + " must be positive, got " + std::to_string(v));
}

inline std::vector<double> diff_norm_table(size_t len) {
    // std::norm({cos(2 pi f/len) - 1, sin(2 pi f/len)}) with exact 0 at DC
    // (src/operators.cpp:233-240); same libm as the reference build.
    std::vector<double> t(len);
    const double two_pi = 2.0 * 3.14159265358979323846;
    for (size_t f = 0; f < len; ++f) {
        if (f == 0) {
            t[f] = 0.0;
            continue;
        }
        const double ang = two_pi * (double)f / (double)len;
        const double re = std::cos(ang) - 1.0, im = std::sin(ang);
        t[f] = re * re + im * im;
    }
    return t;
}

// make_gamma validity (src/solvers.cpp:192-201): tau >= 0, every
// denominator > 0; the smallest denominator is the DC bin, equal to tau.
inline void validate_tau(double tau) {
    if (tau < 0.0) throw std::invalid_argument("make_gamma: tau must be nonnegative");
    if (!(tau > 0.0))
        throw numeric_error(
            "make_gamma: difference-operator gram is singular at the zero frequency (DC); "
            "a positive tau floor is required");
}

}  // namespace vsr_host
