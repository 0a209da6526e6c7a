// CPU fp64 3D DFT backing the FFTW3-API shim (oracle/shim/fftw3.h) — TEST
// INFRASTRUCTURE for the reference build in oracle/_ref.  Row-column
// algorithm: out = in, then an in-place 1D transform along each axis.
// Powers of two use an iterative radix-2 decimation-in-time FFT with a
// twiddle table computed in long double; other lengths use a direct DFT with
// (j*k mod n) table indexing.  Optional threading over lines
// (VSR_SHIM_THREADS, default 1): each line is computed identically whatever
// the thread count, so results do not depend on it.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "fftw3.h"

namespace {

using cd = std::complex<double>;

struct Plan1D {
    int n = 1;
    int sign = -1;
    bool pow2 = true;
    std::vector<cd> tw;   // exp(sign 2 pi i k / n), k in [0, n)
    std::vector<int> rev; // bit reversal (pow2)
    void init(int len, int sgn) {
        n = len;
        sign = sgn;
        pow2 = (n & (n - 1)) == 0;
        tw.resize(n);
        for (int k = 0; k < n; ++k) {
            const long double ang = 2.0L * 3.141592653589793238462643383279502884L * (long double)k /
                                    (long double)n;
            tw[k] = cd((double)cosl(ang), (double)(sign * sinl(ang)));
        }
        if (pow2) {
            rev.resize(n);
            int bits = 0;
            while ((1 << bits) < n) ++bits;
            for (int i = 0; i < n; ++i) {
                int r = 0;
                for (int b = 0; b < bits; ++b)
                    if (i & (1 << b)) r |= 1 << (bits - 1 - b);
                rev[i] = r;
            }
        }
    }
    // in-place transform of a contiguous line; scratch has n entries
    void run(cd* a, cd* scratch) const {
        if (n == 1) return;
        if (pow2) {
            for (int i = 0; i < n; ++i)
                if (i < rev[i]) std::swap(a[i], a[rev[i]]);
            for (int len = 2; len <= n; len <<= 1) {
                const int half = len >> 1, step = n / len;
                for (int i = 0; i < n; i += len) {
                    for (int j = 0; j < half; ++j) {
                        const cd w = tw[j * step];
                        const cd u = a[i + j];
                        const cd v = a[i + j + half] * w;
                        a[i + j] = u + v;
                        a[i + j + half] = u - v;
                    }
                }
            }
        } else {
            for (int k = 0; k < n; ++k) {
                cd acc = 0.0;
                long long idx = 0;
                for (int j = 0; j < n; ++j) {
                    acc += a[j] * tw[idx];
                    idx += k;
                    if (idx >= n) idx -= n;
                }
                scratch[k] = acc;
            }
            std::copy(scratch, scratch + n, a);
        }
    }
};

int shim_threads() {
    const char* e = std::getenv("VSR_SHIM_THREADS");
    int t = e ? std::atoi(e) : 1;
    return std::max(1, t);
}

}  // namespace

struct vsr_fftw_plan_s {
    int n[3];  // n0 slowest, n2 fastest (contiguous)
    int sign;
    Plan1D p[3];
};

extern "C" {

fftw_plan fftw_plan_dft_3d(int n0, int n1, int n2, fftw_complex*, fftw_complex*, int sign, unsigned) {
    if (n0 <= 0 || n1 <= 0 || n2 <= 0) return nullptr;
    auto* pl = new vsr_fftw_plan_s();
    pl->n[0] = n0;
    pl->n[1] = n1;
    pl->n[2] = n2;
    pl->sign = sign;
    for (int a = 0; a < 3; ++a) pl->p[a].init(pl->n[a], sign);
    return pl;
}

void fftw_execute_dft(const fftw_plan pl, fftw_complex* in_, fftw_complex* out_) {
    const long long n0 = pl->n[0], n1 = pl->n[1], n2 = pl->n[2];
    const long long N = n0 * n1 * n2;
    cd* out = reinterpret_cast<cd*>(out_);
    const cd* in = reinterpret_cast<const cd*>(in_);
    if (out != in) std::memcpy(out, in, sizeof(cd) * N);
    const int T = shim_threads();
    // axis with length L, element stride S; lines enumerated by (outer, inner)
    auto do_axis = [&](int axis) {
        const long long L = pl->n[axis];
        if (L == 1) return;
        const long long S = axis == 2 ? 1 : (axis == 1 ? n2 : n1 * n2);
        const long long inner = S, outer = N / (L * S);
        constexpr long long B = 8;  // lines gathered together (cache-line reuse)
        const long long inner_blocks = (inner + B - 1) / B;
        const long long units = outer * inner_blocks;
        auto work = [&](long long u0, long long u1) {
            std::vector<cd> buf(B * L), scratch(L);
            for (long long u = u0; u < u1; ++u) {
                const long long o = u / inner_blocks, ib = u % inner_blocks;
                const long long p0 = ib * B, pb = std::min(B, inner - p0);
                const long long base = o * L * S + p0;
                for (long long q = 0; q < L; ++q)
                    for (long long b = 0; b < pb; ++b) buf[b * L + q] = out[base + q * S + b];
                for (long long b = 0; b < pb; ++b) pl->p[axis].run(&buf[b * L], scratch.data());
                for (long long q = 0; q < L; ++q)
                    for (long long b = 0; b < pb; ++b) out[base + q * S + b] = buf[b * L + q];
            }
        };
        if (T == 1 || units < 2 * T) {
            work(0, units);
        } else {
            std::vector<std::thread> th;
            for (int t = 0; t < T; ++t)
                th.emplace_back(work, units * t / T, units * (t + 1) / T);
            for (auto& x : th) x.join();
        }
    };
    do_axis(2);
    do_axis(1);
    do_axis(0);
}

void fftw_execute(const fftw_plan) {}

void fftw_destroy_plan(fftw_plan p) { delete p; }

}  // extern "C"
