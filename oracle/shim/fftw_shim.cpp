// oracle/shim/fftw_shim.cpp — TEST INFRASTRUCTURE ONLY. Radix-2 restatement of
// the FFTW3 r2c/c2r API subset the reference calls (see fftw3.h for the contract).
#include "fftw3.h"

#include <cmath>
#include <complex>
#include <cstdlib>
#include <map>
#include <mutex>
#include <stdexcept>
#include <vector>

namespace {

using cplx = std::complex<double>;

// Twiddle table per size, evaluated directly (no recurrence) for accuracy.
const std::vector<cplx>& twiddles(std::size_t n) {
    static std::mutex mu;
    static std::map<std::size_t, std::vector<cplx>> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(n);
    if (it != cache.end()) return it->second;
    std::vector<cplx> w(n / 2 + 1);
    for (std::size_t k = 0; k <= n / 2; ++k) {
        const double a = -2.0 * M_PI * static_cast<double>(k) / static_cast<double>(n);
        w[k] = cplx(std::cos(a), std::sin(a));
    }
    return cache.emplace(n, std::move(w)).first->second;
}

// In-place FFT of a strided line; sign = -1 forward, +1 backward (unnormalised).
void fft_line(cplx* a, std::size_t n, std::size_t stride, int sign, std::vector<cplx>& buf) {
    if (n == 1) return;
    if ((n & (n - 1)) != 0) throw std::invalid_argument("fftw shim: size must be a power of 2");
    buf.resize(n);
    for (std::size_t i = 0; i < n; ++i) buf[i] = a[i * stride];
    // bit reversal
    for (std::size_t i = 1, j = 0; i < n; ++i) {
        std::size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(buf[i], buf[j]);
    }
    const auto& w = twiddles(n);
    for (std::size_t len = 2; len <= n; len <<= 1) {
        const std::size_t step = n / len;
        for (std::size_t i = 0; i < n; i += len) {
            for (std::size_t k = 0; k < len / 2; ++k) {
                cplx t = w[k * step];
                if (sign > 0) t = std::conj(t);
                const cplx u = buf[i + k];
                const cplx v = buf[i + k + len / 2] * t;
                buf[i + k] = u + v;
                buf[i + k + len / 2] = u - v;
            }
        }
    }
    for (std::size_t i = 0; i < n; ++i) a[i * stride] = buf[i];
}

// Full complex 2-D (or 1-D when n0 == 1) transform in place.
void fft_2d(std::vector<cplx>& a, std::size_t n0, std::size_t n1, int sign) {
    std::vector<cplx> buf;
    for (std::size_t r = 0; r < n0; ++r) fft_line(a.data() + r * n1, n1, 1, sign, buf);
    if (n0 > 1)
        for (std::size_t c = 0; c < n1; ++c) fft_line(a.data() + c, n0, n1, sign, buf);
}

}  // namespace

struct wbx_fftw_plan_s {
    bool r2c;
    std::size_t n0, n1;  // n0 == 1 for 1-D
    double* real;
    cplx* spec;
};

extern "C" {

fftw_plan fftw_plan_dft_r2c_1d(int n, double* in, fftw_complex* out, unsigned) {
    return new wbx_fftw_plan_s{true, 1, static_cast<std::size_t>(n), in,
                               reinterpret_cast<cplx*>(out)};
}

fftw_plan fftw_plan_dft_r2c_2d(int n0, int n1, double* in, fftw_complex* out, unsigned) {
    return new wbx_fftw_plan_s{true, static_cast<std::size_t>(n0), static_cast<std::size_t>(n1),
                               in, reinterpret_cast<cplx*>(out)};
}

fftw_plan fftw_plan_dft_c2r_1d(int n, fftw_complex* in, double* out, unsigned) {
    return new wbx_fftw_plan_s{false, 1, static_cast<std::size_t>(n), out,
                               reinterpret_cast<cplx*>(in)};
}

fftw_plan fftw_plan_dft_c2r_2d(int n0, int n1, fftw_complex* in, double* out, unsigned) {
    return new wbx_fftw_plan_s{false, static_cast<std::size_t>(n0), static_cast<std::size_t>(n1),
                               out, reinterpret_cast<cplx*>(in)};
}

void fftw_execute(const fftw_plan p) {
    const std::size_t n0 = p->n0, n1 = p->n1, h = n1 / 2 + 1;
    std::vector<cplx> a(n0 * n1);
    if (p->r2c) {
        for (std::size_t i = 0; i < n0 * n1; ++i) a[i] = cplx(p->real[i], 0.0);
        fft_2d(a, n0, n1, -1);
        for (std::size_t r = 0; r < n0; ++r)
            for (std::size_t c = 0; c < h; ++c) p->spec[r * h + c] = a[r * n1 + c];
    } else {
        // rebuild the full Hermitian spectrum from the half spectrum
        for (std::size_t r = 0; r < n0; ++r) {
            for (std::size_t c = 0; c < n1; ++c) {
                if (c < h) {
                    a[r * n1 + c] = p->spec[r * h + c];
                } else {
                    const std::size_t rr = (n0 - r) % n0, cc = n1 - c;
                    a[r * n1 + c] = std::conj(p->spec[rr * h + cc]);
                }
            }
        }
        fft_2d(a, n0, n1, +1);
        for (std::size_t i = 0; i < n0 * n1; ++i) p->real[i] = a[i].real();
    }
}

void fftw_destroy_plan(fftw_plan p) { delete p; }

}  // extern "C"
