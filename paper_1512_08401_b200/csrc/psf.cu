// PSF generators, FFT convolution and degradation (operators.cpp:78-387).
//
// * generate_psf (operators.cpp:298-318): the kernels of GaussianSpec, SkewedGaussianSpec,
//   MotionSpec, AirySpec, DefocusSpec on the full grid, centred at index 0 with wrap-around,
//   unit mass. The analytic kernels are evaluated on the host with the reference's
//   expressions (libm exp / hypot / cyl_bessel_j, no contraction) — bitwise the reference's.
//   The motion kernel's control-point curve (CounterRng + natural cubic spline + bilinear
//   splat) is host work too; its Gaussian post-smoothing is an FFT convolution on the device.
// * convolve / apply_adjoint (operators.cpp:320-326 -> convolve_spectral :20-77): circular
//   convolution through the device FFT of fft.cuh, in the oracle build's exact operation
//   order (bitwise the oracle build; FFTW itself is not in this image).
// * degrade = add_noise(convolve(u, psf)) (operators.cpp:344-356, 385-387): the convolution
//   and the per-index Box-Muller noise on the device (CUDA's log/cos: within 2 ulp of glibc).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "fft.cuh"
#include "internal.hpp"

extern "C" void wbx_set_last_error(const char* msg);

namespace wbx {
namespace {

double wrapped_coord(uint64_t i, uint64_t n) {  // operators.cpp:78-82
    return i < n / 2 ? static_cast<double>(i) : static_cast<double>(i) - static_cast<double>(n);
}

void normalize_sum(double* k, uint64_t n) {  // operators.cpp:84-89
    double s = 0.0;
    for (uint64_t i = 0; i < n; ++i) s += k[i];
    if (s <= 0.0) fail(WBX_BAD_SPEC, "PSF has nonpositive mass");
    for (uint64_t i = 0; i < n; ++i) k[i] /= s;
}

bool is_pow2(uint64_t x) { return x && !(x & (x - 1)); }

// one kernel value per grid point from the wrapped coordinates (t1 = row, t2 = column; 1-D: t2 = 0)
template <typename F>
void fill(double* k, uint32_t ndim, const uint64_t* dims, F value) {
    if (ndim == 1) {
        for (uint64_t i = 0; i < dims[0]; ++i) k[i] = value(wrapped_coord(i, dims[0]), 0.0, true);
    } else {
        for (uint64_t r = 0; r < dims[0]; ++r)
            for (uint64_t c = 0; c < dims[1]; ++c)
                k[r * dims[1] + c] = value(wrapped_coord(r, dims[0]), wrapped_coord(c, dims[1]), false);
    }
}

void gaussian_kernel(double* k, uint32_t ndim, const uint64_t* dims, uint64_t n, double sigma) {  // :98-117
    if (sigma <= 0.0) fail(WBX_BAD_SPEC, "Gaussian sigma must be positive");
    if (sigma < 1.0) {  // sub-pixel width degenerates to a delta
        std::fill(k, k + n, 0.0);
        k[0] = 1.0;
        return;
    }
    fill(k, ndim, dims, [&](double t1, double t2, bool one_d) {
        return one_d ? std::exp(-t1 * t1 / (2.0 * sigma * sigma))
                     : std::exp(-(t1 * t1 + t2 * t2) / (2.0 * sigma * sigma));
    });
    normalize_sum(k, n);
}

void skewed_kernel(double* k, uint32_t ndim, const uint64_t* dims, uint64_t n, double sigma) {  // :119-135
    if (sigma <= 0.0) fail(WBX_BAD_SPEC, "SkewedGaussian sigma must be positive");
    fill(k, ndim, dims, [&](double t1, double t2, bool) {
        const double a = t1 >= 0.0 ? 1.0 : 4.0;  // four-fold sharper decay on the negative side
        return std::exp(-(a * t1 * t1 + t2 * t2) / (2.0 * sigma * sigma));
    });
    normalize_sum(k, n);
}

void airy_kernel(double* k, uint32_t ndim, const uint64_t* dims, uint64_t n, double scale) {  // :236-255
    if (scale <= 0.0) fail(WBX_BAD_SPEC, "Airy scale must be positive");
    auto value = [&](double r) {
        const double x = M_PI * r / scale;
        if (x < 1e-12) return 1.0;
        const double j1 = std::cyl_bessel_j(1.0, x);
        const double a = 2.0 * j1 / x;
        return a * a;
    };
    fill(k, ndim, dims, [&](double t1, double t2, bool one_d) { return value(one_d ? std::abs(t1) : std::hypot(t1, t2)); });
    normalize_sum(k, n);
}

void defocus_kernel(double* k, uint32_t ndim, const uint64_t* dims, uint64_t n, double radius) {  // :257-274
    if (radius <= 0.0) fail(WBX_BAD_SPEC, "defocus radius must be positive");
    fill(k, ndim, dims, [&](double t1, double t2, bool one_d) {
        return (one_d ? std::abs(t1) : std::hypot(t1, t2)) <= radius ? 1.0 : 0.0;
    });
    normalize_sum(k, n);
}

// CounterRng (rng.hpp:11-51): sequential next_normal with the cached Box-Muller spare
struct HostRng {
    uint64_t seed, counter = 0;
    double spare = 0.0;
    bool have_spare = false;
    uint64_t at(uint64_t i) const {
        uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (i + 1);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    double uniform() { return (static_cast<double>(at(counter++) >> 11) + 0.5) * 0x1p-53; }
    double normal() {
        if (have_spare) {
            have_spare = false;
            return spare;
        }
        const double u1 = uniform();
        const double u2 = uniform();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 2.0 * M_PI * u2;
        spare = r * std::sin(a);
        have_spare = true;
        return r * std::cos(a);
    }
};

// natural cubic spline through (i, y_i) (operators.cpp:137-176)
struct Spline {
    std::vector<double> y, m2;
    explicit Spline(std::vector<double> pts) : y(std::move(pts)) {
        const size_t n = y.size();
        m2.assign(n, 0.0);
        if (n < 3) return;
        std::vector<double> a(n, 0.0), b(n, 0.0), c(n, 0.0), d(n, 0.0);
        for (size_t i = 1; i + 1 < n; ++i) {
            a[i] = 1.0;
            b[i] = 4.0;
            c[i] = 1.0;
            d[i] = 6.0 * (y[i + 1] - 2.0 * y[i] + y[i - 1]);
        }
        for (size_t i = 2; i + 1 < n; ++i) {  // forward elimination (Thomas)
            const double w = a[i] / b[i - 1];
            b[i] -= w * c[i - 1];
            d[i] -= w * d[i - 1];
        }
        for (size_t i = n - 2; i >= 1; --i) {  // back substitution, m2[0] = m2[n-1] = 0
            const double upper = (i + 2 < n) ? c[i] * m2[i + 1] : 0.0;
            m2[i] = (d[i] - upper) / b[i];
            if (i == 1) break;
        }
    }
    double operator()(double t) const {
        const size_t n = y.size();
        if (n == 1) return y[0];
        const double tc = std::clamp(t, 0.0, static_cast<double>(n - 1));
        const size_t i = std::min(static_cast<size_t>(tc), n - 2);
        const double h = tc - static_cast<double>(i);
        const double hm = 1.0 - h;
        return hm * y[i] + h * y[i + 1] + (hm * (hm * hm - 1.0) * m2[i] + h * (h * h - 1.0) * m2[i + 1]) / 6.0;
    }
};

// circular convolution / its adjoint on the device (convolve_spectral, operators.cpp:70-77)
void convolve_dev(wbx_ctx* ctx, uint32_t ndim, const uint64_t* dims, const double* kernel_dev, const double* u_dev,
                  int adjoint, double* out_dev) {
    const uint64_t n0 = ndim == 2 ? dims[0] : 1, n1 = ndim == 2 ? dims[1] : dims[0];
    Fft2 fft(n0, n1, ctx->stream);
    DevBuf<double2> sk(n0 * (n1 / 2 + 1)), su(n0 * (n1 / 2 + 1));
    fft.r2c(kernel_dev, sk.p);
    fft.r2c(u_dev, su.p);
    fft.conv_c2r(su.p, sk.p, adjoint, out_dev);
    count_launch(ctx, 9);
    WBX_CUDA(cudaGetLastError());
}

void motion_kernel(wbx_ctx* ctx, double* k, uint32_t ndim, const uint64_t* dims, uint64_t n, unsigned points,
                   double sigma1, double sigma2, uint64_t seed) {  // operators.cpp:177-234
    if (points < 2) fail(WBX_BAD_SPEC, "motion blur needs at least 2 points");
    if (sigma1 <= 0.0 || sigma2 <= 0.0) fail(WBX_BAD_SPEC, "motion blur sigmas must be positive");
    if (!ctx) fail(WBX_INVALID_ARGUMENT, "motion kernel: a context is needed (device FFT smoothing)");
    HostRng rng{seed};
    const unsigned l = points;
    std::vector<double> px(l), py(l);
    for (unsigned i = 0; i < l; ++i) px[i] = sigma1 * rng.normal();
    if (ndim == 2)
        for (unsigned i = 0; i < l; ++i) py[i] = sigma1 * rng.normal();
    const Spline sx(px), sy(py);
    // polyline length estimate -> sampling density (10 samples per pixel of length)
    double length = 0.0;
    const int probe = 64 * static_cast<int>(l);
    double prevx = sx(0.0), prevy = ndim == 2 ? sy(0.0) : 0.0;
    for (int i = 1; i <= probe; ++i) {
        const double t = static_cast<double>(i) / probe * (l - 1);
        const double cx = sx(t), cy = ndim == 2 ? sy(t) : 0.0;
        length += std::hypot(cx - prevx, cy - prevy);
        prevx = cx;
        prevy = cy;
    }
    const size_t samples = std::max<size_t>(2, static_cast<size_t>(10.0 * length) + 1);
    std::vector<double> curve(n, 0.0);
    auto wrap = [](double x, uint64_t m) {
        const double r = std::fmod(x, static_cast<double>(m));
        return r < 0.0 ? r + static_cast<double>(m) : r;
    };
    for (size_t s = 0; s < samples; ++s) {
        const double t = static_cast<double>(s) / static_cast<double>(samples - 1) * (l - 1);
        if (ndim == 1) {
            const double x = wrap(sx(t), dims[0]);
            const size_t i0 = static_cast<size_t>(x) % dims[0];
            const double f = x - std::floor(x);
            curve[i0] += 1.0 - f;
            curve[(i0 + 1) % dims[0]] += f;
        } else {
            const double x = wrap(sx(t), dims[0]);
            const double y = wrap(sy(t), dims[1]);
            const size_t r0 = static_cast<size_t>(x) % dims[0];
            const size_t c0 = static_cast<size_t>(y) % dims[1];
            const double fr = x - std::floor(x), fc = y - std::floor(y);
            const uint64_t W = dims[1];
            curve[r0 * W + c0] += (1.0 - fr) * (1.0 - fc);
            curve[((r0 + 1) % dims[0]) * W + c0] += fr * (1.0 - fc);
            curve[r0 * W + (c0 + 1) % dims[1]] += (1.0 - fr) * fc;
            curve[((r0 + 1) % dims[0]) * W + (c0 + 1) % dims[1]] += fr * fc;
        }
    }
    normalize_sum(curve.data(), n);
    std::vector<double> smooth(n);
    gaussian_kernel(smooth.data(), ndim, dims, n, sigma2);
    DevBuf<double> dc(n), dg(n), dk(n);
    dc.upload(curve.data(), n, ctx->stream);
    dg.upload(smooth.data(), n, ctx->stream);
    convolve_dev(ctx, ndim, dims, dg.p, dc.p, 0, dk.p);
    WBX_CUDA(cudaMemcpyAsync(k, dk.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    WBX_CUDA(cudaStreamSynchronize(ctx->stream));
    for (uint64_t i = 0; i < n; ++i) k[i] = std::max(k[i], 0.0);  // FFT roundoff can go slightly negative
    normalize_sum(k, n);
}

uint64_t check_dims(uint32_t ndim, const uint64_t* dims) {  // Image::require_dyadic (image.hpp:73-78)
    if (!dims || ndim < 1 || ndim > 2) fail(WBX_SHAPE_MISMATCH, "image must be 1D or 2D");
    uint64_t n = 1;
    for (uint32_t d = 0; d < ndim; ++d) {
        if (!is_pow2(dims[d])) fail(WBX_SHAPE_MISMATCH, "side lengths must be powers of 2");
        n *= dims[d];
    }
    return n;
}

__global__ void add_noise_kernel(uint64_t n, const double* in, double sigma, uint64_t seed, double* out) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        auto at = [&](uint64_t k) {
            uint64_t z = seed + 0x9e3779b97f4a7c15ull * (k + 1);
            z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
            z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
            return z ^ (z >> 31);
        };
        const double u1 = (static_cast<double>(at(2 * i) >> 11) + 0.5) * 0x1p-53;
        const double u2 = (static_cast<double>(at(2 * i + 1) >> 11) + 0.5) * 0x1p-53;
        // operators.cpp:353: out[i] += sigma * sqrt(-2 log u1) * cos(2 pi u2), no contraction
        const double b = __dmul_rn(__dmul_rn(sigma, __dsqrt_rn(__dmul_rn(-2.0, log(u1)))), cos(__dmul_rn(2.0 * M_PI, u2)));
        out[i] = __dadd_rn(in[i], b);
    }
}

}  // namespace
}  // namespace wbx

extern "C" {

int wbx_generate_psf(wbx_ctx* ctx, uint32_t kind, const double* params, uint32_t ndim, const uint64_t* dims,
                     double* kernel) {
    using namespace wbx;
    try {
        if (!params || !kernel) fail(WBX_INVALID_ARGUMENT, "null argument to wbx_generate_psf");
        const uint64_t n = check_dims(ndim, dims);
        switch (kind) {
            case WBX_PSF_GAUSSIAN: gaussian_kernel(kernel, ndim, dims, n, params[0]); break;
            case WBX_PSF_SKEWED: skewed_kernel(kernel, ndim, dims, n, params[0]); break;
            case WBX_PSF_MOTION: {
                if (!(params[0] >= 0.0) || params[0] > 4294967295.0 || params[3] < 0.0)
                    fail(WBX_BAD_SPEC, "motion blur: bad point count or seed");
                motion_kernel(ctx, kernel, ndim, dims, n, static_cast<unsigned>(params[0]), params[1], params[2],
                              static_cast<uint64_t>(params[3]));
                break;
            }
            case WBX_PSF_AIRY: airy_kernel(kernel, ndim, dims, n, params[0]); break;
            case WBX_PSF_DEFOCUS: defocus_kernel(kernel, ndim, dims, n, params[0]); break;
            default: fail(WBX_BAD_SPEC, "unknown PSF kind");
        }
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

int wbx_convolve(wbx_ctx* ctx, uint32_t ndim, const uint64_t* dims, const double* kernel, const double* u, int adjoint,
                 double* out) {
    using namespace wbx;
    try {
        if (!ctx || !kernel || !u || !out) fail(WBX_INVALID_ARGUMENT, "null argument to wbx_convolve");
        const uint64_t n = check_dims(ndim, dims);
        DevBuf<double> dk(n), du(n), dy(n);
        dk.upload(kernel, n, ctx->stream);
        du.upload(u, n, ctx->stream);
        convolve_dev(ctx, ndim, dims, dk.p, du.p, adjoint ? 1 : 0, dy.p);
        WBX_CUDA(cudaMemcpyAsync(out, dy.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        WBX_CUDA(cudaStreamSynchronize(ctx->stream));
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

int wbx_add_noise(wbx_ctx* ctx, uint64_t n, const double* u, double sigma, uint64_t seed, double* out) {
    using namespace wbx;
    try {
        if (!ctx || !u || !out) fail(WBX_INVALID_ARGUMENT, "null argument to wbx_add_noise");
        if (sigma < 0.0) fail(WBX_BAD_SPEC, "noise sigma must be >= 0");
        if (sigma == 0.0) {
            if (out != u) std::memcpy(out, u, n * sizeof(double));
            return WBX_OK;
        }
        DevBuf<double> du(n);
        du.upload(u, n, ctx->stream);
        add_noise_kernel<<<static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 4096)), 256, 0, ctx->stream>>>(
            n, du.p, sigma, seed, du.p);
        count_launch(ctx);
        WBX_CUDA(cudaGetLastError());
        WBX_CUDA(cudaMemcpyAsync(out, du.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        WBX_CUDA(cudaStreamSynchronize(ctx->stream));
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

int wbx_degrade(wbx_ctx* ctx, uint32_t ndim, const uint64_t* dims, const double* kernel, const double* u,
                double noise_sigma, uint64_t seed, double* out) {
    using namespace wbx;
    try {
        if (!ctx || !kernel || !u || !out) fail(WBX_INVALID_ARGUMENT, "null argument to wbx_degrade");
        const uint64_t n = check_dims(ndim, dims);
        if (noise_sigma < 0.0) fail(WBX_BAD_SPEC, "noise sigma must be >= 0");
        DevBuf<double> dk(n), du(n), dy(n);
        dk.upload(kernel, n, ctx->stream);
        du.upload(u, n, ctx->stream);
        convolve_dev(ctx, ndim, dims, dk.p, du.p, 0, dy.p);
        if (noise_sigma > 0.0) {
            add_noise_kernel<<<static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 4096)), 256, 0,
                               ctx->stream>>>(n, dy.p, noise_sigma, seed, dy.p);
            count_launch(ctx);
        }
        WBX_CUDA(cudaGetLastError());
        WBX_CUDA(cudaMemcpyAsync(out, dy.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        WBX_CUDA(cudaStreamSynchronize(ctx->stream));
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    }
}

}  // extern "C"
