// Complex fp64 FFT of power-of-two images in the oracle build's exact arithmetic (the
// radix-2 restatement of FFTW in oracle/shim/fftw_shim.cpp), and the FFT convolution of
// convolve_spectral (operators.cpp:20-77). Shared by the Theta_K construction
// (theta_gpu.cu) and the exact FFT operator (exact_op.cu).
#pragma once

#include <cmath>
#include <cstdint>
#include <vector>

#include "internal.hpp"

namespace wbx {
namespace {  // internal linkage: each including TU gets its own kernels
namespace fft_detail {

__device__ __forceinline__ double2 cmul(double2 b, double2 t) {  // (br + i bi)(tr + i ti)
    return make_double2(__dsub_rn(__dmul_rn(b.x, t.x), __dmul_rn(b.y, t.y)),
                        __dadd_rn(__dmul_rn(b.x, t.y), __dmul_rn(b.y, t.x)));
}

// One line of length n (power of two) per CTA: load in bit-reversed order, log2(n) stages.
__global__ void fft_lines_kernel(double2* data, uint32_t n, uint32_t logn, uint64_t elem_stride,
                                 uint64_t line_stride, int inverse, const double2* __restrict__ tw) {
    extern __shared__ double2 buf[];
    double2* a = data + static_cast<uint64_t>(blockIdx.x) * line_stride;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t r = __brev(i) >> (32 - logn);
        buf[r] = a[static_cast<uint64_t>(i) * elem_stride];
    }
    __syncthreads();
    for (uint32_t len = 2; len <= n; len <<= 1) {
        const uint32_t half = len >> 1, step = n / len;
        for (uint32_t j = threadIdx.x; j < n / 2; j += blockDim.x) {
            const uint32_t i = (j / half) * len, k = j % half;
            double2 t = tw[k * step];
            if (inverse) t.y = -t.y;
            const double2 u = buf[i + k];
            const double2 v = cmul(buf[i + k + half], t);
            buf[i + k] = make_double2(__dadd_rn(u.x, v.x), __dadd_rn(u.y, v.y));
            buf[i + k + half] = make_double2(__dsub_rn(u.x, v.x), __dsub_rn(u.y, v.y));
        }
        __syncthreads();
    }
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) a[static_cast<uint64_t>(i) * elem_stride] = buf[i];
}

__global__ void real_to_complex_kernel(const double* x, double2* a, uint64_t n) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) a[i] = make_double2(x[i], 0.0);
}

// half spectrum (c < h) of a full spectrum a[n0][n1]
__global__ void take_half_kernel(const double2* a, double2* spec, uint64_t n0, uint64_t n1, uint64_t h) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n0 * h) spec[i] = a[(i / h) * n1 + i % h];
}

// product of half spectra then the c2r rebuild of the full spectrum (fftw_shim execute)
__global__ void product_rebuild_kernel(const double2* su, const double2* sk, int conj_kernel, double2* a,
                                       uint64_t n0, uint64_t n1, uint64_t h) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n0 * n1) return;
    const uint64_t r = i / n1, c = i % n1;
    auto prod = [&](uint64_t q) {
        double2 k = sk[q];
        if (conj_kernel) k.y = -k.y;
        return cmul(su[q], k);
    };
    if (c < h) {
        a[i] = prod(r * h + c);
    } else {
        const double2 p = prod(((n0 - r) % n0) * h + (n1 - c));
        a[i] = make_double2(p.x, -p.y);
    }
}

__global__ void real_scale_kernel(const double2* a, double* x, uint64_t n, double scale) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) x[i] = __dmul_rn(a[i].x, scale);
}

inline unsigned grid_of(uint64_t n, unsigned t = 256) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace fft_detail

// Full-spectrum FFT helper bound to one image size.
struct Fft2 {
    uint64_t n0, n1, n, h;
    uint32_t log0 = 0, log1 = 0;
    DevBuf<double2> tw0, tw1, a;
    cudaStream_t st;
    Fft2(uint64_t d0, uint64_t d1, cudaStream_t s) : n0(d0), n1(d1), n(d0 * d1), h(d1 / 2 + 1), st(s) {
        auto is_pow2 = [](uint64_t x) { return x && !(x & (x - 1)); };
        if (!is_pow2(n0) || !is_pow2(n1)) fail(WBX_BAD_SPEC, "theta build: FFT sizes must be powers of two");
        if (n1 > 8192 || n0 > 8192) fail(WBX_TOO_LARGE, "theta build: FFT lines longer than 8192");
        while ((1ull << log0) < n0) ++log0;
        while ((1ull << log1) < n1) ++log1;
        auto table = [](uint64_t m) {  // fftw_shim twiddles(): evaluated directly on the host
            std::vector<double2> w(m / 2 + 1);
            for (uint64_t k = 0; k <= m / 2; ++k) {
                const double ang = -2.0 * M_PI * static_cast<double>(k) / static_cast<double>(m);
                w[k] = make_double2(std::cos(ang), std::sin(ang));
            }
            return w;
        };
        tw0.upload(table(n0), st);
        tw1.upload(table(n1), st);
        a.alloc(n);
    }
    static void smem_for(uint64_t m) {
        const int bytes = static_cast<int>(m * sizeof(double2));
        if (bytes > 48 * 1024)
            WBX_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fft_detail::fft_lines_kernel),
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    }
    void lines(int inverse) {  // rows then columns (fft_2d)
        smem_for(std::max(n0, n1));
        const unsigned t1 = static_cast<unsigned>(std::min<uint64_t>(512, std::max<uint64_t>(32, n1 / 2)));
        if (n1 > 1)
            fft_detail::fft_lines_kernel<<<static_cast<unsigned>(n0), t1, n1 * sizeof(double2), st>>>(a.p, static_cast<uint32_t>(n1), log1,
                                                                                         1, n1, inverse, tw1.p);
        if (n0 > 1) {
            const unsigned t0 = static_cast<unsigned>(std::min<uint64_t>(512, std::max<uint64_t>(32, n0 / 2)));
            fft_detail::fft_lines_kernel<<<static_cast<unsigned>(n1), t0, n0 * sizeof(double2), st>>>(a.p, static_cast<uint32_t>(n0), log0,
                                                                                         n1, 1, inverse, tw0.p);
        }
    }
    void r2c(const double* x, double2* spec) {
        fft_detail::real_to_complex_kernel<<<fft_detail::grid_of(n), 256, 0, st>>>(x, a.p, n);
        lines(0);
        fft_detail::take_half_kernel<<<fft_detail::grid_of(n0 * h), 256, 0, st>>>(a.p, spec, n0, n1, h);
    }
    void conv_c2r(const double2* su, const double2* sk, int conj_kernel, double* x) {
        fft_detail::product_rebuild_kernel<<<fft_detail::grid_of(n), 256, 0, st>>>(su, sk, conj_kernel, a.p, n0, n1, h);
        lines(1);
        fft_detail::real_scale_kernel<<<fft_detail::grid_of(n), 256, 0, st>>>(a.p, x, n, 1.0 / static_cast<double>(n));
    }
};

}  // namespace
}  // namespace wbx
