// ExactThetaOp on the device (solver.cpp:21-29): Theta x = analyze(convolve(
// synthesize(x), psf)), Theta^T x with the conjugated kernel spectrum; and the generic
// estimate_step / run_pgd (solver.cpp:69-157) over it (the exact-fista comparator of the
// reference's bench protocol, waveblur.cpp:387-397).
//
// Arithmetic: the FFT convolution and the DWTs are the oracle build's exact operations
// (fft.cuh, wavelet.cu), so an application is bitwise the reference's. The elementwise steps
// follow the reference's expressions without contraction. The reductions (norm, dot, energy)
// use a fixed-order two-level tree instead of the reference's serial loops: deterministic,
// equal to the serial sums within rounding (rel ~1e-15).
#include <chrono>
#include <cmath>
#include <memory>

#include "fft.cuh"
#include "internal.hpp"

extern "C" void wbx_set_last_error(const char* msg);

struct wbx_exact_op {
    wbx_ctx* ctx = nullptr;
    wbx_basis* basis = nullptr;
    uint64_t n = 0;
    std::unique_ptr<wbx::Fft2> fft;
    wbx::DevBuf<double2> sk, su;
    wbx::DevBuf<double> img, u;
};

namespace wbx {
namespace {

constexpr int kRedBlocks = 296, kRedThreads = 256;

__device__ double ex_rng_normal(uint64_t seed, uint64_t i) {  // CounterRng::next_normal, i-th draw
    auto at = [](uint64_t s, uint64_t k) {
        uint64_t z = s + 0x9e3779b97f4a7c15ull * (k + 1);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    };
    auto u01 = [](uint64_t v) { return (static_cast<double>(v >> 11) + 0.5) * 0x1p-53; };
    const uint64_t m = i >> 1;
    const double u1 = u01(at(seed, 2 * m)), u2 = u01(at(seed, 2 * m + 1));
    const double r = sqrt(-2.0 * log(u1)), a = 2.0 * M_PI * u2;
    return (i & 1) ? r * sin(a) : r * cos(a);
}

// per-block partial of sum_i f(i) in a fixed order (grid-stride, then a fixed tree)
template <typename F>
__device__ void block_partial(uint64_t n, F f, double* out) {
    __shared__ double sm[kRedThreads];
    double s = 0.0;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kRedThreads + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * kRedThreads)
        s = __dadd_rn(s, f(i));
    sm[threadIdx.x] = s;
    __syncthreads();
    for (int w = kRedThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sm[threadIdx.x] = __dadd_rn(sm[threadIdx.x], sm[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = sm[0];
}

__global__ void dot_kernel(uint64_t n, const double* a, const double* b, double* part) {
    block_partial(n, [&](uint64_t i) { return __dmul_rn(a[i], b[i]); }, part);
}

// energy terms: sum (r - x0)^2 and sum w |x|
__global__ void energy_kernel(uint64_t n, const double* r, const double* x0, const double* w, const double* x,
                              double* part) {
    block_partial(n, [&](uint64_t i) { const double d = __dsub_rn(r[i], x0[i]); return __dmul_rn(d, d); }, part);
    block_partial(n, [&](uint64_t i) { return __dmul_rn(w[i], fabs(x[i])); }, part + kRedBlocks);
}

__global__ void support_kernel(uint64_t n, const double* x, unsigned long long* cnt) {
    unsigned long long c = 0;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        c += x[i] != 0.0;
    atomicAdd(cnt, c);
}

__global__ void final_sum_kernel(const double* part, int nparts, double* out) {  // in block order
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < nparts; ++i) s = __dadd_rn(s, part[i]);
        *out = s;
    }
}

__global__ void init_power_kernel(uint64_t n, const double* p, double* isp, double* v) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        isp[i] = __ddiv_rn(1.0, __dsqrt_rn(p[i]));
        v[i] = ex_rng_normal(0x5eedull, i);
    }
}

__global__ void scale_div_kernel(uint64_t n, double* v, double s) {  // v /= s
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        v[i] = __ddiv_rn(v[i], s);
}

__global__ void mul_kernel(uint64_t n, const double* a, const double* b, double* c) {  // c = a * b
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        c[i] = __dmul_rn(a[i], b[i]);
}

__global__ void sub_kernel(uint64_t n, double* r, const double* x0) {  // r -= x0
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        r[i] = __dsub_rn(r[i], x0[i]);
}

// z0 = y - tau * g / p; x_new = prox (solver.cpp:57-67, 126-128)
__global__ void prox_step_kernel(uint64_t n, const double* y, const double* g, const double* p, const double* w,
                                 double tau, double lambda, double* xn) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double z0 = __dsub_rn(y[i], __ddiv_rn(__dmul_rn(tau, g[i]), p[i]));
        const double thr = __ddiv_rn(__dmul_rn(__dmul_rn(tau, lambda), w[i]), p[i]);
        const double a = __dsub_rn(fabs(z0), thr);
        xn[i] = a > 0.0 ? (z0 > 0.0 ? a : -a) : 0.0;
    }
}

// y = x_new + beta * (x_new - x_prev); x_prev = x_new
__global__ void momentum_kernel(uint64_t n, const double* xn, double* xp, double* y, double beta) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        y[i] = __dadd_rn(xn[i], __dmul_rn(beta, __dsub_rn(xn[i], xp[i])));
        xp[i] = xn[i];
    }
}

constexpr unsigned kEwGrid = 1184, kEwThreads = 256;

void apply_dev(wbx_exact_op* e, int adjoint, const double* x, double* y) {
    cudaStream_t st = e->ctx->stream;
    synthesize_dev(e->basis, x, e->u.p, st);
    e->fft->r2c(e->u.p, e->su.p);
    e->fft->conv_c2r(e->su.p, e->sk.p, adjoint, e->img.p);
    analyze_dev(e->basis, e->img.p, y, st);
    count_launch(e->ctx, 12);
}

struct Reducer {  // fixed-order device reductions, read back synchronously
    DevBuf<double> part, out;
    Reducer() : part(2 * kRedBlocks), out(2) {}
    double dot(wbx_exact_op* e, const double* a, const double* b) {
        cudaStream_t st = e->ctx->stream;
        dot_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(e->n, a, b, part.p);
        final_sum_kernel<<<1, 32, 0, st>>>(part.p, kRedBlocks, out.p);
        double h = 0.0;
        WBX_CUDA(cudaMemcpyAsync(&h, out.p, sizeof h, cudaMemcpyDeviceToHost, st));
        WBX_CUDA(cudaStreamSynchronize(st));
        return h;
    }
    void energy2(wbx_exact_op* e, const double* r, const double* x0, const double* w, const double* x, double* quad,
                 double* reg) {
        cudaStream_t st = e->ctx->stream;
        energy_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(e->n, r, x0, w, x, part.p);
        final_sum_kernel<<<1, 32, 0, st>>>(part.p, kRedBlocks, out.p);
        final_sum_kernel<<<1, 32, 0, st>>>(part.p + kRedBlocks, kRedBlocks, out.p + 1);
        double h[2];
        WBX_CUDA(cudaMemcpyAsync(h, out.p, sizeof h, cudaMemcpyDeviceToHost, st));
        WBX_CUDA(cudaStreamSynchronize(st));
        *quad = h[0];
        *reg = h[1];
    }
};

// estimate_step (solver.cpp:69-99) over the exact operator; returns tau, sets iters
double estimate_step_exact(wbx_exact_op* e, const double* p_dev, double safety, uint32_t* iters) {
    const uint64_t n = e->n;
    cudaStream_t st = e->ctx->stream;
    DevBuf<double> isp(n), v(n), w(n), w2(n);
    Reducer red;
    init_power_kernel<<<kEwGrid, kEwThreads, 0, st>>>(n, p_dev, isp.p, v.p);
    const double nv = std::sqrt(red.dot(e, v.p, v.p));
    scale_div_kernel<<<kEwGrid, kEwThreads, 0, st>>>(n, v.p, nv);
    double lambda_prev = 0.0;
    uint32_t it = 0;
    for (; it < 200; ++it) {
        mul_kernel<<<kEwGrid, kEwThreads, 0, st>>>(n, isp.p, v.p, w.p);
        apply_dev(e, 0, w.p, w2.p);
        apply_dev(e, 1, w2.p, w.p);
        mul_kernel<<<kEwGrid, kEwThreads, 0, st>>>(n, w.p, isp.p, w.p);
        const double lambda = red.dot(e, v.p, w.p);
        const double nw = std::sqrt(red.dot(e, w.p, w.p));
        if (nw == 0.0) {
            *iters = it + 1;
            return 1.0;  // zero operator sentinel
        }
        std::swap(v, w);
        scale_div_kernel<<<kEwGrid, kEwThreads, 0, st>>>(n, v.p, nw);
        if (it > 0 && std::fabs(lambda - lambda_prev) <= 1e-6 * std::fabs(lambda)) {
            lambda_prev = lambda;
            ++it;
            break;
        }
        lambda_prev = lambda;
    }
    *iters = it;
    if (lambda_prev <= 0.0) return 1.0;
    return 1.0 / (lambda_prev * safety);
}

}  // namespace
}  // namespace wbx

extern "C" {

int wbx_exact_op_create(wbx_ctx* ctx, wbx_basis* basis, const double* psf, wbx_exact_op** out) {
    using namespace wbx;
    wbx_exact_op* e = nullptr;
    try {
        if (!ctx || !basis || !psf || !out) fail(WBX_INVALID_ARGUMENT, "null argument to wbx_exact_op_create");
        e = new wbx_exact_op;
        e->ctx = ctx;
        e->basis = basis;
        e->n = basis->n;
        const uint64_t n0 = basis->ndim == 2 ? basis->dims[0] : 1;
        const uint64_t n1 = basis->ndim == 2 ? basis->dims[1] : basis->dims[0];
        e->fft = std::make_unique<Fft2>(n0, n1, ctx->stream);
        const uint64_t hs = n0 * (n1 / 2 + 1);
        e->sk.alloc(hs);
        e->su.alloc(hs);
        e->img.alloc(e->n);
        e->u.alloc(e->n);
        e->img.upload(psf, e->n, ctx->stream);
        e->fft->r2c(e->img.p, e->sk.p);  // the kernel spectrum, as fft_forward(kernel) computes it
        WBX_CUDA(cudaStreamSynchronize(ctx->stream));
        *out = e;
        return WBX_OK;
    } catch (const wbx::Error& err) {
        delete e;
        wbx_set_last_error(err.what());
        return err.status;
    }
}

int wbx_exact_op_destroy(wbx_exact_op* e) {
    delete e;
    return WBX_OK;
}

int wbx_exact_apply_dev(wbx_exact_op* e, int adjoint, const double* x_dev, double* y_dev) {
    try {
        if (!e || !x_dev || !y_dev) wbx::fail(WBX_INVALID_ARGUMENT, "null argument to wbx_exact_apply_dev");
        wbx::apply_dev(e, adjoint, x_dev, y_dev);
        WBX_CUDA(cudaGetLastError());
        return WBX_OK;
    } catch (const wbx::Error& err) {
        wbx_set_last_error(err.what());
        return err.status;
    }
}

int wbx_exact_apply(wbx_exact_op* e, int adjoint, const double* x, double* y) {
    try {
        if (!e || !x || !y) wbx::fail(WBX_INVALID_ARGUMENT, "null argument to wbx_exact_apply");
        wbx::DevBuf<double> dx(e->n), dy(e->n);
        dx.upload(x, e->n, e->ctx->stream);
        wbx::apply_dev(e, adjoint, dx.p, dy.p);
        WBX_CUDA(cudaMemcpyAsync(y, dy.p, e->n * sizeof(double), cudaMemcpyDeviceToHost, e->ctx->stream));
        WBX_CUDA(cudaStreamSynchronize(e->ctx->stream));
        return WBX_OK;
    } catch (const wbx::Error& err) {
        wbx_set_last_error(err.what());
        return err.status;
    }
}

int wbx_estimate_step_exact(wbx_exact_op* e, const double* p, double step_safety, double* tau, uint32_t* iters) {
    try {
        if (!e || !p || !tau || !iters) wbx::fail(WBX_INVALID_ARGUMENT, "null argument to wbx_estimate_step_exact");
        for (uint64_t i = 0; i < e->n; ++i)
            if (!(p[i] > 0.0)) wbx::fail(WBX_BAD_SPEC, "preconditioner entries must be strictly positive");
        wbx::DevBuf<double> dp(e->n);
        dp.upload(p, e->n, e->ctx->stream);
        *tau = wbx::estimate_step_exact(e, dp.p, step_safety, iters);
        return WBX_OK;
    } catch (const wbx::Error& err) {
        wbx_set_last_error(err.what());
        return err.status;
    }
}

// run_pgd (solver.cpp:103-157) over the exact operator, fp64, reference expressions
int wbx_pgd_exact(wbx_exact_op* e, const double* x0, const double* w, double lambda, const double* p,
                  const wbx_solver_cfg* cfg, int accelerate, double* x_final, wbx_report* rep) {
    using namespace wbx;
    try {
        if (!e || !x0 || !w || !p || !cfg || !x_final || !rep)
            fail(WBX_INVALID_ARGUMENT, "null argument to wbx_pgd_exact");
        const uint64_t n = e->n;
        for (uint64_t i = 0; i < n; ++i)
            if (!(p[i] > 0.0)) fail(WBX_BAD_SPEC, "preconditioner entries must be strictly positive");
        cudaStream_t st = e->ctx->stream;
        const auto t0 = std::chrono::steady_clock::now();
        DevBuf<double> dx0(n), dw(n), dp(n), y(n), xp(n), xn(n), r(n), g(n);
        dx0.upload(x0, n, st);
        dw.upload(w, n, st);
        dp.upload(p, n, st);
        uint32_t tau_iters = 0;
        const double tau = cfg->tau > 0.0 ? cfg->tau : estimate_step_exact(e, dp.p, cfg->step_safety, &tau_iters);
        WBX_CUDA(cudaMemcpyAsync(y.p, dx0.p, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
        WBX_CUDA(cudaMemcpyAsync(xp.p, dx0.p, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
        Reducer red;
        const bool track = cfg->track_energy || std::isfinite(cfg->ref_energy);
        auto energy = [&](const double* x) {  // energy(x) (solver.cpp:44-55)
            apply_dev(e, 0, x, r.p);
            double quad = 0.0, reg = 0.0;
            red.energy2(e, r.p, dx0.p, dw.p, x, &quad, &reg);
            return 0.5 * quad + lambda * reg;
        };
        rep->initial_energy = track ? energy(dx0.p) : 0.0;
        const double stop_gap = cfg->rel_energy_tol * rep->initial_energy;
        DevBuf<unsigned long long> dcnt(1);
        uint64_t used = 0;
        for (uint64_t k = 1; k <= cfg->max_iters; ++k) {
            apply_dev(e, 0, y.p, r.p);
            sub_kernel<<<kEwGrid, kEwThreads, 0, st>>>(n, r.p, dx0.p);
            apply_dev(e, 1, r.p, g.p);
            prox_step_kernel<<<kEwGrid, kEwThreads, 0, st>>>(n, y.p, g.p, dp.p, dw.p, tau, lambda, xn.p);
            double en = 0.0;
            if (track) {
                en = energy(xn.p);
                if (!std::isfinite(en))
                    fail(WBX_NONFINITE_ENERGY, "solver diverged at iteration " + std::to_string(k));
                if (rep->energies) rep->energies[k - 1] = en;
            }
            if (cfg->track_support && rep->support_sizes) {
                WBX_CUDA(cudaMemsetAsync(dcnt.p, 0, sizeof(unsigned long long), st));
                support_kernel<<<kEwGrid, kEwThreads, 0, st>>>(n, xn.p, dcnt.p);
                unsigned long long c = 0;
                WBX_CUDA(cudaMemcpyAsync(&c, dcnt.p, sizeof c, cudaMemcpyDeviceToHost, st));
                WBX_CUDA(cudaStreamSynchronize(st));
                rep->support_sizes[k - 1] = c;
            }
            double beta = 0.0;
            if (accelerate && !cfg->zero_momentum)
                beta = (static_cast<double>(k) - 1.0) / (static_cast<double>(k) + 2.0);
            momentum_kernel<<<kEwGrid, kEwThreads, 0, st>>>(n, xn.p, xp.p, y.p, beta);
            used = k;
            if (std::isfinite(cfg->ref_energy) && en - cfg->ref_energy <= stop_gap) break;
        }
        WBX_CUDA(cudaMemcpyAsync(x_final, xp.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
        WBX_CUDA(cudaStreamSynchronize(st));
        rep->iters_used = used;
        rep->tau = tau;
        rep->tau_iters = tau_iters;
        rep->ops_per_pixel_per_iter = 0.0;
        rep->wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return WBX_OK;
    } catch (const wbx::Error& err) {
        wbx_set_last_error(err.what());
        return err.status;
    }
}

}  // extern "C"
