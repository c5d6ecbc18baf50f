// extern "C" entry points of libwbx.so (declared in include/wbx.h).
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "internal.hpp"
#include "wbx_diag.h"

struct wbx_solver;

namespace wbx {
void solver_setup(wbx_solver* s, const double* p, const double* w);
wbx_solver* pgd_acquire(wbx_ctx* ctx, const wbx_op* op, const wbx_solver_cfg& cfg, int accelerate, double lambda,
                        const double* p, const double* w);
void pgd_release(wbx_solver* s);
void pgd_purge(const wbx_ctx* ctx, const wbx_op* op);
double* solver_x0_buf(wbx_solver* s);
double* solver_x_buf(wbx_solver* s);
void solver_run(wbx_solver* s, const double* x0_full_dev, double* x_full_dev);
void solver_report(wbx_solver* s, wbx_report* rep);
void launch_clamp(wbx_ctx* ctx, double* u, uint64_t n, cudaStream_t st);
wbx_solver* solver_new(wbx_ctx* ctx, const wbx_op* op, wbx_basis* basis, double lambda,
                       const wbx_solver_cfg& cfg, int accelerate);
void solver_free(wbx_solver* s);
double* solver_buf(wbx_solver* s, int which);  // 0 u0, 1 x0full, 2 xfull, 3 uout
void solver_alloc_images(wbx_solver* s);
}  // namespace wbx

namespace {

thread_local std::string g_last_error;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return WBX_OK;
    } catch (const wbx::Error& e) {
        g_last_error = e.what();
        return e.status;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return WBX_MEMORY_GUARD;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return WBX_CUDA_ERROR;
    }
}

void need(const void* p, const char* what) {
    if (p == nullptr) wbx::fail(WBX_INVALID_ARGUMENT, std::string("null argument: ") + what);
}

// ---------------------------------------------------------------- elementwise kernels
// prox_weighted_l1_P (solver.cpp:57-67), exact fp64 expression order
__global__ void prox_kernel(uint64_t n, const double* z0, double tau, const double* w, double lambda,
                            const double* p, double* z) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double thr = __ddiv_rn(__dmul_rn(__dmul_rn(tau, lambda), w[i]), p[i]);
    const double a = __dsub_rn(fabs(z0[i]), thr);
    z[i] = a > 0.0 ? (z0[i] > 0.0 ? a : -a) : 0.0;
}

// per-block partial sums of (r - x0)^2 and w |x| for energy (solver.cpp:44-55)
__global__ void energy_partials(uint64_t n, const double* r, const double* x0, const double* x,
                                const double* w, double* part) {
    __shared__ double sq[256], sr[256];
    double q = 0.0, g = 0.0;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double d = r[i] - x0[i];
        q += d * d;
        g += w[i] * fabs(x[i]);
    }
    sq[threadIdx.x] = q;
    sr[threadIdx.x] = g;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            sq[threadIdx.x] += sq[threadIdx.x + o];
            sr[threadIdx.x] += sr[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = sq[0];
        part[2 * blockIdx.x + 1] = sr[0];
    }
}

__global__ void sub_kernel(uint64_t n, double* r, const double* x0) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) r[i] = __dsub_rn(r[i], x0[i]);
}

__global__ void delta_kernel(double* x, uint64_t i) { x[i] = 1.0; }

unsigned nblocks(uint64_t n, unsigned t = 256) { return static_cast<unsigned>((n + t - 1) / t); }

// Gram diagonals (precond.cpp:16-67) on the device (gram.cu): the reference's exact
// accumulation and first-touch order, bitwise; no host path.
void gram(wbx_ctx* ctx, const wbx_op* op, uint64_t cap_factor, double* diagM, double* diagM2) {
    need(ctx, "ctx");
    wbx::gram_device(ctx, op, cap_factor, diagM, diagM2);
}

}  // namespace

extern "C" {

const char* wbx_last_error(void) { return g_last_error.c_str(); }
int wbx_abi_version(void) { return WBX_ABI_VERSION; }

int wbx_ctx_create(int device, wbx_ctx** out) {
    return guard([&] {
        need(out, "out");
        auto ctx = std::make_unique<wbx_ctx>();
        ctx->device = device;
        WBX_CUDA(cudaSetDevice(device));
        WBX_CUDA(cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device));
        int coop = 0;
        WBX_CUDA(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
        if (!coop) wbx::fail(WBX_CUDA_ERROR, "device does not support cooperative launch");
        WBX_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        *out = ctx.release();
    });
}

int wbx_ctx_destroy(wbx_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        wbx::pgd_purge(ctx, nullptr);
        cudaStreamSynchronize(ctx->stream);
        cudaStreamDestroy(ctx->stream);
        delete ctx;
    });
}

void* wbx_ctx_stream(wbx_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int wbx_ctx_synchronize(wbx_ctx* ctx) {
    return guard([&] {
        need(ctx, "ctx");
        WBX_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

uint64_t wbx_ctx_launch_count(const wbx_ctx* ctx) { return ctx ? ctx->launches : 0; }

// ---------------------------------------------------------------- wavelets
int wbx_make_filters(uint32_t family, uint32_t order, double* lo, double* hi, uint32_t* length) {
    return guard([&] {
        need(lo, "lo");
        need(hi, "hi");
        need(length, "length");
        wbx::make_filters(family, order, lo, hi, length);
    });
}

int wbx_parse_filter(const char* name, uint32_t* family, uint32_t* order) {
    return guard([&] {
        need(name, "name");
        std::string s;
        for (const char* c = name; *c; ++c) s.push_back(static_cast<char>(std::tolower(*c)));
        auto tail = [&](size_t pre) -> uint32_t {
            const std::string t = s.substr(pre);
            if (t.empty() || t.find_first_not_of("0123456789") != std::string::npos)
                wbx::fail(WBX_UNSUPPORTED_FILTER, "cannot parse filter name: " + std::string(name));
            return static_cast<uint32_t>(std::stoul(t));
        };
        uint32_t f, o;
        if (s == "haar") {
            f = WBX_HAAR;
            o = 1;
        } else if (s.rfind("db", 0) == 0) {
            f = WBX_DAUBECHIES;
            o = tail(2);
        } else if (s.rfind("symmlet", 0) == 0) {
            f = WBX_SYMMLET;
            o = tail(7);
        } else if (s.rfind("sym", 0) == 0) {
            f = WBX_SYMMLET;
            o = tail(3);
        } else {
            wbx::fail(WBX_UNSUPPORTED_FILTER, "unknown filter name: " + std::string(name));
        }
        double lo[20], hi[20];
        uint32_t l;
        wbx::make_filters(f, o, lo, hi, &l);  // validates the order
        *family = f;
        *order = o;
    });
}

int wbx_make_layout(uint32_t ndim, const uint64_t* dims, uint32_t J, wbx_band* bands,
                    uint32_t* nbands) {
    return guard([&] {
        need(dims, "dims");
        std::vector<wbx_band> b;
        wbx::make_layout(ndim, dims, J, b);
        if (nbands) *nbands = static_cast<uint32_t>(b.size());
        if (bands) std::copy(b.begin(), b.end(), bands);
    });
}

int wbx_basis_create(wbx_ctx* ctx, uint32_t family, uint32_t order, uint32_t ndim,
                     const uint64_t* dims, uint32_t J, wbx_basis** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(dims, "dims");
        need(out, "out");
        auto b = std::make_unique<wbx_basis>();
        b->ctx = ctx;
        b->family = family;
        b->order = order;
        b->ndim = ndim;
        b->J = J;
        wbx::make_filters(family, order, b->lo, b->hi, &b->len);
        wbx::make_layout(ndim, dims, J, b->bands);
        b->dims[0] = dims[0];
        b->dims[1] = ndim == 2 ? dims[1] : 1;
        b->n = b->dims[0] * b->dims[1];
        b->work_a.alloc(b->n);
        b->work_b.alloc(b->n);
        *out = b.release();
    });
}

int wbx_basis_destroy(wbx_basis* basis) {
    return guard([&] { delete basis; });
}

int wbx_analyze_dev(wbx_ctx* ctx, const wbx_basis* basis, const double* u_dev, double* x_dev) {
    return guard([&] {
        need(ctx, "ctx");
        need(basis, "basis");
        wbx::analyze_dev(const_cast<wbx_basis*>(basis), u_dev, x_dev, ctx->stream);
    });
}

int wbx_synthesize_dev(wbx_ctx* ctx, const wbx_basis* basis, const double* x_dev, double* u_dev) {
    return guard([&] {
        need(ctx, "ctx");
        need(basis, "basis");
        wbx::synthesize_dev(const_cast<wbx_basis*>(basis), x_dev, u_dev, ctx->stream);
    });
}

int wbx_analyze(wbx_ctx* ctx, const wbx_basis* basis, const double* u, double* x) {
    return guard([&] {
        need(ctx, "ctx");
        need(basis, "basis");
        need(u, "u");
        need(x, "x");
        const uint64_t n = basis->n;
        wbx::DevBuf<double> du(n), dx(n);
        du.upload(u, n, ctx->stream);
        wbx::analyze_dev(const_cast<wbx_basis*>(basis), du.p, dx.p, ctx->stream);
        WBX_CUDA(cudaMemcpyAsync(x, dx.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        WBX_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int wbx_synthesize(wbx_ctx* ctx, const wbx_basis* basis, const double* x, double* u) {
    return guard([&] {
        need(ctx, "ctx");
        need(basis, "basis");
        need(u, "u");
        need(x, "x");
        const uint64_t n = basis->n;
        wbx::DevBuf<double> du(n), dx(n);
        dx.upload(x, n, ctx->stream);
        wbx::synthesize_dev(const_cast<wbx_basis*>(basis), dx.p, du.p, ctx->stream);
        WBX_CUDA(cudaMemcpyAsync(u, du.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        WBX_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int wbx_single_wavelet(wbx_ctx* ctx, const wbx_basis* basis, uint32_t level, uint32_t orientation,
                       double* u) {
    return guard([&] {
        need(ctx, "ctx");
        need(basis, "basis");
        need(u, "u");
        const wbx_band* band = nullptr;
        for (const auto& b : basis->bands)
            if (b.level == level && b.orientation == orientation) band = &b;
        if (!band)
            wbx::fail(WBX_BAND_NOT_FOUND, "no band (level=" + std::to_string(level) +
                                              ", e=" + std::to_string(orientation) + ")");
        const uint64_t n = basis->n;
        wbx::DevBuf<double> dx(n), du(n);
        WBX_CUDA(cudaMemsetAsync(dx.p, 0, n * sizeof(double), ctx->stream));
        delta_kernel<<<1, 1, 0, ctx->stream>>>(dx.p, band->offset);
        wbx::count_launch(ctx);
        wbx::synthesize_dev(const_cast<wbx_basis*>(basis), dx.p, du.p, ctx->stream);
        WBX_CUDA(cudaMemcpyAsync(u, du.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        WBX_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// ---------------------------------------------------------------- Theta_K
int wbx_op_create(wbx_ctx* ctx, uint64_t n, const uint64_t* row_offsets, const uint32_t* col_indices,
                  const double* values, wbx_op** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(out, "out");
        auto op = std::make_unique<wbx_op>();
        op->ctx = ctx;
        wbx::build_op(op.get(), n, row_offsets, col_indices, values);
        *out = op.release();
    });
}

int wbx_op_destroy(wbx_op* op) {
    return guard([&] {
        if (op) wbx::pgd_purge(nullptr, op);  // cached wbx_pgd solvers on it
        delete op;
    });
}

int wbx_op_set_layout(wbx_op* op, uint32_t ndim, const uint64_t* dims, uint32_t J) {
    return guard([&] {
        need(op, "op");
        need(dims, "dims");
        std::vector<wbx_band> bands;
        wbx::make_layout(ndim, dims, J, bands);  // make_layout's own errors (wavelet.cpp:32-70)
        if (dims[0] * (ndim == 2 ? dims[1] : 1) != op->n)
            wbx::fail(WBX_SHAPE_MISMATCH, "layout and operator sizes differ");
        wbx::pgd_purge(nullptr, op);  // cached wbx_pgd solvers chose engines for the old layout
        std::lock_guard<std::mutex> g(op->win_mu);
        op->has_layout = true;
        op->l_ndim = ndim;
        op->l_J = J;
        op->l_dims[0] = dims[0];
        op->l_dims[1] = ndim == 2 ? dims[1] : 1;
        op->l_bands = std::move(bands);
        op->circ_cache.clear();
    });
}

int wbx_op_get_info(const wbx_op* op, wbx_op_info* info) {
    return guard([&] {
        need(op, "op");
        need(info, "info");
        info->n = op->n;
        info->nnz = op->nnz;
        info->nonempty_rows = op->nR;
        info->nonempty_cols = op->nC;
        info->sell_rows_padded = op->A.slices * 32;
        info->sell_cols_padded = op->T.slices * 32;
        info->device_bytes = op->device_bytes;
        // one FISTA iteration, fp32: A stream (16 B per element pair, padded) + T stream +
        // y gather source (read once, |C|) + x0R, res write (|R|) + res read (|R|) +
        // y, x_prev, tau/p, thr read and y, x_prev write on C.
        info->bytes_per_iter_fp32 = 16 * (op->A.pairs + op->T.pairs) + 4 * op->nC + 4 * 3 * op->nR +
                                    4 * 6 * op->nC;
    });
}

int wbx_spmv(wbx_ctx* ctx, const wbx_op* op, int transpose, const double* x, double* y) {
    return guard([&] {
        need(ctx, "ctx");
        need(op, "op");
        need(x, "x");
        need(y, "y");
        const uint64_t n = op->n;
        wbx::DevBuf<double> dx(n), dy(n);
        dx.upload(x, n, ctx->stream);
        wbx::spmv_full_fp64(ctx, op, transpose, dx.p, dy.p);
        WBX_CUDA(cudaMemcpyAsync(y, dy.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        WBX_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int wbx_spmv_dev(wbx_ctx* ctx, const wbx_op* op, int transpose, int precision, const void* x_dev,
                 void* y_dev) {
    return guard([&] {
        need(ctx, "ctx");
        need(op, "op");
        if (precision == WBX_FP64)
            wbx::spmv_full_fp64(ctx, op, transpose, static_cast<const double*>(x_dev), static_cast<double*>(y_dev));
        else
            wbx::spmv_full_fp32(ctx, op, transpose, static_cast<const float*>(x_dev), static_cast<float*>(y_dev));
    });
}

int wbx_spmv_compact_dev(wbx_ctx* ctx, const wbx_op* op, int transpose, int precision,
                         const void* x_dev, void* y_dev) {
    return guard([&] {
        need(ctx, "ctx");
        need(op, "op");
        const wbx_sell& M = transpose ? op->T : op->A;
        if (precision == WBX_FP64) {
            wbx::spmv_compact<double>(ctx, M, static_cast<const double*>(x_dev), static_cast<double*>(y_dev),
                                      ctx->stream);
        } else {
            if (!(op->A.seg_ok && op->T.seg_ok))
                wbx::fail(WBX_TOO_LARGE, "operator rows longer than 496 nonzeros: fp32 layout unavailable");
            wbx::spmv_compact<float>(ctx, M, static_cast<const float*>(x_dev), static_cast<float*>(y_dev),
                                     ctx->stream);
        }
    });
}

int wbx_diag_spmv_compact_mode(wbx_ctx* ctx, const wbx_op* op, int transpose, int mode, const float* x_dev,
                               float* y_dev) {
    return guard([&] {
        need(ctx, "ctx");
        need(op, "op");
        if (mode < 0 || mode > 8) wbx::fail(WBX_BAD_SPEC, "unknown SpMV kernel mode");
        if (!(op->A.seg_ok && op->T.seg_ok)) wbx::fail(WBX_TOO_LARGE, "fp32 layout unavailable");
        wbx::spmv_compact<float>(ctx, transpose ? op->T : op->A, x_dev, y_dev, ctx->stream, mode);
    });
}

int wbx_diag_set_spmv_pf(long long bytes) {
    wbx::set_spmv_pf_bytes(bytes);
    return WBX_OK;
}

int wbx_approx_gradient(wbx_ctx* ctx, const wbx_op* op, const double* x, const double* x0, double* g) {
    return guard([&] {
        need(ctx, "ctx");
        need(op, "op");
        need(x, "x");
        need(x0, "x0");
        need(g, "g");
        const uint64_t n = op->n;
        wbx::DevBuf<double> dx(n), dx0(n), dr(n), dg(n);
        dx.upload(x, n, ctx->stream);
        dx0.upload(x0, n, ctx->stream);
        wbx::spmv_full_fp64(ctx, op, 0, dx.p, dr.p);
        sub_kernel<<<nblocks(n), 256, 0, ctx->stream>>>(n, dr.p, dx0.p);
        wbx::count_launch(ctx);
        wbx::spmv_full_fp64(ctx, op, 1, dr.p, dg.p);
        WBX_CUDA(cudaMemcpyAsync(g, dg.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        WBX_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// Thresholded circulant operator from its kept generator groups -> CSR.
// Walk (theta.cpp:236-275) + assemble (:180-201).
int wbx_theta_expand(uint32_t ndim, const uint64_t* dims, uint32_t J, uint64_t n_gens,
                     const uint32_t* blocks, const uint32_t* gen_index, const uint64_t* counts,
                     const double* values, uint64_t* nnz, uint64_t* row_offsets, uint32_t* col_indices,
                     double* out_values) {
    return guard([&] {
        need(dims, "dims");
        need(nnz, "nnz");
        std::vector<wbx_band> bands;
        wbx::make_layout(ndim, dims, J, bands);
        const uint64_t nb = bands.size();
        uint64_t total = 0;
        for (uint64_t g = 0; g < n_gens; ++g) {
            if (blocks[g] >= nb * nb) wbx::fail(WBX_BAND_NOT_FOUND, "block index out of range");
            const wbx_band& bi = bands[blocks[g] % nb];
            const wbx_band& bo = bands[blocks[g] / nb];
            const wbx_band& small = bi.level <= bo.level ? bo : bi;
            const wbx_band& big = bi.level <= bo.level ? bi : bo;
            if (counts[g] > small.shape[0] * small.shape[1])
                wbx::fail(WBX_BAD_SPEC, "generator count exceeds its multiplicity");
            if (gen_index[g] >= big.shape[0] * big.shape[1])
                wbx::fail(WBX_BAD_SPEC, "generator index out of range");
            total += counts[g];
        }
        if (row_offsets == nullptr) {
            *nnz = total;
            return;
        }
        need(col_indices, "col_indices");
        need(out_values, "values");
        const uint64_t n = dims[0] * (ndim == 2 ? dims[1] : 1);
        wbx::HostCsr csr = wbx::expand_generators(bands, ndim, n, n_gens, blocks, gen_index, counts, values);
        std::copy(csr.rowptr.begin(), csr.rowptr.end(), row_offsets);
        std::copy(csr.col.begin(), csr.col.end(), col_indices);
        std::copy(csr.val.begin(), csr.val.end(), out_values);
        *nnz = total;
    });
}

// ---------------------------------------------------------------- preconditioners
int wbx_gram_diagonals(wbx_ctx* ctx, const wbx_op* op, uint64_t nnz_cap_factor, double* diagM,
                       double* diagM2) {
    return guard([&] {
        need(op, "op");
        need(diagM, "diagM");
        need(diagM2, "diagM2");
        gram(ctx, op, nnz_cap_factor, diagM, diagM2);
    });
}

int wbx_spai(wbx_ctx* ctx, const wbx_op* op, double* p) {
    return guard([&] {
        need(op, "op");
        need(p, "p");
        std::vector<double> m(op->n), m2(op->n);
        gram(ctx, op, 50, m.data(), m2.data());
        for (uint64_t i = 0; i < op->n; ++i) p[i] = m[i] > 0.0 ? m2[i] / m[i] : 1.0;
    });
}

int wbx_jacobi(wbx_ctx* ctx, const wbx_op* op, double eps, double* p) {
    return guard([&] {
        need(op, "op");
        need(p, "p");
        if (eps <= 0.0) wbx::fail(WBX_BAD_EPSILON, "jacobi: epsilon must be positive");
        std::vector<double> m(op->n), m2(op->n);
        gram(ctx, op, 50, m.data(), m2.data());
        for (uint64_t i = 0; i < op->n; ++i) p[i] = std::max(m[i], eps);
    });
}

// ---------------------------------------------------------------- solver
int wbx_scale_weights(uint32_t ndim, const uint64_t* dims, uint32_t J, double* w) {
    return guard([&] {
        need(dims, "dims");
        need(w, "w");
        std::vector<wbx_band> bands;
        wbx::make_layout(ndim, dims, J, bands);
        for (const auto& b : bands) {
            const double v = b.orientation == 0 ? static_cast<double>(J) : static_cast<double>(b.level);
            std::fill(w + b.offset, w + b.offset + b.shape[0] * b.shape[1], v);
        }
    });
}

int wbx_prox_l1w(wbx_ctx* ctx, uint64_t n, const double* z0, double tau, const double* w, double lambda,
                 const double* p, double* z) {
    return guard([&] {
        need(ctx, "ctx");
        need(z0, "z0");
        need(w, "w");
        need(p, "p");
        need(z, "z");
        if (n == 0) return;
        wbx::DevBuf<double> d0(n), dw(n), dp(n), dz(n);
        d0.upload(z0, n, ctx->stream);
        dw.upload(w, n, ctx->stream);
        dp.upload(p, n, ctx->stream);
        prox_kernel<<<nblocks(n), 256, 0, ctx->stream>>>(n, d0.p, tau, dw.p, lambda, dp.p, dz.p);
        wbx::count_launch(ctx);
        WBX_CUDA(cudaMemcpyAsync(z, dz.p, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        WBX_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int wbx_energy(wbx_ctx* ctx, const wbx_op* op, const double* x, const double* x0, const double* w,
               double lambda, double* e) {
    return guard([&] {
        need(ctx, "ctx");
        need(op, "op");
        need(x, "x");
        need(x0, "x0");
        need(w, "w");
        need(e, "e");
        const uint64_t n = op->n;
        wbx::DevBuf<double> dx(n), dx0(n), dw(n), dr(n);
        dx.upload(x, n, ctx->stream);
        dx0.upload(x0, n, ctx->stream);
        dw.upload(w, n, ctx->stream);
        wbx::spmv_full_fp64(ctx, op, 0, dx.p, dr.p);
        const unsigned G = 2 * ctx->num_sms;
        wbx::DevBuf<double> part(2 * G);
        energy_partials<<<G, 256, 0, ctx->stream>>>(n, dr.p, dx0.p, dx.p, dw.p, part.p);
        wbx::count_launch(ctx);
        std::vector<double> h(2 * G);
        WBX_CUDA(cudaMemcpyAsync(h.data(), part.p, 2 * G * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        WBX_CUDA(cudaStreamSynchronize(ctx->stream));
        double q = 0.0, r = 0.0;
        for (unsigned b = 0; b < G; ++b) {
            q += h[2 * b];
            r += h[2 * b + 1];
        }
        *e = 0.5 * q + lambda * r;
    });
}

void wbx_solver_cfg_default(wbx_solver_cfg* cfg) {
    if (!cfg) return;
    cfg->max_iters = 500;
    cfg->rel_energy_tol = 1e-3;
    cfg->step_safety = 1.01;
    cfg->ref_energy = std::nan("");
    cfg->zero_momentum = 0;
    cfg->track_support = 0;
    cfg->track_energy = 0;
    cfg->precision = WBX_FP32;
    cfg->tau = 0.0;
}

int wbx_estimate_step(wbx_ctx* ctx, const wbx_op* op, const double* p, double step_safety, double* tau,
                      uint32_t* iters) {
    wbx_solver* s = nullptr;
    int st = guard([&] {
        need(ctx, "ctx");
        need(op, "op");
        need(p, "p");
        need(tau, "tau");
        wbx_solver_cfg cfg;
        wbx_solver_cfg_default(&cfg);
        cfg.max_iters = 0;
        cfg.step_safety = step_safety;
        cfg.precision = WBX_FP64;
        s = wbx::solver_new(ctx, op, nullptr, 0.0, cfg, 1);
        std::vector<double> w(op->n, 0.0);
        wbx::solver_setup(s, p, w.data());
        wbx::DevBuf<double> x0(op->n), xf(op->n);
        WBX_CUDA(cudaMemsetAsync(x0.p, 0, x0.bytes(), ctx->stream));
        wbx::solver_run(s, x0.p, xf.p);
        wbx_report rep{};
        wbx::solver_report(s, &rep);
        *tau = rep.tau;
        if (iters) *iters = rep.tau_iters;
    });
    if (s) wbx::solver_free(s);
    return st;
}

int wbx_pgd(wbx_ctx* ctx, const wbx_op* op, const double* x0, const double* w, double lambda, const double* p,
            const wbx_solver_cfg* cfg, int accelerate, double* x_final, wbx_report* report) {
    wbx_solver* s = nullptr;
    int st = guard([&] {
        need(ctx, "ctx");
        need(op, "op");
        need(x0, "x0");
        need(w, "w");
        need(p, "p");
        need(cfg, "cfg");
        need(x_final, "x_final");
        // a solver for (ctx, op, cfg, accelerate), reused across calls (layouts and buffers kept)
        s = wbx::pgd_acquire(ctx, op, *cfg, accelerate, lambda, p, w);
        const uint64_t n = op->n;
        double* dx0 = wbx::solver_x0_buf(s);
        double* dxf = wbx::solver_x_buf(s);
        WBX_CUDA(cudaMemcpyAsync(dx0, x0, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        wbx::solver_run(s, dx0, dxf);
        wbx::solver_report(s, report);
        WBX_CUDA(cudaMemcpyAsync(x_final, dxf, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        WBX_CUDA(cudaStreamSynchronize(ctx->stream));
        wbx::pgd_release(s);
        s = nullptr;
    });
    if (s) wbx::solver_free(s);  // an error: not returned to the cache
    return st;
}

int wbx_solver_create(wbx_ctx* ctx, const wbx_op* op, const wbx_basis* basis, const double* p, const double* w,
                      double lambda, const wbx_solver_cfg* cfg, wbx_solver** out) {
    return guard([&] {
        need(ctx, "ctx");
        need(op, "op");
        need(basis, "basis");
        need(p, "p");
        need(w, "w");
        need(cfg, "cfg");
        need(out, "out");
        if (basis->n != op->n) wbx::fail(WBX_SHAPE_MISMATCH, "operator and basis sizes differ");
        wbx_solver* s = wbx::solver_new(ctx, op, const_cast<wbx_basis*>(basis), lambda, *cfg, 1);
        try {
            wbx::solver_setup(s, p, w);
            wbx::solver_alloc_images(s);
        } catch (...) {
            wbx::solver_free(s);
            throw;
        }
        *out = s;
    });
}

int wbx_solver_destroy(wbx_solver* s) {
    return guard([&] {
        if (s) wbx::solver_free(s);
    });
}

int wbx_deblur_dev(wbx_solver* s, const double* u0_dev, double* u_dev, int clamp);

}  // extern "C"

extern "C" void wbx_set_last_error(const char* msg) { g_last_error = msg ? msg : ""; }
