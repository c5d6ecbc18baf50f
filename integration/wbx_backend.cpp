// proj/src/wbx_backend.cpp — route the hot path of waveblur to libwbx.so (B200).
//
// Defines the reference's hot-path functions (wavelet.hpp:88,91; theta.hpp:83-89;
// precond.hpp:26-34; solver.hpp:86-105; SparseThetaOp::apply/apply_adjoint) and the PSF side
// (operators.hpp:44-77: generate_psf, convolve, apply_adjoint, add_noise, degrade) on top of
// the C ABI in include/wbx.h. The reference's CPU definitions stay in the library under a
// `*_host` name. SparseThetaOp and ExactThetaOp (solver.cpp:11-31) run on
// the device (ExactThetaOp::apply/apply_adjoint/ops_per_pixel are defined here, so the exact
// operator's FFT route, its estimate_step and its fista/ista run through wbx_exact_*); only
// user-defined ThetaOps keep the host loop. WBX_BACKEND_PRECISION=32 selects the fp32 hot
// path; the default is the fp64 mode, bitwise equal to the reference.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <list>
#include <map>
#include <mutex>
#include <stdexcept>
#include <type_traits>
#include <variant>
#include <vector>

#include "waveblur/operators.hpp"
#include "waveblur/precond.hpp"
#include "waveblur/solver.hpp"
#include "waveblur/theta.hpp"
#include "waveblur/wavelet.hpp"
#include "wbx.h"

namespace waveblur {

// the reference's own definitions, renamed by the build
double energy_host(const std::vector<double>& x, const DeblurProblem& problem);
double estimate_step_host(const ThetaOp& op, const DiagonalPreconditioner& P, double step_safety);
SolveReport ista_host(const DeblurProblem& problem, const DiagonalPreconditioner& P, const SolverConfig& c);
SolveReport fista_host(const DeblurProblem& problem, const DiagonalPreconditioner& P, const SolverConfig& c);

namespace {

std::recursive_mutex mu;  // one libwbx context, calls serialised (the reference's are re-entrant)

void check(int st) {  // status -> the reference's exception types (image.hpp:10-36)
    if (st == WBX_OK) return;
    const char* m = wbx_last_error();
    switch (st) {
        case WBX_SHAPE_MISMATCH: throw ShapeMismatch(m);
        case WBX_UNSUPPORTED_FILTER: throw UnsupportedFilter(m);
        case WBX_BAND_NOT_FOUND: throw BandNotFound(m);
        case WBX_BAD_SPEC: throw BadSpec(m);
        case WBX_TOO_LARGE: throw TooLarge(m);
        case WBX_BAD_EPSILON: throw BadEpsilon(m);
        case WBX_MEMORY_GUARD: throw MemoryGuard(m);
        case WBX_NONFINITE_ENERGY: throw NonFiniteEnergy(m);
        case WBX_IO_ERROR: throw IoError(m);
        default: throw std::runtime_error(m);
    }
}

wbx_ctx* ctx() {
    static wbx_ctx* c = [] {
        wbx_ctx* p = nullptr;
        check(wbx_ctx_create(0, &p));
        return p;
    }();
    return c;
}

int precision() {
    static const int p = [] {
        const char* e = std::getenv("WBX_BACKEND_PRECISION");
        return e && std::atoi(e) == 32 ? WBX_FP32 : WBX_FP64;
    }();
    return p;
}

void mix(uint64_t& h, const void* data, std::size_t bytes) {
    const auto* p = static_cast<const unsigned char*>(data);
    for (; bytes >= 8; bytes -= 8, p += 8) {
        uint64_t w;
        std::memcpy(&w, p, 8);
        h = (h ^ w) * 0x100000001b3ULL;
    }
    for (; bytes; --bytes, ++p) h = (h ^ *p) * 0x100000001b3ULL;
}

// Device layouts of Theta and its transpose, cached by content: building them costs more
// than a product, and the reference's loops apply one operator many times.
wbx_op* device_op(const SparseOperator& s) {
    if (s.row_offsets.size() != s.n + 1 || s.col_indices.size() != s.values.size())
        throw ShapeMismatch("SparseOperator: inconsistent CSR arrays");
    uint64_t key = 0xcbf29ce484222325ULL;
    mix(key, &s.n, sizeof s.n);
    mix(key, s.row_offsets.data(), s.row_offsets.size() * sizeof(uint64_t));
    mix(key, s.col_indices.data(), s.col_indices.size() * sizeof(uint32_t));
    mix(key, s.values.data(), s.values.size() * sizeof(double));
    mix(key, s.layout.dims.data(), s.layout.dims.size() * sizeof(std::size_t));
    mix(key, &s.layout.J, sizeof s.layout.J);
    struct Entry {
        uint64_t key;
        wbx_op* op;
    };
    static std::list<Entry> cache;  // most recent first
    for (auto it = cache.begin(); it != cache.end(); ++it)
        if (it->key == key) {
            cache.splice(cache.begin(), cache, it);
            return cache.front().op;
        }
    wbx_op* op = nullptr;
    check(wbx_op_create(ctx(), s.n, s.row_offsets.data(), s.col_indices.data(), s.values.data(), &op));
    if (!s.layout.dims.empty() && s.layout.total() == s.n) {  // SparseOperator::layout (theta.hpp:55)
        const uint64_t d[2] = {s.layout.dims[0], s.layout.dims.size() == 2 ? s.layout.dims[1] : 1};
        const int st = wbx_op_set_layout(op, static_cast<uint32_t>(s.layout.dims.size()), d, s.layout.J);
        if (st != WBX_OK) {
            wbx_op_destroy(op);
            check(st);
        }
    }
    cache.push_front({key, op});
    if (cache.size() > 4) {
        wbx_op_destroy(cache.back().op);
        cache.pop_back();
    }
    return op;
}

wbx_basis* device_basis(const WaveletBasis& b) {
    struct Entry {
        uint32_t family, order, J;
        std::vector<uint64_t> dims;
        wbx_basis* basis;
    };
    static std::list<Entry> cache;
    const auto fam = static_cast<uint32_t>(b.filters.family);
    const std::vector<uint64_t> dims(b.dims().begin(), b.dims().end());
    for (auto& e : cache)
        if (e.family == fam && e.order == b.filters.order && e.J == b.levels() && e.dims == dims) return e.basis;
    wbx_basis* p = nullptr;
    check(wbx_basis_create(ctx(), fam, b.filters.order, static_cast<uint32_t>(dims.size()), dims.data(),
                           b.levels(), &p));
    cache.push_front({fam, b.filters.order, b.levels(), dims, p});
    return p;
}

const SparseOperator* sparse_of(const ThetaOp* op) {
    const auto* s = dynamic_cast<const SparseThetaOp*>(op);
    return s ? &s->sparse() : nullptr;
}

// ExactThetaOp keeps its PSF and basis private (solver.hpp:41-52); its member functions,
// defined below, register them here so that the free functions (estimate_step, fista) can
// route an exact operator to the device.
struct ExactParts {
    const Psf* psf;
    const WaveletBasis* basis;
};
std::map<const ExactThetaOp*, ExactParts>& exact_registry() {
    static std::map<const ExactThetaOp*, ExactParts> m;
    return m;
}

// the device exact operator of (PSF kernel, basis), cached by content (building it plans
// the FFTs and uploads the kernel spectrum)
wbx_exact_op* device_exact(const Psf& psf, const WaveletBasis& b) {
    const Image& k = psf.kernel;
    if (k.dims != b.dims()) throw ShapeMismatch("ExactThetaOp: PSF and basis dims differ");
    uint64_t key = 0xcbf29ce484222325ULL;
    mix(key, k.v.data(), k.v.size() * sizeof(double));
    const auto fam = static_cast<uint32_t>(b.filters.family);
    const uint32_t meta[3] = {fam, static_cast<uint32_t>(b.filters.order), static_cast<uint32_t>(b.levels())};
    mix(key, meta, sizeof meta);
    for (std::size_t d : b.dims()) {
        const uint64_t dd = d;
        mix(key, &dd, sizeof dd);
    }
    struct Entry {
        uint64_t key;
        wbx_exact_op* e;
    };
    static std::list<Entry> cache;
    for (auto it = cache.begin(); it != cache.end(); ++it)
        if (it->key == key) {
            cache.splice(cache.begin(), cache, it);
            return cache.front().e;
        }
    wbx_exact_op* e = nullptr;
    check(wbx_exact_op_create(ctx(), device_basis(b), k.v.data(), &e));
    cache.push_front({key, e});
    if (cache.size() > 4) {
        wbx_exact_op_destroy(cache.back().e);
        cache.pop_back();
    }
    return e;
}

const ExactParts* exact_of(const ThetaOp* op) {
    const auto* e = dynamic_cast<const ExactThetaOp*>(op);
    if (!e) return nullptr;
    e->ops_per_pixel();  // (re)registers this operator's PSF and basis
    return &exact_registry().at(e);
}

void require_len(std::size_t got, std::size_t want, const char* what) {
    if (got != want) throw ShapeMismatch(std::string(what) + ": vector length mismatch");
}

SolveReport pgd(const DeblurProblem& p, const DiagonalPreconditioner& P, const SolverConfig& c, int accelerate) {
    const SparseOperator* s = sparse_of(p.op);
    const ExactParts* ex = s ? nullptr : exact_of(p.op);
    if (!s && !ex) return accelerate ? fista_host(p, P, c) : ista_host(p, P, c);
    const std::size_t n = p.op->dim();
    if (p.x0.size() != n || p.weights.size() != n || P.p.size() != n)
        throw ShapeMismatch("solver: inconsistent problem dimensions");  // solver.cpp:106-107
    std::lock_guard<std::recursive_mutex> g(mu);
    wbx_solver_cfg cfg;
    wbx_solver_cfg_default(&cfg);
    cfg.max_iters = c.max_iters;
    cfg.rel_energy_tol = c.rel_energy_tol;
    cfg.step_safety = c.step_safety;
    cfg.ref_energy = c.ref_energy;
    cfg.zero_momentum = c.zero_momentum;
    cfg.track_support = c.track_support;
    cfg.track_energy = 1;  // SolveReport always carries E(x_k)
    cfg.precision = precision();
    SolveReport r;
    r.x_final.resize(n);
    r.energies.resize(c.max_iters);
    std::vector<uint64_t> supp(c.max_iters);
    wbx_report rep{};
    rep.energies = r.energies.data();
    rep.support_sizes = supp.data();
    if (s) {
        check(wbx_pgd(ctx(), device_op(*s), p.x0.data(), p.weights.data(), p.lambda, P.p.data(), &cfg, accelerate,
                      r.x_final.data(), &rep));
        r.ops_per_pixel_per_iter = rep.ops_per_pixel_per_iter;
    } else {  // the exact FFT operator: fp64, the reference's expressions (exact_op.cu)
        check(wbx_pgd_exact(device_exact(*ex->psf, *ex->basis), p.x0.data(), p.weights.data(), p.lambda,
                            P.p.data(), &cfg, accelerate, r.x_final.data(), &rep));
        r.ops_per_pixel_per_iter = p.op->ops_per_pixel();
    }
    r.iters_used = rep.iters_used;
    r.energies.resize(rep.iters_used);
    if (c.track_support) r.support_sizes.assign(supp.begin(), supp.begin() + rep.iters_used);
    r.wall_time_s = rep.wall_time_s;
    r.initial_energy = rep.initial_energy;
    return r;
}

}  // namespace

WaveletCoeffs analyze(const Image& signal, const WaveletBasis& basis) {
    signal.require_dyadic();
    if (signal.dims != basis.dims()) throw ShapeMismatch("signal dims do not match basis");
    std::lock_guard<std::recursive_mutex> g(mu);
    WaveletCoeffs x;
    x.layout = &basis.layout;
    x.values.resize(basis.layout.total());
    check(wbx_analyze(ctx(), device_basis(basis), signal.v.data(), x.values.data()));
    return x;
}

Image synthesize(const WaveletCoeffs& coeffs, const WaveletBasis& basis) {
    if (coeffs.values.size() != basis.layout.total())
        throw ShapeMismatch("coefficient length does not match basis");
    std::lock_guard<std::recursive_mutex> g(mu);
    Image u(basis.dims());
    check(wbx_synthesize(ctx(), device_basis(basis), coeffs.values.data(), u.v.data()));
    return u;
}

std::vector<double> spmv(const SparseOperator& op, const std::vector<double>& x) {
    require_len(x.size(), op.n, "spmv");
    std::lock_guard<std::recursive_mutex> g(mu);
    std::vector<double> y(op.n);
    check(wbx_spmv(ctx(), device_op(op), 0, x.data(), y.data()));
    return y;
}

std::vector<double> spmv_t(const SparseOperator& op, const std::vector<double>& x) {
    require_len(x.size(), op.n, "spmv_t");
    std::lock_guard<std::recursive_mutex> g(mu);
    std::vector<double> y(op.n);
    check(wbx_spmv(ctx(), device_op(op), 1, x.data(), y.data()));
    return y;
}

std::vector<double> approx_gradient(const SparseOperator& op, const std::vector<double>& x,
                                    const std::vector<double>& x0) {
    require_len(x.size(), op.n, "approx_gradient");
    require_len(x0.size(), op.n, "approx_gradient");
    std::lock_guard<std::recursive_mutex> g(mu);
    std::vector<double> y(op.n);
    check(wbx_approx_gradient(ctx(), device_op(op), x.data(), x0.data(), y.data()));
    return y;
}

// ---- PSFs and the FFT convolution (operators.cpp:98-387)
Psf generate_psf(const PsfSpec& spec, const std::vector<std::size_t>& dims) {
    double params[4] = {0.0, 0.0, 0.0, 0.0};
    uint32_t kind = WBX_PSF_GAUSSIAN;
    std::visit(
        [&](const auto& sp) {
            using T = std::decay_t<decltype(sp)>;
            if constexpr (std::is_same_v<T, GaussianSpec>) {
                params[0] = sp.sigma;
            } else if constexpr (std::is_same_v<T, SkewedGaussianSpec>) {
                kind = WBX_PSF_SKEWED;
                params[0] = sp.sigma;
            } else if constexpr (std::is_same_v<T, MotionSpec>) {
                kind = WBX_PSF_MOTION;
                params[0] = sp.points;
                params[1] = sp.sigma1;
                params[2] = sp.sigma2;
                params[3] = static_cast<double>(sp.seed);
                if (sp.seed >= (1ULL << 53)) throw BadSpec("motion blur: seed must be < 2^53 here");
            } else if constexpr (std::is_same_v<T, AirySpec>) {
                kind = WBX_PSF_AIRY;
                params[0] = sp.scale;
            } else {
                kind = WBX_PSF_DEFOCUS;
                params[0] = sp.radius;
            }
        },
        spec);
    Image tmp(dims);
    tmp.require_dyadic();
    std::lock_guard<std::recursive_mutex> g(mu);
    const std::vector<uint64_t> d(dims.begin(), dims.end());
    check(wbx_generate_psf(kind == WBX_PSF_MOTION ? ctx() : nullptr, kind, params,
                           static_cast<uint32_t>(d.size()), d.data(), tmp.v.data()));
    return Psf{std::move(tmp), spec};
}

namespace {
Image conv(const Image& u, const Psf& psf, int adjoint) {
    if (u.dims != psf.kernel.dims) throw ShapeMismatch("convolve: image/kernel dims differ");
    u.require_dyadic();
    std::lock_guard<std::recursive_mutex> g(mu);
    Image out(u.dims);
    const std::vector<uint64_t> d(u.dims.begin(), u.dims.end());
    check(wbx_convolve(ctx(), static_cast<uint32_t>(d.size()), d.data(), psf.kernel.v.data(), u.v.data(), adjoint,
                       out.v.data()));
    return out;
}
}  // namespace

Image convolve(const Image& u, const Psf& psf) { return conv(u, psf, 0); }

Image apply_adjoint(const Image& u, const Psf& psf) { return conv(u, psf, 1); }

Image add_noise(const Image& u, double sigma, std::uint64_t seed) {
    if (sigma < 0.0) throw BadSpec("noise sigma must be >= 0");
    std::lock_guard<std::recursive_mutex> g(mu);
    Image out(u.dims);
    check(wbx_add_noise(ctx(), u.size(), u.v.data(), sigma, seed, out.v.data()));
    return out;
}

Image degrade(const Image& u, const DegradationModel& model) {
    if (u.dims != model.psf.kernel.dims) throw ShapeMismatch("convolve: image/kernel dims differ");
    if (model.noise_sigma < 0.0) throw BadSpec("noise sigma must be >= 0");
    u.require_dyadic();
    std::lock_guard<std::recursive_mutex> g(mu);
    Image out(u.dims);
    const std::vector<uint64_t> d(u.dims.begin(), u.dims.end());
    check(wbx_degrade(ctx(), static_cast<uint32_t>(d.size()), d.data(), model.psf.kernel.v.data(), u.v.data(),
                      model.noise_sigma, model.seed, out.v.data()));
    return out;
}

std::vector<double> SparseThetaOp::apply(const std::vector<double>& x) const { return spmv(sparse(), x); }

std::vector<double> SparseThetaOp::apply_adjoint(const std::vector<double>& x) const {
    return spmv_t(sparse(), x);
}

// ExactThetaOp (solver.cpp:21-31): analyze(convolve(synthesize(x), psf)) and the adjoint
// with the conjugate kernel spectrum, on the device in the reference's arithmetic (bitwise)
double ExactThetaOp::ops_per_pixel() const {
    std::lock_guard<std::recursive_mutex> g(mu);
    exact_registry()[this] = ExactParts{&psf_, basis_};
    return exact_ops_per_pixel(*basis_);
}

std::vector<double> ExactThetaOp::apply(const std::vector<double>& x) const {
    require_len(x.size(), basis_->layout.total(), "ExactThetaOp::apply");
    std::lock_guard<std::recursive_mutex> g(mu);
    std::vector<double> y(x.size());
    check(wbx_exact_apply(device_exact(psf_, *basis_), 0, x.data(), y.data()));
    return y;
}

std::vector<double> ExactThetaOp::apply_adjoint(const std::vector<double>& x) const {
    require_len(x.size(), basis_->layout.total(), "ExactThetaOp::apply_adjoint");
    std::lock_guard<std::recursive_mutex> g(mu);
    std::vector<double> y(x.size());
    check(wbx_exact_apply(device_exact(psf_, *basis_), 1, x.data(), y.data()));
    return y;
}

GramDiagonals gram_diagonals(const SparseOperator& op, std::size_t nnz_cap_factor) {
    std::lock_guard<std::recursive_mutex> g(mu);
    GramDiagonals d;
    d.diagM.resize(op.n);
    d.diagM2.resize(op.n);
    check(wbx_gram_diagonals(ctx(), device_op(op), nnz_cap_factor, d.diagM.data(), d.diagM2.data()));
    return d;
}

DiagonalPreconditioner jacobi(const SparseOperator& op, double eps) {
    std::lock_guard<std::recursive_mutex> g(mu);
    DiagonalPreconditioner P{std::vector<double>(op.n), PrecondKind::Jacobi};
    check(wbx_jacobi(ctx(), device_op(op), eps, P.p.data()));
    return P;
}

DiagonalPreconditioner spai(const SparseOperator& op) {
    std::lock_guard<std::recursive_mutex> g(mu);
    DiagonalPreconditioner P{std::vector<double>(op.n), PrecondKind::Spai};
    check(wbx_spai(ctx(), device_op(op), P.p.data()));
    return P;
}

double energy(const std::vector<double>& x, const DeblurProblem& problem) {
    const SparseOperator* s = sparse_of(problem.op);
    if (!s) return energy_host(x, problem);
    require_len(x.size(), problem.x0.size(), "energy");
    require_len(x.size(), s->n, "energy");
    std::lock_guard<std::recursive_mutex> g(mu);
    double e = 0.0;
    check(wbx_energy(ctx(), device_op(*s), x.data(), problem.x0.data(), problem.weights.data(), problem.lambda,
                     &e));
    return e;
}

std::vector<double> prox_weighted_l1_P(const std::vector<double>& z0, double tau, const std::vector<double>& weights,
                                       double lambda, const DiagonalPreconditioner& P) {
    require_len(weights.size(), z0.size(), "prox_weighted_l1_P");
    require_len(P.p.size(), z0.size(), "prox_weighted_l1_P");
    std::lock_guard<std::recursive_mutex> g(mu);
    std::vector<double> z(z0.size());
    check(wbx_prox_l1w(ctx(), z0.size(), z0.data(), tau, weights.data(), lambda, P.p.data(), z.data()));
    return z;
}

double estimate_step(const ThetaOp& op, const DiagonalPreconditioner& P, double step_safety) {
    const SparseOperator* s = sparse_of(&op);
    const ExactParts* ex = s ? nullptr : exact_of(&op);
    if (!s && !ex) return estimate_step_host(op, P, step_safety);
    require_len(P.p.size(), op.dim(), "estimate_step");
    std::lock_guard<std::recursive_mutex> g(mu);
    double tau = 0.0;
    uint32_t iters = 0;
    if (s)
        check(wbx_estimate_step(ctx(), device_op(*s), P.p.data(), step_safety, &tau, &iters));
    else
        check(wbx_estimate_step_exact(device_exact(*ex->psf, *ex->basis), P.p.data(), step_safety, &tau, &iters));
    return tau;
}

SolveReport ista(const DeblurProblem& p, const DiagonalPreconditioner& P, const SolverConfig& c) {
    return pgd(p, P, c, 0);
}

SolveReport fista(const DeblurProblem& p, const DiagonalPreconditioner& P, const SolverConfig& c) {
    return pgd(p, P, c, 1);
}

}  // namespace waveblur
