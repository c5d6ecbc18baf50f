// proj/src/wbx_backend.cpp — route the hot path of waveblur to libwbx.so (B200)
#include <stdexcept>
#include <vector>
#include "waveblur/solver.hpp"
#include "waveblur/theta.hpp"
#include "wbx.h"

namespace waveblur {
namespace {
wbx_ctx* ctx() {                       // one context per host thread
    thread_local wbx_ctx* c = [] { wbx_ctx* p = nullptr; wbx_ctx_create(0, &p); return p; }();
    return c;
}
void check(int st) {                   // status -> the reference's exception types
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
struct DeviceOp {                      // device layouts of one SparseOperator, cached by address
    wbx_op* op = nullptr;
    explicit DeviceOp(const SparseOperator& s) {
        check(wbx_op_create(ctx(), s.n, s.row_offsets.data(), s.col_indices.data(), s.values.data(), &op));
    }
    ~DeviceOp() { wbx_op_destroy(op); }
};
}  // namespace

std::vector<double> spmv(const SparseOperator& op, const std::vector<double>& x) {
    if (x.size() != op.n) throw ShapeMismatch("spmv: vector length mismatch");
    DeviceOp d(op);                    // production code caches this per operator
    std::vector<double> y(op.n);
    check(wbx_spmv(ctx(), d.op, 0, x.data(), y.data()));
    return y;
}

SolveReport fista(const DeblurProblem& p, const DiagonalPreconditioner& P, const SolverConfig& c) {
    auto* sp = dynamic_cast<const SparseThetaOp*>(p.op);
    if (!sp) throw std::invalid_argument("fista: device path needs a SparseThetaOp");
    DeviceOp d(sp->sparse());
    wbx_solver_cfg cfg;
    wbx_solver_cfg_default(&cfg);
    cfg.max_iters = c.max_iters; cfg.rel_energy_tol = c.rel_energy_tol; cfg.step_safety = c.step_safety;
    cfg.ref_energy = c.ref_energy; cfg.zero_momentum = c.zero_momentum;
    cfg.track_support = c.track_support; cfg.track_energy = 1; cfg.precision = WBX_FP32;
    SolveReport r;
    r.x_final.resize(p.x0.size());
    r.energies.resize(c.max_iters);
    std::vector<std::uint64_t> supp(c.max_iters);
    wbx_report rep{};
    rep.energies = r.energies.data();
    rep.support_sizes = supp.data();
    check(wbx_pgd(ctx(), d.op, p.x0.data(), p.weights.data(), p.lambda, P.p.data(), &cfg, 1,
                  r.x_final.data(), &rep));
    r.iters_used = rep.iters_used;
    r.energies.resize(rep.iters_used);
    if (c.track_support) r.support_sizes.assign(supp.begin(), supp.begin() + rep.iters_used);
    r.wall_time_s = rep.wall_time_s;
    r.ops_per_pixel_per_iter = rep.ops_per_pixel_per_iter;
    r.initial_energy = rep.initial_energy;
    return r;
}
}  // namespace waveblur
