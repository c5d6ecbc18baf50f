// oracle/tools/oracle_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// Runs the UNMODIFIED reference library (oracle/_ref/libwaveblur_ref.so, built from
// /root/reference/proj/src by oracle/Makefile) through the same steps as the
// reference CLI's `deblur` command (`proj/tools/waveblur.cpp:252-319`):
//   synthetic_scene -> degrade -> build_theta_conv -> threshold_weighted|naive
//   -> analyze -> scale_weights -> spai|jacobi|identity -> fista -> synthesize
// and writes golden fixtures (raw little-endian binaries + meta.json) that the
// tests/ parity suite and bench.py's reference arm consume.
//
// It also emits the thresholded operator in "generator-list" form: the kept
// (block, generator index, count, value) groups of the reference's global top-K
// walk (`proj/src/theta.cpp:206-276`, restated below). Expanding that list over
// the circulant blocks reproduces the reference CSR exactly; the driver checks
// this bitwise before writing anything (`expand_ok` in meta.json).
//
// Usage:
//   oracle_driver --out DIR [--dims H W | --dims N] [--family F --order O] [--J J]
//                 [--psf gaussian --sigma S] [--K K | --Kfactor F] [--mode dyadic|uniform]
//                 [--noise SIG] [--seed SEED] [--lambda L] [--iters I]
//                 [--precond spai|jacobi|identity] [--write-op] [--u0 FILE]
//                 [--bench-reps R] [--bench-warmup W] [--no-solve] [--exact]
//                 [--gens FILE]
// --gens FILE: take the thresholded operator from a generator list (24-byte records
// {u32 block, u32 gen_index, u64 count, f64 value}, e.g. tests/golden/*.npz gen_*) expanded
// by the reference's walk, instead of running build_theta_conv + threshold (the bench's
// reference arm: the timed unit is the deblur, not the operator build).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "waveblur/image.hpp"
#include "waveblur/operators.hpp"
#include "waveblur/precond.hpp"
#include "waveblur/solver.hpp"
#include "waveblur/theta.hpp"
#include "waveblur/wavelet.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

using namespace waveblur;
using clk = std::chrono::steady_clock;

namespace {

struct Gen {
    std::uint32_t block;
    std::uint32_t gen_index;
    std::uint64_t count;
    double value;
};

double secs(clk::time_point a, clk::time_point b) {
    return std::chrono::duration<double>(b - a).count();
}

template <typename T>
void write_bin(const std::filesystem::path& p, const std::vector<T>& v) {
    std::ofstream f(p, std::ios::binary);
    f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(T)));
    if (!f) throw std::runtime_error("write failed: " + p.string());
}

std::vector<double> read_f64(const std::string& path, std::size_t n) {
    std::ifstream f(path, std::ios::binary);
    std::vector<double> v(n);
    f.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(n * sizeof(double)));
    if (!f) throw std::runtime_error("short read: " + path);
    return v;
}

// Restatement of the candidate ordering + walk of threshold_impl (theta.cpp:215-274),
// keeping only (block, generator, count) groups instead of triplets.
std::vector<Gen> kept_generators(const CirculantTheta& theta, std::size_t K,
                                 const std::vector<double>& col_band_weight) {
    const auto& bands = theta.basis->layout.bands;
    struct Cand {
        double key;
        std::uint32_t block, v;
    };
    std::vector<Cand> cands;
    for (std::size_t b = 0; b < theta.blocks.size(); ++b) {
        const auto& blk = theta.blocks[b];
        const double w = col_band_weight[blk.in_band];
        for (std::size_t v = 0; v < blk.generator.size(); ++v) {
            double key = std::abs(blk.generator[v]) * w;
            if (key > 0.0) cands.push_back({key, static_cast<std::uint32_t>(b), static_cast<std::uint32_t>(v)});
        }
    }
    std::sort(cands.begin(), cands.end(), [](const Cand& a, const Cand& b) {
        if (a.key != b.key) return a.key > b.key;
        if (a.block != b.block) return a.block < b.block;
        return a.v < b.v;
    });
    std::vector<Gen> out;
    std::size_t kept = 0;
    for (const auto& c : cands) {
        if (kept >= K) break;
        const auto& blk = theta.blocks[c.block];
        const Band& bi = bands[blk.in_band];
        const Band& bo = bands[blk.out_band];
        const std::size_t mult = (bi.level <= bo.level ? bo : bi).count();
        const std::size_t take = std::min(mult, K - kept);
        out.push_back({c.block, c.v, take, blk.generator[c.v]});
        kept += take;
    }
    return out;
}

// Expand a generator list to CSR (theta.cpp:236-275 walk + assemble :180-201).
SparseOperator expand(const SubbandLayout& layout, const std::vector<Gen>& gens) {
    struct Tri {
        std::uint32_t row, col;
        double value;
    };
    const auto& bands = layout.bands;
    const std::size_t nb = bands.size(), d = layout.dims.size();
    std::vector<Tri> tri;
    for (const auto& g : gens) {
        const Band& bi = bands[g.block % nb];
        const Band& bo = bands[g.block / nb];
        const bool in_finer = bi.level <= bo.level;
        const auto& gshape = in_finer ? bi.shape : bo.shape;
        const Band& small = in_finer ? bo : bi;
        std::vector<std::size_t> v(d);
        std::size_t rem = g.gen_index;
        for (std::size_t k = d; k-- > 0;) {
            v[k] = rem % gshape[k];
            rem /= gshape[k];
        }
        for (std::uint64_t q = 0; q < g.count; ++q) {
            std::vector<std::size_t> idx(d);
            std::size_t r = q;
            for (std::size_t k = d; k-- > 0;) {
                idx[k] = r % small.shape[k];
                r /= small.shape[k];
            }
            std::size_t nflat = 0, mflat = 0;
            for (std::size_t k = 0; k < d; ++k) {
                std::size_t nk, mk;
                if (in_finer) {
                    std::size_t s = bi.shape[k] / bo.shape[k];
                    nk = idx[k];
                    mk = (v[k] + s * idx[k]) % bi.shape[k];
                } else {
                    std::size_t s = bo.shape[k] / bi.shape[k];
                    mk = idx[k];
                    nk = (v[k] + s * idx[k]) % bo.shape[k];
                }
                nflat = nflat * bo.shape[k] + nk;
                mflat = mflat * bi.shape[k] + mk;
            }
            tri.push_back({static_cast<std::uint32_t>(bo.offset + nflat),
                           static_cast<std::uint32_t>(bi.offset + mflat), g.value});
        }
    }
    std::sort(tri.begin(), tri.end(), [](const Tri& a, const Tri& b) {
        return a.row != b.row ? a.row < b.row : a.col < b.col;
    });
    SparseOperator op;
    op.n = layout.total();
    op.layout = layout;
    op.row_offsets.assign(op.n + 1, 0);
    for (const auto& t : tri) {
        ++op.row_offsets[t.row + 1];
        op.col_indices.push_back(t.col);
        op.values.push_back(t.value);
    }
    for (std::size_t i = 0; i < op.n; ++i) op.row_offsets[i + 1] += op.row_offsets[i];
    return op;
}

bool same_csr(const SparseOperator& a, const SparseOperator& b) {
    if (a.n != b.n || a.row_offsets != b.row_offsets || a.col_indices != b.col_indices) return false;
    if (a.values.size() != b.values.size()) return false;
    return std::memcmp(a.values.data(), b.values.data(), a.values.size() * sizeof(double)) == 0;
}

std::string fmt(double x) {
    char buf[40];
    std::snprintf(buf, sizeof buf, "%.17g", x);
    return buf;
}

std::string json_array(const std::vector<double>& v) {
    std::string s = "[";
    for (std::size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + fmt(v[i]);
    return s + "]";
}

}  // namespace

int main(int argc, char** argv) {
    std::string out, family = "daubechies", mode = "dyadic", precond = "spai", u0_path, method = "fista", gens_path;
    std::vector<std::size_t> dims = {256, 256};
    unsigned order = 4, J = 4;
    double sigma = 5.0, noise = 5e-3, lambda = 1e-4, kfactor = 3.0;
    std::size_t K = 0, iters = 50, bench_reps = 0, bench_warmup = 0;
    std::uint64_t seed = 2024;
    bool write_op = false, solve = true, exact = false;
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        auto next = [&]() -> std::string {
            if (i + 1 >= argc) throw std::runtime_error("missing value for " + a);
            return argv[++i];
        };
        if (a == "--out") out = next();
        else if (a == "--dims") {
            dims.clear();
            while (i + 1 < argc && argv[i + 1][0] != '-') dims.push_back(std::stoull(argv[++i]));
        } else if (a == "--family") family = next();
        else if (a == "--order") order = static_cast<unsigned>(std::stoul(next()));
        else if (a == "--J") J = static_cast<unsigned>(std::stoul(next()));
        else if (a == "--sigma") sigma = std::stod(next());
        else if (a == "--K") K = std::stoull(next());
        else if (a == "--Kfactor") kfactor = std::stod(next());
        else if (a == "--mode") mode = next();
        else if (a == "--noise") noise = std::stod(next());
        else if (a == "--seed") seed = std::stoull(next());
        else if (a == "--lambda") lambda = std::stod(next());
        else if (a == "--iters") iters = std::stoull(next());
        else if (a == "--precond") precond = next();
        else if (a == "--write-op") write_op = true;
        else if (a == "--u0") u0_path = next();
        else if (a == "--bench-reps") bench_reps = std::stoull(next());
        else if (a == "--bench-warmup") bench_warmup = std::stoull(next());
        else if (a == "--no-solve") solve = false;
        else if (a == "--method") method = next();
        else if (a == "--exact") exact = true;
        else if (a == "--gens") gens_path = next();
        else throw std::runtime_error("unknown flag " + a);
    }
    if (out.empty()) throw std::runtime_error("--out required");
    std::filesystem::create_directories(out);
    const std::filesystem::path od(out);

    FilterFamily fam = family == "haar" ? FilterFamily::Haar
                       : family == "symmlet" ? FilterFamily::Symmlet
                                             : FilterFamily::Daubechies;
    WaveletBasis basis = make_basis(fam, order, dims, J);
    const std::size_t n = basis.layout.total();
    if (K == 0) K = static_cast<std::size_t>(std::llround(kfactor * static_cast<double>(n)));

    auto t0 = clk::now();
    Psf psf = generate_psf(GaussianSpec{sigma}, dims);
    Image clean = synthetic_scene(dims);
    Image observed = u0_path.empty() ? degrade(clean, DegradationModel{psf, noise, seed})
                                     : Image(dims);
    if (!u0_path.empty()) observed.v = read_f64(u0_path, n);
    auto t1 = clk::now();
    std::vector<Gen> gens;
    SparseOperator sp;
    bool expand_ok = true;
    auto t2 = clk::now(), t3 = t2;
    if (!gens_path.empty()) {
        std::ifstream f(gens_path, std::ios::binary);
        Gen g;
        while (f.read(reinterpret_cast<char*>(&g.block), 4) && f.read(reinterpret_cast<char*>(&g.gen_index), 4) &&
               f.read(reinterpret_cast<char*>(&g.count), 8) && f.read(reinterpret_cast<char*>(&g.value), 8))
            gens.push_back(g);
        if (gens.empty()) throw std::runtime_error("no generator records in " + gens_path);
        sp = expand(basis.layout, gens);
        t2 = t3 = clk::now();
    } else {
        CirculantTheta theta = build_theta_conv(psf, basis);
        t2 = clk::now();
        std::vector<double> band_w(basis.layout.bands.size(), 1.0);
        if (mode == "uniform") {
            sp = threshold_naive(theta, K);
        } else {
            WeightVector wv = dyadic_weights(basis.layout);
            for (std::size_t b = 0; b < band_w.size(); ++b) band_w[b] = wv.sigma[basis.layout.bands[b].offset];
            sp = threshold_weighted(theta, K, wv);
        }
        t3 = clk::now();
        gens = kept_generators(theta, K, band_w);
        SparseOperator re = expand(basis.layout, gens);
        expand_ok = same_csr(re, sp);
    }
    if (!expand_ok) std::fprintf(stderr, "generator-list expansion does NOT reproduce the reference CSR\n");

    {
        std::ofstream f(od / "gens.bin", std::ios::binary);
        for (const auto& g : gens) {
            f.write(reinterpret_cast<const char*>(&g.block), 4);
            f.write(reinterpret_cast<const char*>(&g.gen_index), 4);
            f.write(reinterpret_cast<const char*>(&g.count), 8);
            f.write(reinterpret_cast<const char*>(&g.value), 8);
        }
    }
    if (write_op) write_operator(sp, (od / "op.wtheta").string());
    write_bin(od / "u_clean.bin", clean.v);
    write_bin(od / "u0.bin", observed.v);

    std::ostringstream meta;
    meta << "{\n  \"dims\": [" << dims[0];
    for (std::size_t k = 1; k < dims.size(); ++k) meta << ", " << dims[k];
    meta << "],\n  \"family\": \"" << family << "\", \"order\": " << order << ", \"J\": " << J
         << ",\n  \"psf\": \"gaussian\", \"sigma\": " << fmt(sigma) << ", \"K\": " << K
         << ", \"mode\": \"" << mode << "\", \"noise\": " << fmt(noise) << ", \"seed\": " << seed
         << ", \"lambda\": " << fmt(lambda) << ", \"method\": \"" << method << "\", \"iters\": " << iters << ", \"precond\": \""
         << precond << "\",\n  \"nnz\": " << sp.nnz() << ", \"n_gens\": " << gens.size()
         << ", \"expand_ok\": " << (expand_ok ? "true" : "false") << ", \"u0_from_file\": "
         << (u0_path.empty() ? "false" : "true")
         << ",\n  \"t_degrade_s\": " << fmt(secs(t0, t1)) << ", \"t_build_theta_s\": "
         << fmt(secs(t1, t2)) << ", \"t_threshold_s\": " << fmt(secs(t2, t3));
#ifdef _OPENMP
    meta << ", \"omp_threads\": " << omp_get_max_threads();
#endif

    if (solve) {
        SparseThetaOp op(sp);
        auto s0 = clk::now();
        std::vector<double> x0 = analyze(observed, basis).values;
        auto s1 = clk::now();
        DiagonalPreconditioner P = precond == "spai" ? spai(sp)
                                   : precond == "jacobi"
                                       ? [&] {
                                             GramDiagonals g = gram_diagonals(sp);
                                             double mx = 0.0;
                                             for (double dd : g.diagM) mx = std::max(mx, dd);
                                             return jacobi(sp, std::max(1e-3 * mx, 1e-300));
                                         }()
                                       : identity_precond(n);
        auto s2 = clk::now();
        DeblurProblem prob;
        prob.op = &op;
        prob.x0 = x0;
        prob.weights = scale_weights(basis.layout);
        prob.lambda = lambda;
        SolverConfig cfg;
        cfg.max_iters = iters;
        const double tau = estimate_step(op, P, cfg.step_safety);
        auto s3 = clk::now();
        SolveReport rep = method == "ista" ? ista(prob, P, cfg) : fista(prob, P, cfg);
        auto s4 = clk::now();
        Image restored = synthesize(WaveletCoeffs{&basis.layout, rep.x_final}, basis);
        auto s5 = clk::now();
        write_bin(od / "x0.bin", x0);
        write_bin(od / "p.bin", P.p);
        write_bin(od / "x_final.bin", rep.x_final);
        write_bin(od / "restored.bin", restored.v);
        write_bin(od / "energies.bin", rep.energies);
        meta << ",\n  \"tau\": " << fmt(tau) << ", \"iters_used\": " << rep.iters_used
             << ", \"initial_energy\": " << fmt(rep.initial_energy)
             << ", \"final_energy\": " << fmt(rep.energies.back())
             << ",\n  \"t_analyze_s\": " << fmt(secs(s0, s1)) << ", \"t_precond_s\": "
             << fmt(secs(s1, s2)) << ", \"t_estimate_step_s\": " << fmt(secs(s2, s3))
             << ", \"t_fista_s\": " << fmt(secs(s3, s4)) << ", \"fista_wall_time_s\": "
             << fmt(rep.wall_time_s) << ", \"t_synthesize_s\": " << fmt(secs(s4, s5));
        Image clamped = restored;
        for (auto& v : clamped.v) v = std::clamp(v, 0.0, 1.0);
        meta << ",\n  \"psnr_observed_db\": " << fmt(psnr(clean, observed))
             << ", \"psnr_restored_db\": " << fmt(psnr(clean, clamped));

        // Reference-arm timing: the deblur unit (analyze + fista incl. tau + synthesize),
        // the reference's own code path, repeated.
        if (bench_reps > 0) {
            std::vector<double> times;
            for (std::size_t r = 0; r < bench_warmup + bench_reps; ++r) {
                auto b0 = clk::now();
                DeblurProblem pb = prob;
                pb.x0 = analyze(observed, basis).values;
                SolveReport rr = fista(pb, P, cfg);
                Image rs = synthesize(WaveletCoeffs{&basis.layout, rr.x_final}, basis);
                auto b1 = clk::now();
                if (r >= bench_warmup) times.push_back(secs(b0, b1));
                if (rs.v.size() != n) return 3;
            }
            meta << ",\n  \"bench_deblur_s\": " << json_array(times);
        }
    }
    // ExactThetaOp (solver.cpp:21-29, the FFT operator): the PSF kernel, one forward and one
    // adjoint application to x0 = analyze(u0), estimate_step and `iters` FISTA iterations
    // with the identity preconditioner (the exact-fista comparator, waveblur.cpp:387-397)
    if (exact) {
        write_bin(od / "psf.bin", psf.kernel.v);
        ExactThetaOp eop(psf, basis);
        const std::vector<double> x0 = analyze(observed, basis).values;
        write_bin(od / "exact_apply.bin", eop.apply(x0));
        write_bin(od / "exact_adjoint.bin", eop.apply_adjoint(x0));
        DiagonalPreconditioner I = identity_precond(n);
        DeblurProblem pe;
        pe.op = &eop;
        pe.x0 = x0;
        pe.weights = scale_weights(basis.layout);
        pe.lambda = lambda;
        SolverConfig ce;
        ce.max_iters = iters;
        const double tau_e = estimate_step(eop, I, ce.step_safety);
        SolveReport re = fista(pe, I, ce);
        write_bin(od / "exact_x_final.bin", re.x_final);
        write_bin(od / "exact_energies.bin", re.energies);
        meta << ",\n  \"exact_tau\": " << fmt(tau_e) << ", \"exact_iters_used\": " << re.iters_used;
    }
    meta << "\n}\n";
    std::ofstream(od / "meta.json") << meta.str();
    std::cout << meta.str();
    return expand_ok ? 0 : 2;
}
