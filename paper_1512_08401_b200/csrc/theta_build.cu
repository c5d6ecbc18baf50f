// Host-side assembly of thresholded wavelet-domain operators Theta_K.
//
// * expand_generators: the kept (block, generator, count) groups of the reference's global
//   top-K walk -> CSR, exactly as threshold_impl's walk (theta.cpp:236-275) and assemble
//   (:180-201) would produce it (rows, then columns ascending).
// * wbx_theta_varying: the spatially varying operator of BASELINE configs C3/C4, which has
//   no reference implementation. Each column mu of Theta is the wavelet
//   expansion of the blurred wavelet psi_mu; for a blur whose PSF varies smoothly with the
//   spatial row, the column of the stationary operator of the PSF at psi_mu's position is
//   the natural approximation. Columns are linearly interpolated between the two
//   bracketing levels of a sigma ladder of stationary operators (each the reference's own
//   thresholded Theta_K); the index set of a column is the union of the two levels' sets.
#include <algorithm>
#include <cmath>
#include <thread>

#include "internal.hpp"

extern "C" void wbx_set_last_error(const char* msg);

namespace wbx {

HostCsr expand_generators(const std::vector<wbx_band>& bands, uint32_t ndim, uint64_t n, uint64_t n_gens,
                          const uint32_t* blocks, const uint32_t* gen_index, const uint64_t* counts,
                          const double* values) {
    const uint64_t nb = bands.size();
    struct Tri {
        uint32_t row, col;
        double v;
    };
    uint64_t total = 0;
    for (uint64_t g = 0; g < n_gens; ++g) total += counts[g];
    std::vector<Tri> tri;
    tri.reserve(total);
    const uint32_t d = ndim;
    for (uint64_t g = 0; g < n_gens; ++g) {
        const wbx_band& bi = bands[blocks[g] % nb];
        const wbx_band& bo = bands[blocks[g] / nb];
        const bool in_finer = bi.level <= bo.level;
        const uint64_t* gshape = in_finer ? bi.shape : bo.shape;
        const wbx_band& small = in_finer ? bo : bi;
        uint64_t v[2] = {0, 0}, rem = gen_index[g];
        for (uint32_t k = d; k-- > 0;) {
            v[k] = rem % gshape[k];
            rem /= gshape[k];
        }
        for (uint64_t q = 0; q < counts[g]; ++q) {
            uint64_t idx[2] = {0, 0}, r = q;
            for (uint32_t k = d; k-- > 0;) {
                idx[k] = r % small.shape[k];
                r /= small.shape[k];
            }
            uint64_t nf = 0, mf = 0;
            for (uint32_t k = 0; k < d; ++k) {
                uint64_t nk, mk;
                if (in_finer) {
                    const uint64_t s = bi.shape[k] / bo.shape[k];
                    nk = idx[k];
                    mk = (v[k] + s * idx[k]) % bi.shape[k];
                } else {
                    const uint64_t s = bo.shape[k] / bi.shape[k];
                    mk = idx[k];
                    nk = (v[k] + s * idx[k]) % bo.shape[k];
                }
                nf = nf * bo.shape[k] + nk;
                mf = mf * bi.shape[k] + mk;
            }
            tri.push_back({static_cast<uint32_t>(bo.offset + nf), static_cast<uint32_t>(bi.offset + mf), values[g]});
        }
    }
    // counting sort by row, then columns ascending within each row
    HostCsr out;
    out.rowptr.assign(n + 1, 0);
    for (const auto& t : tri) ++out.rowptr[t.row + 1];
    for (uint64_t i = 0; i < n; ++i) out.rowptr[i + 1] += out.rowptr[i];
    out.col.resize(tri.size());
    out.val.resize(tri.size());
    {
        std::vector<uint64_t> cur(out.rowptr.begin(), out.rowptr.end() - 1);
        for (const auto& t : tri) {
            const uint64_t p = cur[t.row]++;
            out.col[p] = t.col;
            out.val[p] = t.v;
        }
    }
    for (uint64_t r = 0; r < n; ++r) {
        const uint64_t b = out.rowptr[r], e = out.rowptr[r + 1];
        if (e - b < 2) continue;
        std::vector<std::pair<uint32_t, double>> row(e - b);
        for (uint64_t k = b; k < e; ++k) row[k - b] = {out.col[k], out.val[k]};
        std::sort(row.begin(), row.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
        for (uint64_t k = b; k < e; ++k) {
            out.col[k] = row[k - b].first;
            out.val[k] = row[k - b].second;
        }
    }
    return out;
}

}  // namespace wbx

extern "C" int wbx_theta_varying(uint32_t ndim, const uint64_t* dims, uint32_t J, uint32_t nlevels,
                                 const double* sigmas, const uint64_t* level_ngens, const uint32_t* blocks,
                                 const uint32_t* gen_index, const uint64_t* counts, const double* values,
                                 double sigma_first_row, double sigma_last_row, uint64_t* nnz,
                                 uint64_t** row_offsets, uint32_t** col_indices, double** out_values) {
    try {
        if (!dims || !sigmas || !level_ngens || !nnz || !row_offsets || !col_indices || !out_values)
            wbx::fail(WBX_INVALID_ARGUMENT, "null argument to wbx_theta_varying");
        if (nlevels < 1) wbx::fail(WBX_BAD_SPEC, "sigma ladder needs at least one level");
        for (uint32_t l = 1; l < nlevels; ++l)
            if (!(sigmas[l] > sigmas[l - 1])) wbx::fail(WBX_BAD_SPEC, "sigma ladder must be increasing");
        std::vector<wbx_band> bands;
        wbx::make_layout(ndim, dims, J, bands);
        const uint64_t n = dims[0] * (ndim == 2 ? dims[1] : 1);
        // expand every level
        std::vector<wbx::HostCsr> lv(nlevels);
        uint64_t g0 = 0;
        for (uint32_t l = 0; l < nlevels; ++l) {
            lv[l] = wbx::expand_generators(bands, ndim, n, level_ngens[l], blocks + g0, gen_index + g0, counts + g0,
                                           values + g0);
            g0 += level_ngens[l];
        }
        // per column: bracketing level and interpolation weight from the spatial row of
        // the column's wavelet (band level t, index i along dim 0: row (i + 0.5) 2^t)
        std::vector<uint8_t> lev(n);
        std::vector<double> alpha(n);
        const double H = static_cast<double>(dims[0]);
        for (const auto& b : bands) {
            const uint64_t cnt = b.shape[0] * b.shape[1];
            for (uint64_t q = 0; q < cnt; ++q) {
                const uint64_t i = q / b.shape[1];
                const double y = (static_cast<double>(i) + 0.5) * std::ldexp(1.0, static_cast<int>(b.level));
                double s = sigma_first_row + (sigma_last_row - sigma_first_row) * (y / H);
                s = std::min(std::max(s, sigmas[0]), sigmas[nlevels - 1]);
                uint32_t l = 0;
                while (l + 1 < nlevels && sigmas[l + 1] <= s) ++l;
                double a = 0.0;
                if (l + 1 < nlevels) a = (s - sigmas[l]) / (sigmas[l + 1] - sigmas[l]);
                lev[b.offset + q] = static_cast<uint8_t>(l);
                alpha[b.offset + q] = a;
            }
        }
        // merge: row r gets, for every level L, the entries whose column brackets L
        std::vector<uint64_t> rp(n + 1, 0);
        std::vector<std::vector<std::pair<uint32_t, double>>> rows_by_thread;
        const unsigned nth = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
        std::vector<std::vector<uint32_t>> tcol(nth);
        std::vector<std::vector<double>> tval(nth);
        std::vector<std::vector<uint64_t>> tlen(nth);
        const uint64_t chunk = (n + nth - 1) / nth;
        std::vector<std::thread> pool;
        for (unsigned t = 0; t < nth; ++t) {
            pool.emplace_back([&, t] {
                const uint64_t r0 = t * chunk, r1 = std::min<uint64_t>(n, r0 + chunk);
                std::vector<std::pair<uint32_t, double>> acc;
                for (uint64_t r = r0; r < r1; ++r) {
                    acc.clear();
                    for (uint32_t L = 0; L < nlevels; ++L) {
                        const auto& c = lv[L];
                        for (uint64_t k = c.rowptr[r]; k < c.rowptr[r + 1]; ++k) {
                            const uint32_t mu = c.col[k];
                            const uint32_t l = lev[mu];
                            const double a = alpha[mu];
                            double w;
                            if (L == l)
                                w = 1.0 - a;
                            else if (L == l + 1 && a > 0.0)
                                w = a;
                            else
                                continue;
                            acc.push_back({mu, w * c.val[k]});
                        }
                    }
                    std::stable_sort(acc.begin(), acc.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
                    uint64_t len = 0;
                    for (size_t k = 0; k < acc.size();) {
                        double v = acc[k].second;
                        size_t j = k + 1;
                        for (; j < acc.size() && acc[j].first == acc[k].first; ++j) v += acc[j].second;
                        if (v != 0.0) {
                            tcol[t].push_back(acc[k].first);
                            tval[t].push_back(v);
                            ++len;
                        }
                        k = j;
                    }
                    tlen[t].push_back(len);
                }
            });
        }
        for (auto& th : pool) th.join();
        uint64_t r = 0;
        for (unsigned t = 0; t < nth; ++t)
            for (uint64_t len : tlen[t]) {
                rp[r + 1] = rp[r] + len;
                ++r;
            }
        const uint64_t total = rp[n];
        auto* ro = static_cast<uint64_t*>(std::malloc((n + 1) * sizeof(uint64_t)));
        auto* ci = static_cast<uint32_t*>(std::malloc(std::max<uint64_t>(total, 1) * sizeof(uint32_t)));
        auto* va = static_cast<double*>(std::malloc(std::max<uint64_t>(total, 1) * sizeof(double)));
        if (!ro || !ci || !va) wbx::fail(WBX_MEMORY_GUARD, "wbx_theta_varying: host allocation failed");
        std::copy(rp.begin(), rp.end(), ro);
        uint64_t p = 0;
        for (unsigned t = 0; t < nth; ++t) {
            std::copy(tcol[t].begin(), tcol[t].end(), ci + p);
            std::copy(tval[t].begin(), tval[t].end(), va + p);
            p += tcol[t].size();
        }
        *nnz = total;
        *row_offsets = ro;
        *col_indices = ci;
        *out_values = va;
        return WBX_OK;
    } catch (const wbx::Error& e) {
        wbx_set_last_error(e.what());
        return e.status;
    } catch (const std::exception& e) {
        wbx_set_last_error(e.what());
        return WBX_MEMORY_GUARD;
    }
}

extern "C" void wbx_free(void* p) { std::free(p); }
