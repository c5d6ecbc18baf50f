// Gram diagonals of M = Theta^T Theta on the device (gram_diagonals, precond.cpp:16-67):
//   diag(M)_i  = sum_k Theta_ki^2                       (column i, ascending row k)
//   diag(M2)_i = sum_c M_ic^2,  M_ic = sum_k Theta_ki Theta_kc
// with the reference's exact fp64 operation order, so SPAI / Jacobi are bitwise equal:
//   for each row k of column i (ascending), for each column c of row k (ascending):
//       acc[c] = acc[c] + Theta_ki * Theta_kc          (no contraction)
//   then s = s + acc[c]^2 over c in FIRST-TOUCH order.
// One warp per column. A row's columns are distinct, so the 32 lanes of one step update
// distinct accumulators: each (c) sees its contributions in ascending k, as on the host. The
// accumulators live in a per-warp open-addressing table in shared memory; first touches are
// appended to a list in (k, c) order by a warp prefix count. A column whose 2-hop set does
// not fit the shared-memory table is queued and recomputed by a second pass whose per-warp
// tables live in global memory, sized from the column's 2-hop bound (sum of the lengths of
// the rows it touches): no host fallback, every column is computed on the device with the
// same operation order.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "internal.hpp"

namespace wbx {
namespace {

constexpr int kGramWarps = 4;            // warps per CTA
constexpr uint32_t kGramCap = 2048;      // shared-memory table slots per warp (power of two)
constexpr uint32_t kEmpty = 0xffffffffu;

// one warp's accumulator table: key / val / first-touch order, `cap` slots (power of two);
// the shared-memory tables keep 16-bit order entries (14 B per slot: 2 CTAs of 4 warps per SM)
template <typename ORD>
struct GramTab {
    uint32_t* key;
    double* val;
    ORD* order;
    uint32_t cap;
};

template <typename ORD>
__global__ void __launch_bounds__(kGramWarps * 32) gram_kernel(uint64_t ncols, const uint32_t* __restrict__ cols,
                                                              const uint64_t* __restrict__ rp,
                                                              const uint32_t* __restrict__ cl,
                                                              const double* __restrict__ vl,
                                                              const uint64_t* __restrict__ toff,
                                                              const uint32_t* __restrict__ trow,
                                                              const double* __restrict__ tval, double* diagM,
                                                              double* diagM2, unsigned long long* touched,
                                                              uint32_t smem_cap, uint32_t* gkey, double* gval,
                                                              uint32_t* gorder, uint32_t gcap, uint32_t* ovf_list,
                                                              unsigned* ovf_count) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kGramWarps + warp;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * kGramWarps;
    GramTab<ORD> S;
    if (gkey == nullptr) {  // shared-memory tables: [val x cap][key x cap][order x cap] per warp
        unsigned char* b = smem_raw + static_cast<size_t>(warp) * smem_cap * (12u + sizeof(ORD));
        S.val = reinterpret_cast<double*>(b);
        S.key = reinterpret_cast<uint32_t*>(b + static_cast<size_t>(smem_cap) * 8u);
        S.order = reinterpret_cast<ORD*>(S.key + smem_cap);
        S.cap = smem_cap;
    } else {  // second pass: this warp's slice of the global tables
        S.key = gkey + gw * gcap;
        S.val = gval + gw * gcap;
        S.order = reinterpret_cast<ORD*>(gorder) + gw * gcap;
        S.cap = gcap;
    }
    for (uint32_t t = lane; t < S.cap; t += 32) {
        S.key[t] = kEmpty;
        S.val[t] = 0.0;
    }
    __syncwarp();
    unsigned long long cnt_total = 0;
    for (uint64_t q = gw; q < ncols; q += nw) {
        const uint64_t i = cols ? cols[q] : q;
        const uint64_t k0 = toff[i], k1 = toff[i + 1];
        if (lane == 0) {  // diag(M): ascending rows, no contraction
            double s = 0.0;
            for (uint64_t k = k0; k < k1; ++k) s = __dadd_rn(s, __dmul_rn(tval[k], tval[k]));
            diagM[i] = s;
        }
        uint32_t nlist = 0;
        bool full = false;
        unsigned long long cnt = 0;
        for (uint64_t k = k0; k < k1; ++k) {
            const uint32_t r = trow[k];
            const double a = tval[k];
            for (uint64_t j0 = rp[r]; j0 < rp[r + 1]; j0 += 32) {
                const uint64_t j = j0 + lane;
                const bool act = j < rp[r + 1];
                uint32_t slot = 0;
                bool fresh = false, zero_before = false;
                if (act) {
                    const uint32_t c = cl[j];
                    uint32_t h = (c * 2654435761u) & (S.cap - 1);
                    for (uint32_t probe = 0;; ++probe) {
                        if (probe == S.cap) {
                            full = true;
                            break;
                        }
                        const uint32_t kk = S.key[h];
                        if (kk == c) break;
                        if (kk == kEmpty) {
                            const uint32_t prev = atomicCAS(&S.key[h], kEmpty, c);
                            if (prev == kEmpty) {
                                fresh = true;
                                break;
                            }
                            if (prev == c) break;
                        }
                        h = (h + 1) & (S.cap - 1);
                    }
                    slot = h;
                }
                if (__any_sync(0xffffffffu, full)) {
                    full = true;
                    break;
                }
                // first touches appended in lane (= ascending column) order
                const unsigned fm = __ballot_sync(0xffffffffu, act && fresh);
                if (act && fresh) S.order[nlist + __popc(fm & ((1u << lane) - 1u))] = static_cast<ORD>(slot);
                nlist += __popc(fm);
                if (act) {
                    const double old = S.val[slot];
                    zero_before = old == 0.0;
                    S.val[slot] = __dadd_rn(old, __dmul_rn(a, vl[j]));
                }
                cnt += __popc(__ballot_sync(0xffffffffu, act && zero_before));
                __syncwarp();
            }
            if (full) break;
        }
        if (full) {  // only in the shared-memory pass: queue the column for the global pass
            if (lane == 0) ovf_list[atomicAdd(ovf_count, 1u)] = static_cast<uint32_t>(i);
            // reset the whole table (its state is unknown) and carry on
            for (uint32_t t = lane; t < S.cap; t += 32) {
                S.key[t] = kEmpty;
                S.val[t] = 0.0;
            }
            __syncwarp();
            continue;
        }
        cnt_total += cnt;
        __syncwarp();
        if (lane == 0) {  // sum of squares in first-touch order
            double s = 0.0;
            for (uint32_t t = 0; t < nlist; ++t) {
                const double v = S.val[S.order[t]];
                s = __dadd_rn(s, __dmul_rn(v, v));
            }
            diagM2[i] = s;
        }
        __syncwarp();
        for (uint32_t t = lane; t < nlist; t += 32) {
            const uint32_t sl = S.order[t];
            S.key[sl] = kEmpty;
            S.val[sl] = 0.0;
        }
        __syncwarp();
    }
    if (lane == 0 && cnt_total) atomicAdd(touched, cnt_total);
}

}  // namespace

void gram_device(wbx_ctx* ctx, const wbx_op* op, uint64_t cap_factor, double* diagM, double* diagM2) {
    const uint64_t n = op->n, nnz = op->nnz;
    const auto& rp = op->h_rowptr;
    const auto& cl = op->h_col;
    const auto& vl = op->h_val;
    // CSC of Theta (rows of each column ascending), as in gram_host
    std::vector<uint64_t> toff(n + 1, 0);
    for (uint64_t k = 0; k < nnz; ++k) ++toff[cl[k] + 1];
    for (uint64_t i = 0; i < n; ++i) toff[i + 1] += toff[i];
    std::vector<uint32_t> trow(nnz);
    std::vector<double> tval(nnz);
    {
        std::vector<uint64_t> cur(toff.begin(), toff.end() - 1);
        for (uint64_t r = 0; r < n; ++r)
            for (uint64_t k = rp[r]; k < rp[r + 1]; ++k) {
                const uint64_t pos = cur[cl[k]]++;
                trow[pos] = static_cast<uint32_t>(r);
                tval[pos] = vl[k];
            }
    }
    cudaStream_t st = ctx->stream;
    DevBuf<uint64_t> d_rp(n + 1), d_toff(n + 1);
    DevBuf<uint32_t> d_cl(std::max<uint64_t>(nnz, 1)), d_trow(std::max<uint64_t>(nnz, 1));
    DevBuf<double> d_vl(std::max<uint64_t>(nnz, 1)), d_tval(std::max<uint64_t>(nnz, 1)), d_m(n), d_m2(n);
    DevBuf<unsigned long long> d_cnt(1);
    DevBuf<unsigned> d_novf(1);
    DevBuf<uint32_t> d_ovf(n);
    d_rp.upload(rp.data(), n + 1, st);
    d_toff.upload(toff.data(), n + 1, st);
    d_cl.upload(cl.data(), nnz, st);
    d_vl.upload(vl.data(), nnz, st);
    d_trow.upload(trow.data(), nnz, st);
    d_tval.upload(tval.data(), nnz, st);
    WBX_CUDA(cudaMemsetAsync(d_cnt.p, 0, sizeof(unsigned long long), st));
    WBX_CUDA(cudaMemsetAsync(d_novf.p, 0, sizeof(unsigned), st));
    // shared-memory table size (WBX_GRAM_CAP: a smaller power of two, to exercise the global
    // pass in tests)
    uint32_t cap = kGramCap;
    if (const char* e = std::getenv("WBX_GRAM_CAP")) {
        const long v = std::atol(e);
        if (v >= 32 && v <= static_cast<long>(kGramCap) && (v & (v - 1)) == 0) cap = static_cast<uint32_t>(v);
    }
    const unsigned smem = kGramWarps * cap * 14u;
    WBX_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(gram_kernel<uint16_t>),
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kGramWarps * kGramCap * 14u)));
    const unsigned grid = 2u * static_cast<unsigned>(ctx->num_sms);
    gram_kernel<uint16_t><<<grid, kGramWarps * 32, smem, st>>>(n, nullptr, d_rp.p, d_cl.p, d_vl.p, d_toff.p, d_trow.p, d_tval.p,
                                                     d_m.p, d_m2.p, d_cnt.p, cap, nullptr, nullptr, nullptr, 0, d_ovf.p,
                                                     d_novf.p);
    count_launch(ctx);
    WBX_CUDA(cudaGetLastError());
    unsigned novf = 0;
    WBX_CUDA(cudaMemcpyAsync(&novf, d_novf.p, sizeof novf, cudaMemcpyDeviceToHost, st));
    WBX_CUDA(cudaStreamSynchronize(st));
    if (novf > 0) {
        // second pass over the overflowed columns: per-warp global tables sized from the
        // largest 2-hop bound among them (distinct touched columns <= sum of row lengths)
        std::vector<uint32_t> ovf(novf);
        WBX_CUDA(cudaMemcpy(ovf.data(), d_ovf.p, novf * sizeof(uint32_t), cudaMemcpyDeviceToHost));
        uint64_t bound = 0;
        for (uint32_t i : ovf) {
            uint64_t b = 0;
            for (uint64_t k = toff[i]; k < toff[i + 1]; ++k) b += rp[trow[k] + 1] - rp[trow[k]];
            bound = std::max(bound, std::min<uint64_t>(b, n));
        }
        uint64_t gcap = 64;
        while (gcap <= bound) gcap <<= 1;
        if (gcap > 0x80000000ull) fail(WBX_TOO_LARGE, "gram_diagonals: 2-hop set too large for 32-bit tables");
        // global tables: at most ~1 GiB, at least one CTA
        const uint64_t per_warp = gcap * 16u;
        uint64_t warps = std::min<uint64_t>(uint64_t(novf), uint64_t(grid) * kGramWarps);
        warps = std::min<uint64_t>(warps, std::max<uint64_t>(kGramWarps, (1ull << 30) / per_warp));
        const unsigned g2 = static_cast<unsigned>((warps + kGramWarps - 1) / kGramWarps);
        const uint64_t tw = uint64_t(g2) * kGramWarps;
        DevBuf<uint32_t> gkey(tw * gcap), gorder(tw * gcap);
        DevBuf<double> gval(tw * gcap);
        if (std::getenv("WBX_VERBOSE"))
            std::fprintf(stderr, "wbx gram: %u columns overflow the shared tables; global pass, %llu-slot tables\n",
                         novf, static_cast<unsigned long long>(gcap));
        gram_kernel<uint32_t><<<g2, kGramWarps * 32, 0, st>>>(novf, d_ovf.p, d_rp.p, d_cl.p, d_vl.p, d_toff.p, d_trow.p, d_tval.p,
                                                    d_m.p, d_m2.p, d_cnt.p, 0, gkey.p, gval.p, gorder.p,
                                                    static_cast<uint32_t>(gcap), d_ovf.p, d_novf.p);
        count_launch(ctx);
        WBX_CUDA(cudaGetLastError());
        WBX_CUDA(cudaStreamSynchronize(st));
    }
    unsigned long long cnt = 0;
    WBX_CUDA(cudaMemcpyAsync(&cnt, d_cnt.p, sizeof cnt, cudaMemcpyDeviceToHost, st));
    WBX_CUDA(cudaMemcpyAsync(diagM, d_m.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    WBX_CUDA(cudaMemcpyAsync(diagM2, d_m2.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    WBX_CUDA(cudaStreamSynchronize(st));
    const uint64_t cap_nnz = cap_factor * std::max<uint64_t>(nnz, 1);
    if (cnt > cap_nnz) fail(WBX_MEMORY_GUARD, "gram_diagonals: nnz(M) exceeds the configured cap");
}

}  // namespace wbx
