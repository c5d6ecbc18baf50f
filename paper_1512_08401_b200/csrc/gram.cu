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
// not fit the table raises a flag and the whole computation falls back to the host.
#include <cstdint>

#include "internal.hpp"

namespace wbx {
namespace {

constexpr int kGramWarps = 4;            // warps per CTA
constexpr uint32_t kGramCap = 2048;      // table slots per warp (power of two)
constexpr uint32_t kEmpty = 0xffffffffu;

struct GramSmem {
    uint32_t key[kGramCap];
    double val[kGramCap];
    uint16_t order[kGramCap];  // first-touch list (slots)
};

__global__ void __launch_bounds__(kGramWarps * 32) gram_kernel(uint64_t n, const uint64_t* __restrict__ rp,
                                                              const uint32_t* __restrict__ cl,
                                                              const double* __restrict__ vl,
                                                              const uint64_t* __restrict__ toff,
                                                              const uint32_t* __restrict__ trow,
                                                              const double* __restrict__ tval, double* diagM,
                                                              double* diagM2, unsigned long long* touched,
                                                              int* overflow) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    GramSmem& S = reinterpret_cast<GramSmem*>(smem_raw)[warp];
    for (uint32_t t = lane; t < kGramCap; t += 32) {
        S.key[t] = kEmpty;
        S.val[t] = 0.0;
    }
    __syncwarp();
    const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kGramWarps + warp;
    const uint64_t nw = static_cast<uint64_t>(gridDim.x) * kGramWarps;
    unsigned long long cnt_total = 0;
    for (uint64_t i = gw; i < n; i += nw) {
        const uint64_t k0 = toff[i], k1 = toff[i + 1];
        if (lane == 0) {  // diag(M): ascending rows, no contraction
            double s = 0.0;
            for (uint64_t k = k0; k < k1; ++k) s = __dadd_rn(s, __dmul_rn(tval[k], tval[k]));
            diagM[i] = s;
        }
        uint32_t nlist = 0;
        bool full = false;
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
                    uint32_t h = (c * 2654435761u) & (kGramCap - 1);
                    for (uint32_t probe = 0;; ++probe) {
                        if (probe == kGramCap) {
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
                        h = (h + 1) & (kGramCap - 1);
                    }
                    slot = h;
                }
                const bool any_full = __any_sync(0xffffffffu, full);
                if (any_full) {
                    full = true;
                    break;
                }
                // first touches appended in lane (= ascending column) order
                const unsigned fm = __ballot_sync(0xffffffffu, act && fresh);
                if (act && fresh) {
                    const uint32_t pos = nlist + __popc(fm & ((1u << lane) - 1u));
                    if (pos < kGramCap) S.order[pos] = static_cast<uint16_t>(slot);
                }
                nlist += __popc(fm);
                if (act) {
                    const double old = S.val[slot];
                    zero_before = old == 0.0;
                    S.val[slot] = __dadd_rn(old, __dmul_rn(a, vl[j]));
                }
                cnt_total += __popc(__ballot_sync(0xffffffffu, act && zero_before));
                __syncwarp();
            }
            if (full) break;
        }
        if (full) {
            if (lane == 0) atomicExch(overflow, 1);
            // reset the whole table (its state is unknown) and carry on; the host recomputes
            for (uint32_t t = lane; t < kGramCap; t += 32) {
                S.key[t] = kEmpty;
                S.val[t] = 0.0;
            }
            __syncwarp();
            continue;
        }
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

bool gram_device(wbx_ctx* ctx, const wbx_op* op, uint64_t cap_factor, double* diagM, double* diagM2) {
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
    DevBuf<int> d_over(1);
    d_rp.upload(rp.data(), n + 1, st);
    d_toff.upload(toff.data(), n + 1, st);
    d_cl.upload(cl.data(), nnz, st);
    d_vl.upload(vl.data(), nnz, st);
    d_trow.upload(trow.data(), nnz, st);
    d_tval.upload(tval.data(), nnz, st);
    WBX_CUDA(cudaMemsetAsync(d_cnt.p, 0, sizeof(unsigned long long), st));
    WBX_CUDA(cudaMemsetAsync(d_over.p, 0, sizeof(int), st));
    const unsigned smem = kGramWarps * sizeof(GramSmem);
    WBX_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(gram_kernel), cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(smem)));
    const unsigned grid = 2u * static_cast<unsigned>(ctx->num_sms);
    gram_kernel<<<grid, kGramWarps * 32, smem, st>>>(n, d_rp.p, d_cl.p, d_vl.p, d_toff.p, d_trow.p, d_tval.p, d_m.p,
                                                     d_m2.p, d_cnt.p, d_over.p);
    count_launch(ctx);
    WBX_CUDA(cudaGetLastError());
    unsigned long long cnt = 0;
    int over = 0;
    WBX_CUDA(cudaMemcpyAsync(&cnt, d_cnt.p, sizeof cnt, cudaMemcpyDeviceToHost, st));
    WBX_CUDA(cudaMemcpyAsync(&over, d_over.p, sizeof over, cudaMemcpyDeviceToHost, st));
    WBX_CUDA(cudaMemcpyAsync(diagM, d_m.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    WBX_CUDA(cudaMemcpyAsync(diagM2, d_m2.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    WBX_CUDA(cudaStreamSynchronize(st));
    if (over) return false;  // a column's 2-hop set exceeded the table: host path
    const uint64_t cap = cap_factor * std::max<uint64_t>(nnz, 1);
    if (cnt > cap) fail(WBX_MEMORY_GUARD, "gram_diagonals: nnz(M) exceeds the configured cap");
    return true;
}

}  // namespace wbx
