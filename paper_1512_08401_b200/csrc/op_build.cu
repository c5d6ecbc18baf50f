// Host-side construction of the device layouts of Theta_K.
//
// Input: the reference's CSR SparseOperator (theta.hpp:50-60: u64 row offsets, u32
// strictly increasing columns, f64 values). Output (wbx_op):
//   * R = nonempty rows, C = nonempty columns. At 1024^2, db4 J=4, K=3N only 14.8 % of
//     rows and 4.7 % of columns are nonempty; every vector the solver
//     streams is COMPACTED to these sets, so per-iteration traffic is the nonzeros plus
//     |R| + |C| entries instead of n.
//   * A = Theta restricted to R x C as SELL-32 (slices of 32 rows, one lane per row,
//     element j of the slice's rows stored contiguously so a warp load is coalesced).
//     Rows are sorted by descending length (stable), which makes padding ~0 and hands
//     the longest slices out first. Within a row, elements keep the reference's order
//     (ascending column), so a lane's sequential sum has the reference's order
//     (theta.cpp:306-308).
//   * T = Theta^T restricted to C x R, built like make_transpose (theta.cpp:324-340):
//     within a row of T, ascending original row — the order spmv on the cached
//     transpose sums in (solver.cpp:15-17).
//   * fp32 values packed with their column as {val0, col0, val1, col1} (one 16-byte
//     load per two nonzeros per lane); fp64 values + u32 columns element-major.
#include <algorithm>
#include <numeric>

#include <cstring>

#include "internal.hpp"
#include "sell.cuh"

namespace wbx {

namespace {

struct HostSell {
    std::vector<uint64_t> slice_ptr;
    std::vector<uint32_t> slice_len;
    std::vector<uint4> pk;
    std::vector<double> v64;
    std::vector<uint32_t> col;
    std::vector<uint32_t> row_len;
};

// rows: list of row ids (in slice order); each row r has [beg[r], end[r]) in (cols, vals),
// cols already remapped to the compacted column space.
template <typename RowRange>
HostSell make_sell(uint64_t nrows, RowRange range) {
    HostSell h;
    const uint64_t slices = (nrows + 31) / 32;
    h.slice_ptr.assign(slices + 1, 0);
    h.slice_len.assign(slices, 0);
    h.row_len.assign(nrows, 0);
    for (uint64_t r = 0; r < nrows; ++r) h.row_len[r] = static_cast<uint32_t>(range.len(r));
    for (uint64_t s = 0; s < slices; ++s) {
        uint64_t L = 0;
        for (uint64_t lane = 0; lane < 32; ++lane) {
            const uint64_t r = s * 32 + lane;
            if (r < nrows) L = std::max<uint64_t>(L, range.len(r));
        }
        L = (L + 1) & ~uint64_t{1};
        h.slice_len[s] = static_cast<uint32_t>(L);
        h.slice_ptr[s + 1] = h.slice_ptr[s] + (L / 2) * 32;
    }
    const uint64_t pairs = h.slice_ptr[slices];
    h.pk.assign(pairs, make_uint4(0, 0, 0, 0));
    h.v64.assign(2 * pairs, 0.0);
    h.col.assign(2 * pairs, 0);
    for (uint64_t s = 0; s < slices; ++s) {
        const uint64_t L = h.slice_len[s];
        for (uint64_t lane = 0; lane < 32; ++lane) {
            const uint64_t r = s * 32 + lane;
            const uint64_t len = r < nrows ? range.len(r) : 0;
            for (uint64_t j = 0; j < L; ++j) {
                double v = 0.0;
                uint32_t c = 0;
                if (j < len) range.get(r, j, c, v);
                const uint64_t e = 2 * h.slice_ptr[s] + j * 32 + lane;
                h.v64[e] = v;
                h.col[e] = c;
                uint4& p = h.pk[h.slice_ptr[s] + (j / 2) * 32 + lane];
                const float vf = static_cast<float>(v);
                uint32_t bits;
                std::memcpy(&bits, &vf, 4);
                if (j % 2 == 0) {
                    p.x = bits;
                    p.y = c;
                } else {
                    p.z = bits;
                    p.w = c;
                }
            }
        }
    }
    return h;
}

void upload_sell(wbx_sell& d, const HostSell& h, uint64_t rows, cudaStream_t s, uint64_t& bytes) {
    d.rows = rows;
    d.slices = h.slice_len.size();
    d.pairs = h.pk.size();
    d.slice_ptr.upload(h.slice_ptr, s);
    d.slice_len.upload(h.slice_len, s);
    d.pk.upload(h.pk, s);
    d.val64.upload(h.v64, s);
    d.col.upload(h.col, s);
    d.row_len.upload(h.row_len, s);
    bytes += d.row_len.bytes() + d.slice_ptr.bytes() + d.slice_len.bytes() + d.pk.bytes() + d.val64.bytes() + d.col.bytes();
}

}  // namespace

SellView view_of(const wbx_sell& m) {
    SellView v;
    v.slice_ptr = m.slice_ptr.p;
    v.slice_len = m.slice_len.p;
    v.pk = m.pk.p;
    v.v64 = m.val64.p;
    v.col = m.col.p;
    v.row_len = m.row_len.p;
    v.rows = static_cast<uint32_t>(m.rows);
    v.slices = static_cast<uint32_t>(m.slices);
    return v;
}

void build_op(wbx_op* op, uint64_t n, const uint64_t* rowptr, const uint32_t* col,
              const double* val) {
    if (n == 0) fail(WBX_SHAPE_MISMATCH, "operator dimension must be positive");
    if (n > 0xffffffffull) fail(WBX_TOO_LARGE, "operator dimension exceeds 32-bit indices");
    if (rowptr == nullptr || (rowptr[n] > 0 && (col == nullptr || val == nullptr)))
        fail(WBX_INVALID_ARGUMENT, "null CSR array");
    // validation as read_operator (theta.cpp:479-488)
    if (rowptr[0] != 0) fail(WBX_SHAPE_MISMATCH, "inconsistent row offsets");
    const uint64_t nnz = rowptr[n];
    for (uint64_t r = 0; r < n; ++r) {
        if (rowptr[r] > rowptr[r + 1]) fail(WBX_SHAPE_MISMATCH, "row offsets not nondecreasing");
        for (uint64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) {
            if (col[k] >= n) fail(WBX_SHAPE_MISMATCH, "column index out of range");
            if (k > rowptr[r] && col[k] <= col[k - 1])
                fail(WBX_SHAPE_MISMATCH, "columns not strictly increasing in a row");
        }
    }
    op->n = n;
    op->nnz = nnz;
    op->h_rowptr.assign(rowptr, rowptr + n + 1);
    op->h_col.assign(col, col + nnz);
    op->h_val.assign(val, val + nnz);

    // transpose (make_transpose order: within a column, ascending row)
    std::vector<uint64_t> toff(n + 1, 0);
    for (uint64_t k = 0; k < nnz; ++k) ++toff[col[k] + 1];
    for (uint64_t i = 0; i < n; ++i) toff[i + 1] += toff[i];
    std::vector<uint32_t> trow(nnz);
    std::vector<double> tval(nnz);
    {
        std::vector<uint64_t> cur(toff.begin(), toff.end() - 1);
        for (uint64_t r = 0; r < n; ++r)
            for (uint64_t k = rowptr[r]; k < rowptr[r + 1]; ++k) {
                const uint64_t pos = cur[col[k]]++;
                trow[pos] = static_cast<uint32_t>(r);
                tval[pos] = val[k];
            }
    }

    // R and C, sorted by descending length (stable on index)
    std::vector<uint32_t> R, C;
    for (uint64_t r = 0; r < n; ++r)
        if (rowptr[r + 1] > rowptr[r]) R.push_back(static_cast<uint32_t>(r));
    for (uint64_t c = 0; c < n; ++c)
        if (toff[c + 1] > toff[c]) C.push_back(static_cast<uint32_t>(c));
    std::stable_sort(R.begin(), R.end(), [&](uint32_t a, uint32_t b) {
        return rowptr[a + 1] - rowptr[a] > rowptr[b + 1] - rowptr[b];
    });
    std::stable_sort(C.begin(), C.end(), [&](uint32_t a, uint32_t b) {
        return toff[a + 1] - toff[a] > toff[b + 1] - toff[b];
    });
    std::vector<uint32_t> rpos(n, 0xffffffffu), cpos(n, 0xffffffffu);
    for (uint64_t i = 0; i < R.size(); ++i) rpos[R[i]] = static_cast<uint32_t>(i);
    for (uint64_t i = 0; i < C.size(); ++i) cpos[C[i]] = static_cast<uint32_t>(i);
    op->nR = R.size();
    op->nC = C.size();

    struct ARange {
        const uint64_t* rp;
        const uint32_t* cl;
        const double* vl;
        const std::vector<uint32_t>* R;
        const std::vector<uint32_t>* cpos;
        uint64_t len(uint64_t i) const { return rp[(*R)[i] + 1] - rp[(*R)[i]]; }
        void get(uint64_t i, uint64_t j, uint32_t& c, double& v) const {
            const uint64_t k = rp[(*R)[i]] + j;
            c = (*cpos)[cl[k]];
            v = vl[k];
        }
    } ar{rowptr, col, val, &R, &cpos};
    struct TRange {
        const uint64_t* tp;
        const uint32_t* tr;
        const double* tv;
        const std::vector<uint32_t>* C;
        const std::vector<uint32_t>* rpos;
        uint64_t len(uint64_t i) const { return tp[(*C)[i] + 1] - tp[(*C)[i]]; }
        void get(uint64_t i, uint64_t j, uint32_t& c, double& v) const {
            const uint64_t k = tp[(*C)[i]] + j;
            c = (*rpos)[tr[k]];
            v = tv[k];
        }
    } tr{toff.data(), trow.data(), tval.data(), &C, &rpos};

    HostSell ha = make_sell(R.size(), ar);
    HostSell ht = make_sell(C.size(), tr);
    cudaStream_t s = op->ctx->stream;
    uint64_t bytes = 0;
    upload_sell(op->A, ha, R.size(), s, bytes);
    upload_sell(op->T, ht, C.size(), s, bytes);
    op->h_R_glob = R;
    op->h_C_glob = C;
    op->R_glob.upload(R, s);
    op->C_glob.upload(C, s);
    std::vector<uint32_t> mask((n + 31) / 32, 0);
    for (uint32_t c : C) mask[c / 32] |= 1u << (c % 32);
    op->isC.upload(mask, s);
    std::vector<uint32_t> rmask((n + 31) / 32, 0);
    for (uint32_t r : R) rmask[r / 32] |= 1u << (r % 32);
    op->isR.upload(rmask, s);
    bytes += op->R_glob.bytes() + op->C_glob.bytes() + op->isC.bytes() + op->isR.bytes();
    op->device_bytes = bytes;
    WBX_CUDA(cudaStreamSynchronize(s));  // host staging vectors die here
}

}  // namespace wbx
