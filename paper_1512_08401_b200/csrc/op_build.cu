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
#include <array>
#include <numeric>

#include <cstring>

#include "internal.hpp"
#include "sell.cuh"

namespace wbx {

namespace {

struct HostSell {
    // exact (fp64) layout: one lane per row, element-major, unpadded rows
    std::vector<uint64_t> xslice_ptr;
    std::vector<uint32_t> xslice_len;
    std::vector<double> v64;
    std::vector<uint32_t> col;
    std::vector<uint32_t> row_len;
    // segmented fp32 layout: rows split into <= kSegElems-element segments, one lane per
    // segment, a row's segments in consecutive lanes of one slice
    std::vector<uint64_t> slice_ptr;
    std::vector<uint32_t> slice_np;
    std::vector<uint4> pk;
    std::vector<uint32_t> lane_info;
    std::vector<uint64_t> rec_off;  // uint4 offset of each slice record (+ total)
    std::vector<uint4> rec;
    // row-per-lane fp32 layout over the exact layout's slices
    std::vector<uint2> rslice;
    std::vector<uint4> rpk;
    bool seg_ok = true;
};

// Row-per-lane fp32 layout (wbx_sell::rslice/rpk): slice s = rows 32s..32s+31 (sorted by
// length, so the slice's rows have ~equal length and padding is ~0), element pairs
// {val, col, val, col} element-major [np x 32 lanes], then for an odd slice length the last
// element [32 lanes x {val, col}]. Padding elements (a lane whose row is shorter, or a lane
// past the last row) carry value 0 and the lane's last real column (the gather then hits a
// line the lane already touched).
template <typename RowRange>
void make_row_layout(HostSell& h, uint64_t nrows, RowRange& range) {
    const uint64_t slices = (nrows + 31) / 32;
    h.rslice.assign(slices, make_uint2(0, 0));
    uint64_t off = 0;
    for (uint64_t s = 0; s < slices; ++s) {
        const uint64_t L = h.xslice_len[s];
        if (off > 0xffffffffull) fail(WBX_TOO_LARGE, "operator stream exceeds 32-bit slice offsets");
        h.rslice[s] = make_uint2(static_cast<uint32_t>(off), static_cast<uint32_t>(L));
        off += (L / 2) * 32 + (L & 1) * 16;
    }
    h.rpk.assign(off, make_uint4(0, 0, 0, 0));
    for (uint64_t s = 0; s < slices; ++s) {
        const uint64_t L = h.xslice_len[s], np = L / 2, base = h.rslice[s].x;
        uint2* tail = reinterpret_cast<uint2*>(h.rpk.data() + base + np * 32);
        for (uint64_t lane = 0; lane < 32; ++lane) {
            const uint64_t r = s * 32 + lane;
            const uint64_t len = r < nrows ? range.len(r) : 0;
            uint32_t last = 0;
            for (uint64_t j = 0; j < L; ++j) {
                uint32_t c = last, bits = 0;
                if (j < len) {
                    double v;
                    range.get(r, j, c, v);
                    const float vf = static_cast<float>(v);
                    std::memcpy(&bits, &vf, 4);
                    last = c;
                }
                if (j < 2 * np) {
                    uint4& p = h.rpk[base + (j / 2) * 32 + lane];
                    if (j % 2 == 0) {
                        p.x = bits;
                        p.y = c;
                    } else {
                        p.z = bits;
                        p.w = c;
                    }
                } else {
                    tail[lane] = make_uint2(bits, c);
                }
            }
        }
    }
}

// rows: list of row ids (in slice order); each row r has [beg[r], end[r]) in (cols, vals),
// cols already remapped to the compacted column space.
template <typename RowRange>
HostSell make_sell(uint64_t nrows, RowRange range) {
    HostSell h;
    // ---- exact layout
    const uint64_t slices = (nrows + 31) / 32;
    h.xslice_ptr.assign(slices + 1, 0);
    h.xslice_len.assign(slices, 0);
    h.row_len.assign(nrows, 0);
    for (uint64_t r = 0; r < nrows; ++r) h.row_len[r] = static_cast<uint32_t>(range.len(r));
    for (uint64_t s = 0; s < slices; ++s) {
        uint64_t L = 0;
        for (uint64_t lane = 0; lane < 32; ++lane) {
            const uint64_t r = s * 32 + lane;
            if (r < nrows) L = std::max<uint64_t>(L, range.len(r));
        }
        h.xslice_len[s] = static_cast<uint32_t>(L);
        h.xslice_ptr[s + 1] = h.xslice_ptr[s] + L * 32;
    }
    h.v64.assign(h.xslice_ptr[slices], 0.0);
    h.col.assign(h.xslice_ptr[slices], 0);
    for (uint64_t s = 0; s < slices; ++s)
        for (uint64_t lane = 0; lane < 32; ++lane) {
            const uint64_t r = s * 32 + lane;
            const uint64_t len = r < nrows ? range.len(r) : 0;
            for (uint64_t j = 0; j < len; ++j) {
                const uint64_t e = h.xslice_ptr[s] + j * 32 + lane;
                range.get(r, j, h.col[e], h.v64[e]);
            }
        }
    make_row_layout(h, nrows, range);
    // ---- segmented fp32 layout
    struct Seg {
        uint64_t row, beg, len;
        uint32_t info;
    };
    // Rows longer than 31 segments (496 nonzeros: untruncated operators of the reference's
    // tests) get no fp32 layout; the fp64 entry points run on the exact layout above.
    for (uint64_t r = 0; r < nrows; ++r)
        if (range.len(r) > 31 * kSegElems) {
            h.seg_ok = false;
            h.slice_ptr.assign(1, 0);
            h.rec_off.assign(1, 0);
            return h;
        }
    // Segment-major placement: a slice holds m rows that all have q segments
    // (m = floor(32 / q)); segment t of the slice's i-th row sits in lane t*m + i. Lanes
    // 0..m-1 (and each further group of m) therefore hold consecutive rows, so a warp's
    // gather instruction touches consecutive rows of one band: for a circulant block,
    // consecutive columns — coalesced. Segments split a row evenly.
    std::vector<std::array<Seg, 32>> sl;
    std::vector<uint32_t> stride;
    uint64_t r = 0;
    while (r < nrows) {
        const uint64_t len0 = range.len(r);
        const uint64_t q = std::max<uint64_t>(1, (len0 + kSegElems - 1) / kSegElems);
        if (q > 31) fail(WBX_TOO_LARGE, "row longer than 31 segments");
        const uint64_t m = 32 / q;
        std::array<Seg, 32> a;
        for (auto& g : a) g = Seg{0, 0, 0, 0xffffffffu};
        uint64_t i = 0;
        for (; i < m && r < nrows; ++i, ++r) {
            const uint64_t len = range.len(r);
            const uint64_t qr = std::max<uint64_t>(1, (len + kSegElems - 1) / kSegElems);
            if (qr != q) break;  // next run of rows (rows are sorted by length)
            for (uint64_t t = 0; t < q; ++t) {
                const uint64_t beg = t * len / q, end = (t + 1) * len / q;
                a[t * m + i] = Seg{r, beg, end - beg,
                                   t == 0 ? static_cast<uint32_t>(r | (q << kInfoShift)) : 0xffffffffu};
            }
        }
        sl.push_back(a);
        stride.push_back(static_cast<uint32_t>(m));
    }
    if (nrows >= (1ull << kInfoShift)) fail(WBX_TOO_LARGE, "too many rows for the segment layout");
    const uint64_t ns = sl.size();
    h.slice_ptr.assign(ns + 1, 0);
    h.slice_np.assign(ns, 0);
    h.lane_info.assign(ns * 32, 0xffffffffu);
    for (uint64_t s = 0; s < ns; ++s) {
        uint64_t np = 0;
        for (const auto& g : sl[s]) np = std::max<uint64_t>(np, (g.len + 1) / 2);
        if (np > kSegElems / 2) fail(WBX_TOO_LARGE, "segment longer than kSegElems");
        // slice metadata word: pairs per lane (bits 0-7) | lane stride between segments (8-15)
        h.slice_np[s] = static_cast<uint32_t>(np) | (stride[s] << 8);
        h.slice_ptr[s + 1] = h.slice_ptr[s] + np * 32;
    }
    // slice records for the TMA-staged solver: [lane_info: 32 x u32][pairs: np x 32 x uint4]
    h.rec_off.assign(ns + 1, 0);
    for (uint64_t s = 0; s < ns; ++s) h.rec_off[s + 1] = h.rec_off[s] + 8 + (h.slice_np[s] & 0xffu) * 32;
    h.pk.assign(h.slice_ptr[ns], make_uint4(0, 0, 0, 0));
    for (uint64_t s = 0; s < ns; ++s)
        for (uint64_t lane = 0; lane < 32; ++lane) {
            const Seg& g = sl[s][lane];
            h.lane_info[s * 32 + lane] = g.info;
            for (uint64_t j = 0; j < g.len; ++j) {
                double v;
                uint32_t c;
                range.get(g.row, g.beg + j, c, v);
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
    h.rec.assign(h.rec_off[ns], make_uint4(0, 0, 0, 0));
    for (uint64_t s = 0; s < ns; ++s) {
        uint32_t* info = reinterpret_cast<uint32_t*>(&h.rec[h.rec_off[s]]);
        for (uint64_t lane = 0; lane < 32; ++lane) info[lane] = h.lane_info[s * 32 + lane];
        const uint64_t np = h.slice_np[s] & 0xffu;
        std::copy(h.pk.begin() + static_cast<long>(h.slice_ptr[s]),
                  h.pk.begin() + static_cast<long>(h.slice_ptr[s] + np * 32), h.rec.begin() + static_cast<long>(h.rec_off[s] + 8));
    }
    return h;
}

void upload_sell(wbx_sell& d, const HostSell& h, uint64_t rows, cudaStream_t s, uint64_t& bytes) {
    d.rows = rows;
    d.seg_ok = h.seg_ok;
    d.xslices = h.xslice_len.size();
    d.slices = h.slice_np.size();
    d.pairs = h.pk.size();
    d.xslice_ptr.upload(h.xslice_ptr, s);
    d.xslice_len.upload(h.xslice_len, s);
    d.val64.upload(h.v64, s);
    d.col.upload(h.col, s);
    d.row_len.upload(h.row_len, s);
    d.slice_ptr.upload(h.slice_ptr, s);
    d.slice_np.upload(h.slice_np, s);
    d.pk.upload(h.pk, s);
    d.lane_info.upload(h.lane_info, s);
    d.rec_off.upload(h.rec_off, s);
    d.rec.upload(h.rec, s);
    d.rslice.upload(h.rslice, s);
    d.rpk.upload(h.rpk, s);
    d.rpk_u4 = h.rpk.size();
    bytes += d.rec_off.bytes() + d.rec.bytes() + d.rslice.bytes() + d.rpk.bytes();
    bytes += d.xslice_ptr.bytes() + d.xslice_len.bytes() + d.val64.bytes() + d.col.bytes() +
             d.row_len.bytes() + d.slice_ptr.bytes() + d.slice_np.bytes() + d.pk.bytes() +
             d.lane_info.bytes();
}

}  // namespace

void build_sell(wbx_sell& out, uint64_t nrows, const std::function<uint64_t(uint64_t)>& len,
                const std::function<void(uint64_t, uint64_t, uint32_t&, double&)>& get, cudaStream_t s,
                uint64_t& bytes) {
    struct Range {
        const std::function<uint64_t(uint64_t)>* l;
        const std::function<void(uint64_t, uint64_t, uint32_t&, double&)>* g;
        uint64_t len(uint64_t i) const { return (*l)(i); }
        void get(uint64_t i, uint64_t j, uint32_t& c, double& v) const { (*g)(i, j, c, v); }
    } r{&len, &get};
    HostSell h = make_sell(nrows, r);
    if (!h.seg_ok) fail(WBX_TOO_LARGE, "row longer than 31 segments");
    upload_sell(out, h, nrows, s, bytes);
    WBX_CUDA(cudaStreamSynchronize(s));
}

SellView view_of(const wbx_sell& m) {
    SellView v;
    v.xslice_ptr = m.xslice_ptr.p;
    v.xslice_len = m.xslice_len.p;
    v.v64 = m.val64.p;
    v.col = m.col.p;
    v.row_len = m.row_len.p;
    v.slice_ptr = m.slice_ptr.p;
    v.slice_np = m.slice_np.p;
    v.pk = m.pk.p;
    v.lane_info = m.lane_info.p;
    v.rec = m.rec.p;
    v.rec_off = m.rec_off.p;
    v.rslice = m.rslice.p;
    v.rpk = m.rpk.p;
    v.rpk_u4 = m.rpk_u4;
    v.rows = static_cast<uint32_t>(m.rows);
    v.xslices = static_cast<uint32_t>(m.xslices);
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

    // compacted host forms (rows in sorted order, columns as positions) for the per-block
    // window layouts built at solver setup (winlayout.cu)
    auto compact = [](HostCompact& hc, uint64_t nrows, auto& range) {
        hc.ptr.assign(nrows + 1, 0);
        for (uint64_t i = 0; i < nrows; ++i) hc.ptr[i + 1] = hc.ptr[i] + range.len(i);
        hc.col.resize(hc.ptr[nrows]);
        hc.val.resize(hc.ptr[nrows]);
        for (uint64_t i = 0; i < nrows; ++i)
            for (uint64_t j = 0; j < range.len(i); ++j) range.get(i, j, hc.col[hc.ptr[i] + j], hc.val[hc.ptr[i] + j]);
    };
    compact(op->hA, R.size(), ar);
    compact(op->hT, C.size(), tr);
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
