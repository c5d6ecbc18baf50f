// Host construction of the per-CTA window layouts (see win.cuh).
#include <algorithm>
#include <array>
#include <cstring>

#include "internal.hpp"
#include "win.cuh"

namespace wbx {

void build_win(WinSide& out, const HostCompact& M, uint32_t G, cudaStream_t st) {
    const uint64_t nrows = M.rows();
    const uint64_t nnz = nrows ? M.ptr[nrows] : 0;
    // contiguous row ranges per CTA balanced by COST = lane segments + nonzeros / 16: a
    // slice's time is dominated by its load round trip, not by its nonzeros, so balancing
    // nonzeros alone leaves the CTAs of short rows with many more slices
    auto cost = [&](uint64_t i) {
        const uint64_t len = M.ptr[i + 1] - M.ptr[i];
        return 16 * std::max<uint64_t>(1, (len + kSegElems - 1) / kSegElems) + len;
    };
    uint64_t total = 0;
    for (uint64_t i = 0; i < nrows; ++i) total += cost(i);
    std::vector<uint64_t> rb(G + 1, nrows);
    rb[0] = 0;
    {
        uint64_t acc = 0, q = 1;
        for (uint64_t i = 0; i < nrows && q < G; ++i) {
            acc += cost(i);
            while (q < G && acc * G >= total * q) rb[q++] = i + 1;
        }
    }
    (void)nnz;
    std::vector<uint32_t> u_off(G + 1, 0), u_idx, s_off(G + 1, 0), s_meta;
    std::vector<uint64_t> s_rec;
    std::vector<uint4> rec;
    uint32_t max_u = 0;
    std::vector<uint32_t> local;  // position -> local window index (scratch)
    for (uint32_t b = 0; b < G; ++b) {
        const uint64_t r0 = rb[b], r1 = rb[b + 1];
        // window: sorted unique referenced positions
        std::vector<uint32_t> u;
        for (uint64_t i = r0; i < r1; ++i)
            for (uint64_t k = M.ptr[i]; k < M.ptr[i + 1]; ++k) u.push_back(M.col[k]);
        std::sort(u.begin(), u.end());
        u.erase(std::unique(u.begin(), u.end()), u.end());
        if (u.size() > 65536) fail(WBX_TOO_LARGE, "CTA window exceeds 16-bit local indices");
        max_u = std::max<uint32_t>(max_u, static_cast<uint32_t>(u.size()));
        u_idx.insert(u_idx.end(), u.begin(), u.end());
        u_off[b + 1] = static_cast<uint32_t>(u_idx.size());
        auto loc = [&](uint32_t pos) {
            return static_cast<uint32_t>(std::lower_bound(u.begin(), u.end(), pos) - u.begin());
        };
        // slices: segment-major placement of rows with equal segment counts
        struct Seg {
            uint64_t row, beg, len;
            uint32_t info;
        };
        uint64_t r = r0;
        while (r < r1) {
            const uint64_t len0 = M.ptr[r + 1] - M.ptr[r];
            const uint64_t q = std::max<uint64_t>(1, (len0 + kSegElems - 1) / kSegElems);
            if (q > 31) fail(WBX_TOO_LARGE, "row longer than 31 segments");
            const uint64_t m = 32 / q;
            std::array<Seg, 32> a;
            for (auto& g : a) g = Seg{0, 0, 0, 0xffffffffu};
            for (uint64_t i = 0; i < m && r < r1; ++i, ++r) {
                const uint64_t len = M.ptr[r + 1] - M.ptr[r];
                if (std::max<uint64_t>(1, (len + kSegElems - 1) / kSegElems) != q) break;
                for (uint64_t t = 0; t < q; ++t) {
                    const uint64_t beg = t * len / q, end = (t + 1) * len / q;
                    a[t * m + i] = Seg{r, beg, end - beg,
                                       t == 0 ? static_cast<uint32_t>(r | (q << kInfoShift)) : 0xffffffffu};
                }
            }
            uint64_t nq = 0;
            for (const auto& g : a) nq = std::max<uint64_t>(nq, (g.len + 3) / 4);
            if (nq == 0) nq = 1;
            s_rec.push_back(rec.size());
            s_meta.push_back(static_cast<uint32_t>(nq) | (static_cast<uint32_t>(m) << 8));
            const uint64_t base = rec.size();
            rec.resize(base + 8 + nq * 32 + nq * 16, make_uint4(0, 0, 0, 0));
            uint32_t* info = reinterpret_cast<uint32_t*>(&rec[base]);
            float* vals = reinterpret_cast<float*>(&rec[base + 8]);
            uint16_t* cols = reinterpret_cast<uint16_t*>(&rec[base + 8 + nq * 32]);
            for (uint64_t lane = 0; lane < 32; ++lane) {
                const Seg& g = a[lane];
                info[lane] = g.info;
                for (uint64_t j = 0; j < g.len; ++j) {
                    const uint64_t k = M.ptr[g.row] + g.beg + j;
                    const uint64_t qd = j / 4, e = j % 4;
                    vals[(qd * 32 + lane) * 4 + e] = static_cast<float>(M.val[k]);
                    cols[(qd * 32 + lane) * 4 + e] = static_cast<uint16_t>(loc(M.col[k]));
                }
            }
        }
        s_off[b + 1] = static_cast<uint32_t>(s_rec.size());
    }
    std::vector<uint32_t> r_off(G + 1);
    uint32_t max_rows = 0;
    for (uint32_t b = 0; b <= G; ++b) {
        r_off[b] = static_cast<uint32_t>(rb[b]);
        if (b < G) max_rows = std::max<uint32_t>(max_rows, static_cast<uint32_t>(rb[b + 1] - rb[b]));
    }
    if (u_idx.empty()) u_idx.push_back(0);
    if (s_rec.empty()) {
        s_rec.push_back(0);
        s_meta.push_back(1);
    }
    if (rec.empty()) rec.resize(1, make_uint4(0, 0, 0, 0));
    out.G = G;
    out.max_u = max_u;
    out.max_rows = max_rows;
    out.r_off.upload(r_off, st);
    out.u_off.upload(u_off, st);
    out.u_idx.upload(u_idx, st);
    out.s_off.upload(s_off, st);
    out.s_rec.upload(s_rec, st);
    out.s_meta.upload(s_meta, st);
    out.rec.upload(rec, st);
    out.bytes = out.r_off.bytes() + out.u_off.bytes() + out.u_idx.bytes() + out.s_off.bytes() + out.s_rec.bytes() + out.s_meta.bytes() +
                out.rec.bytes();
    WBX_CUDA(cudaStreamSynchronize(st));
}

WinView view_of(const WinSide& w) {
    WinView v;
    v.u_off = w.u_off.p;
    v.u_idx = w.u_idx.p;
    v.s_off = w.s_off.p;
    v.s_rec = w.s_rec.p;
    v.s_meta = w.s_meta.p;
    v.r_off = w.r_off.p;
    v.rec = w.rec.p;
    v.max_u = w.max_u;
    v.max_rows = w.max_rows;
    return v;
}

}  // namespace wbx
