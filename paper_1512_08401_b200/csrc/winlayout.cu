// Host construction of the per-CTA window layouts (see win.cuh).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>

#include "internal.hpp"
#include "win.cuh"

namespace wbx {

namespace {

uint64_t segs_of(uint64_t len) { return std::max<uint64_t>(1, (len + kSegElems - 1) / kSegElems); }

// Contiguous row ranges per CTA balanced by a per-row COST. Default: round 1's cost
// 8*q + len (q = segments, len = nonzeros). WBX_WIN_MODEL[_A|_T] = "a,b,c,d,e" selects the
// model fitted by least squares to per-CTA phase times (WBX_TRACE_FILE, tools/win_fit.py):
//   cost(row) = (a + b*nq + c*(q - 1)) / m + d*len + e
// with q = segments of the row, m = floor(32/q) rows per slice, nq = quads per lane (the slice
// chain: record loads, nq gathers + fmas per lane, q - 1 shuffle folds), len = nonzeros (window
// growth, epilogue); it evens the per-CTA times (C2 spread 1.7 -> 0.8 us) but measured no
// faster end to end. WBX_WIN_COST[_A|_T] = "wseg,wnnz" sets round 1's weights.
std::vector<uint64_t> balance(const HostCompact& M, uint32_t G, char side) {
    const uint64_t nrows = M.rows();
    double cm[5] = {0, 0, 0, 0, 0};
    bool model = false;
    uint64_t wseg = 8, wnnz = 1;  // round 1 (tools/cost_sweep.sh): best of 4..12 per side at C2
    {
        const std::string key = std::string("WBX_WIN_MODEL_") + side;
        const char* e = std::getenv(key.c_str());
        if (!e) e = std::getenv("WBX_WIN_MODEL");
        if (e && std::sscanf(e, "%lf,%lf,%lf,%lf,%lf", &cm[0], &cm[1], &cm[2], &cm[3], &cm[4]) == 5) model = true;
    }
    const std::string key = std::string("WBX_WIN_COST_") + side;  // per side, then both sides
    const char* e = std::getenv(key.c_str());
    if (!e) e = std::getenv("WBX_WIN_COST");
    if (e && !model) {  // diagnostics: "segment_weight,nonzero_weight"
        unsigned long long a = 0, b = 0;
        if (std::sscanf(e, "%llu,%llu", &a, &b) == 2) {
            wseg = a;
            wnnz = b;
        }
    }
    std::vector<double> cost(nrows);
    for (uint64_t i = 0; i < nrows; ++i) {
        const uint64_t len = M.ptr[i + 1] - M.ptr[i];
        const uint64_t q = segs_of(len);
        if (model) {
            const double m = static_cast<double>(32 / q);
            const double nq = static_cast<double>((len + q - 1) / q + 3) / 4.0;
            cost[i] = (cm[0] + cm[1] * nq + cm[2] * static_cast<double>(q - 1)) / m + cm[3] * static_cast<double>(len) +
                      cm[4];
        } else {
            cost[i] = static_cast<double>(wseg * q + wnnz * len);
        }
    }
    double total = 0.0;
    for (uint64_t i = 0; i < nrows; ++i) total += cost[i];
    std::vector<uint64_t> rb(G + 1, nrows);
    rb[0] = 0;
    double acc = 0.0;
    uint64_t q = 1;
    for (uint64_t i = 0; i < nrows && q < G; ++i) {
        acc += cost[i];
        while (q < G && acc * G >= total * static_cast<double>(q)) rb[q++] = i + 1;
    }
    return rb;
}

// Per-CTA dictionary of distinct fp32 value sequences: offset (floats) of every row's
// q x 16 block, or false when the dictionary exceeds the budget.
bool build_dict(const HostCompact& M, uint64_t r0, uint64_t r1, std::vector<float>& dict,
                std::vector<uint32_t>& row_off) {
    dict.assign(16, 0.0f);  // offset 0: the zero block of padding lanes
    row_off.assign(r1 - r0, 0);
    std::map<std::vector<uint32_t>, uint32_t> seen;
    for (uint64_t r = r0; r < r1; ++r) {
        const uint64_t len = M.ptr[r + 1] - M.ptr[r];
        std::vector<uint32_t> key(len);
        for (uint64_t k = 0; k < len; ++k) {
            const float f = static_cast<float>(M.val[M.ptr[r] + k]);
            std::memcpy(&key[k], &f, 4);
        }
        auto it = seen.find(key);
        if (it == seen.end()) {
            const uint64_t q = segs_of(len);
            const uint32_t off = static_cast<uint32_t>(dict.size());
            dict.resize(dict.size() + q * 16, 0.0f);
            for (uint64_t t = 0; t < q; ++t) {
                const uint64_t beg = t * len / q, end = (t + 1) * len / q;
                for (uint64_t j = beg; j < end; ++j) std::memcpy(&dict[off + t * 16 + (j - beg)], &key[j], 4);
            }
            if (dict.size() * 4 > kWinDictBudget) return false;
            it = seen.emplace(std::move(key), off).first;
        }
        row_off[r - r0] = it->second;
    }
    return true;
}

// Greedy bank assignment of one CTA's window (nu entries, ranks 0..nu-1) from the gather
// groups of its slices (slices slice0.. in s_tab/rec, columns as ranks): larger groups
// first; each unplaced member goes to the bank least used by the group so far (ties: the
// least filled bank). slot = bank + 32 * (fill of that bank). Returns rank -> slot; updates
// *max_win with the window's slot extent. WBX_WIN_PLACE=sorted keeps slot = rank.
std::vector<uint16_t> place_window(const std::vector<uint4>& rec, const std::vector<uint4>& s_tab, size_t slice0,
                                   bool dict_fmt, size_t nu, uint32_t* max_win) {
    std::vector<uint16_t> slot(nu);
    const char* mode = std::getenv("WBX_WIN_PLACE");
    if (mode && std::string(mode) == "sorted") {  // diagnostics: source order
        for (size_t i = 0; i < nu; ++i) slot[i] = static_cast<uint16_t>(i);
        *max_win = std::max<uint32_t>(*max_win, static_cast<uint32_t>(nu));
        return slot;
    }
    constexpr int kBanks = 32;
    std::vector<std::vector<uint16_t>> groups;
    for (size_t sidx = slice0; sidx < s_tab.size(); ++sidx) {
        const uint32_t nq = s_tab[sidx].y & 0xffu;
        const uint16_t* cols = reinterpret_cast<const uint16_t*>(&rec[s_tab[sidx].x + (dict_fmt ? 4 : nq * 32)]);
        for (uint32_t qd = 0; qd < nq; ++qd)
            for (uint32_t e = 0; e < 4; ++e) {
                std::vector<uint16_t> g;
                for (uint32_t lane = 0; lane < 32; ++lane) g.push_back(cols[(qd * 32 + lane) * 4 + e]);
                std::sort(g.begin(), g.end());
                g.erase(std::unique(g.begin(), g.end()), g.end());
                if (g.size() > 1) groups.push_back(std::move(g));
            }
    }
    std::stable_sort(groups.begin(), groups.end(),
                     [](const std::vector<uint16_t>& x, const std::vector<uint16_t>& y) { return x.size() > y.size(); });
    std::vector<int> bank(nu, -1);
    std::vector<uint32_t> fill(kBanks, 0);
    for (const auto& g : groups) {
        int used[kBanks] = {0};
        for (uint16_t e : g)
            if (bank[e] >= 0) ++used[bank[e]];
        for (uint16_t e : g) {
            if (bank[e] >= 0) continue;
            int best = 0;
            for (int k = 1; k < kBanks; ++k)
                if (used[k] < used[best] || (used[k] == used[best] && fill[k] < fill[best])) best = k;
            bank[e] = best;
            ++used[best];
            ++fill[best];
        }
    }
    for (size_t i = 0; i < nu; ++i)  // entries no group constrains (only in 1-distinct groups)
        if (bank[i] < 0) {
            int best = 0;
            for (int k = 1; k < kBanks; ++k)
                if (fill[k] < fill[best]) best = k;
            bank[i] = best;
            ++fill[best];
        }
    std::vector<uint32_t> next(kBanks, 0);
    uint32_t extent = 0;
    for (size_t i = 0; i < nu; ++i) {
        const uint32_t sl = static_cast<uint32_t>(bank[i]) + kBanks * next[bank[i]]++;
        if (sl > 0xffffu) fail(WBX_TOO_LARGE, "CTA window exceeds 16-bit slots");
        slot[i] = static_cast<uint16_t>(sl);
        extent = std::max(extent, sl + 1);
    }
    *max_win = std::max(*max_win, extent);
    return slot;
}

}  // namespace

// Rotations of the chunks inside each 128-byte line of the (source-order) chunk layout: a
// rotation keeps a line's chunks in that line (the fill still reads and writes contiguous
// 512 B per warp) but moves its entries to other banks. Greedy per line (most-read lines
// first): the rotation whose entries collide least with the entries already placed in the
// gather groups (one gather instruction's 32 lanes) that read them.
std::vector<uint32_t> line_rotations(const std::vector<uint4>& rec, const std::vector<uint4>& s_tab, size_t slice0,
                                     bool dict_fmt, const std::vector<uint32_t>& u,
                                     const std::vector<uint32_t>& chunk_of, size_t nc) {
    const size_t nl = (nc + 7) / 8;
    std::vector<std::vector<uint32_t>> groups_of(u.size());  // rank -> gather groups reading it
    uint32_t ng = 0;
    for (size_t sidx = slice0; sidx < s_tab.size(); ++sidx) {
        const uint32_t nq = s_tab[sidx].y & 0xffu;
        const uint16_t* cols = reinterpret_cast<const uint16_t*>(&rec[s_tab[sidx].x + (dict_fmt ? 4 : nq * 32)]);
        for (uint32_t qd = 0; qd < nq; ++qd)
            for (uint32_t e = 0; e < 4; ++e) {
                std::vector<uint16_t> g;
                for (uint32_t lane = 0; lane < 32; ++lane) g.push_back(cols[(qd * 32 + lane) * 4 + e]);
                std::sort(g.begin(), g.end());
                g.erase(std::unique(g.begin(), g.end()), g.end());
                if (g.size() < 2) continue;
                for (uint16_t r : g) groups_of[r].push_back(ng);
                ++ng;
            }
    }
    std::vector<std::vector<uint32_t>> ranks_of_line(nl);
    std::vector<uint32_t> reads(nl, 0);
    for (size_t r = 0; r < u.size(); ++r) {
        ranks_of_line[chunk_of[r] >> 3].push_back(static_cast<uint32_t>(r));
        reads[chunk_of[r] >> 3] += static_cast<uint32_t>(groups_of[r].size());
    }
    std::vector<uint32_t> order(nl);
    for (uint32_t i = 0; i < nl; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return reads[a] > reads[b]; });
    std::vector<uint8_t> used(static_cast<size_t>(ng) * 32, 0);
    std::vector<uint32_t> rot(nl, 0);
    for (uint32_t L : order) {
        uint32_t best = 0, best_cost = UINT32_MAX;
        for (uint32_t r = 0; r < 8; ++r) {
            uint32_t cost = 0;
            for (uint32_t rk : ranks_of_line[L]) {
                const uint32_t bank = 4 * ((chunk_of[rk] + r) & 7u) + (u[rk] & 3u);
                for (uint32_t g : groups_of[rk]) cost += used[static_cast<size_t>(g) * 32 + bank];
            }
            if (cost < best_cost) {
                best_cost = cost;
                best = r;
            }
        }
        rot[L] = best;
        for (uint32_t rk : ranks_of_line[L]) {
            const uint32_t bank = 4 * ((chunk_of[rk] + best) & 7u) + (u[rk] & 3u);
            for (uint32_t g : groups_of[rk]) {
                uint8_t& c = used[static_cast<size_t>(g) * 32 + bank];
                if (c < 255) ++c;
            }
        }
    }
    return rot;
}

// Chunk layout placement: window chunk c (4 consecutive source floats) goes to chunk slot
// cs[c], its floats to window 4 cs[c] .. 4 cs[c] + 3, so entry u sits in bank
// 4 (cs[c] mod 8) + (u mod 4). Default: cs[c] = c (source order). WBX_WIN_PLACE=chunk-bank
// chooses the bank group cs mod 8 of each chunk greedily, as place_window does per entry, so
// that the entries one gather instruction reads spread over the banks.
// `rank_slot` receives each window entry's float slot (entries in rank order of u).
std::vector<uint16_t> place_chunks(const std::vector<uint4>& rec, const std::vector<uint4>& s_tab, size_t slice0,
                                   bool dict_fmt, const std::vector<uint32_t>& u, const std::vector<uint32_t>& chunks,
                                   std::vector<uint16_t>& rank_slot, uint32_t* max_win) {
    constexpr int kGroups = 8;
    const size_t nc = chunks.size();
    std::vector<uint32_t> chunk_of(u.size());  // rank -> chunk ordinal
    for (size_t i = 0, c = 0; i < u.size(); ++i) {
        while (chunks[c] != u[i] >> 2) ++c;
        chunk_of[i] = static_cast<uint32_t>(c);
    }
    std::vector<int> bg(nc, -1);
    std::vector<uint32_t> fill(kGroups, 0);
    // default: chunks in source order, rotated inside their 128-byte lines (a warp's fill reads
    // and writes contiguous 512 B); WBX_WIN_PLACE=chunk-plain: no rotation; =chunk-bank: chunk
    // slots chosen per chunk (gathers conflict less, but the fills touch scattered lines: C2
    // 2.20 vs 2.13-2.16 ms per deblur for plain)
    const char* mode = std::getenv("WBX_WIN_PLACE");
    const bool plain = !(mode && std::string(mode) == "chunk-bank");
    if (!plain) {
        std::vector<std::vector<uint16_t>> groups;  // ranks one gather reads
        for (size_t sidx = slice0; sidx < s_tab.size(); ++sidx) {
            const uint32_t nq = s_tab[sidx].y & 0xffu;
            const uint16_t* cols = reinterpret_cast<const uint16_t*>(&rec[s_tab[sidx].x + (dict_fmt ? 4 : nq * 32)]);
            for (uint32_t qd = 0; qd < nq; ++qd)
                for (uint32_t e = 0; e < 4; ++e) {
                    std::vector<uint16_t> g;
                    for (uint32_t lane = 0; lane < 32; ++lane) g.push_back(cols[(qd * 32 + lane) * 4 + e]);
                    std::sort(g.begin(), g.end());
                    g.erase(std::unique(g.begin(), g.end()), g.end());
                    if (g.size() > 1) groups.push_back(std::move(g));
                }
        }
        std::stable_sort(groups.begin(), groups.end(),
                         [](const std::vector<uint16_t>& x, const std::vector<uint16_t>& y) { return x.size() > y.size(); });
        for (const auto& g : groups) {
            int used[32] = {0};
            for (uint16_t r : g)
                if (bg[chunk_of[r]] >= 0) ++used[4 * bg[chunk_of[r]] + (u[r] & 3u)];
            for (uint16_t r : g) {
                const uint32_t c = chunk_of[r];
                if (bg[c] >= 0) continue;
                int best = 0;
                for (int k = 1; k < kGroups; ++k) {
                    const int uk = used[4 * k + (u[r] & 3u)], ub = used[4 * best + (u[r] & 3u)];
                    if (uk < ub || (uk == ub && fill[k] < fill[best])) best = k;
                }
                bg[c] = best;
                ++fill[best];
                // the chunk's other entries of this group now occupy their banks too
                for (uint16_t r2 : g)
                    if (chunk_of[r2] == c) ++used[4 * best + (u[r2] & 3u)];
            }
        }
    }
    for (size_t c = 0; c < nc; ++c)
        if (bg[c] < 0) {
            int best = 0;
            for (int k = 1; k < kGroups; ++k)
                if (fill[k] < fill[best]) best = k;
            bg[c] = plain ? static_cast<int>(c % kGroups) : best;
            if (!plain) ++fill[best];
        }
    std::vector<uint16_t> cslot(nc);
    std::vector<uint32_t> next(kGroups, 0);
    uint32_t extent = 0;
    std::vector<uint32_t> rot;  // default: per 128-byte line of 8 chunks, a rotation of its chunks
    if (plain && !(mode && std::string(mode) == "chunk-plain")) rot = line_rotations(rec, s_tab, slice0, dict_fmt, u, chunk_of, nc);
    for (size_t c = 0; c < nc; ++c) {
        uint32_t sl = plain ? static_cast<uint32_t>(c) : static_cast<uint32_t>(bg[c]) + kGroups * next[bg[c]]++;
        if (!rot.empty()) sl = (sl & ~7u) | ((sl + rot[sl >> 3]) & 7u);
        if (4 * sl + 3 > 0xffffu) fail(WBX_TOO_LARGE, "CTA window exceeds 16-bit slots");
        cslot[c] = static_cast<uint16_t>(sl);
        extent = std::max(extent, 4 * sl + 4);
    }
    rank_slot.resize(u.size());
    for (size_t i = 0; i < u.size(); ++i) rank_slot[i] = static_cast<uint16_t>(4 * cslot[chunk_of[i]] + (u[i] & 3u));
    *max_win = std::max(*max_win, extent);
    return cslot;
}

void build_win(WinSide& out, const HostCompact& M, uint32_t G, cudaStream_t st, char side, bool chunk) {
    const std::vector<uint64_t> rb = balance(M, G, side);
    // format: the dictionary when every CTA's fits the budget
    bool dict_fmt = std::getenv("WBX_WIN_FULL") == nullptr;  // diagnostics: force the full format
    std::vector<std::vector<float>> dicts(G);
    std::vector<std::vector<uint32_t>> roffs(G);
    for (uint32_t b = 0; b < G && dict_fmt; ++b) dict_fmt = build_dict(M, rb[b], rb[b + 1], dicts[b], roffs[b]);

    std::vector<uint32_t> u_off(G + 1, 0), u_idx, s_off(G + 1, 0), d_off(G + 1, 0);
    std::vector<uint4> s_tab, rec;
    std::vector<float> d_val;
    uint32_t max_u = 0, max_slices = 0, max_dict = 0, max_win = 0;
    std::vector<uint16_t> u_slot;
    for (uint32_t b = 0; b < G; ++b) {
        const uint64_t r0 = rb[b], r1 = rb[b + 1];
        // window: sorted unique referenced positions
        std::vector<uint32_t> u;
        for (uint64_t i = r0; i < r1; ++i)
            for (uint64_t k = M.ptr[i]; k < M.ptr[i + 1]; ++k) u.push_back(M.col[k]);
        std::sort(u.begin(), u.end());
        u.erase(std::unique(u.begin(), u.end()), u.end());
        if (u.size() > 65536) fail(WBX_TOO_LARGE, "CTA window exceeds 16-bit local indices");
        std::vector<uint32_t> chunks;  // chunk layout: the 16-byte source chunks the window covers
        if (chunk) {
            for (uint32_t v : u)
                if (chunks.empty() || chunks.back() != v >> 2) chunks.push_back(v >> 2);
            if (chunks.size() * 4 > 65536) fail(WBX_TOO_LARGE, "CTA window exceeds 16-bit slots");
            max_u = std::max<uint32_t>(max_u, static_cast<uint32_t>(chunks.size()));
            u_idx.insert(u_idx.end(), chunks.begin(), chunks.end());
        } else {
            max_u = std::max<uint32_t>(max_u, static_cast<uint32_t>(u.size()));
            u_idx.insert(u_idx.end(), u.begin(), u.end());
        }
        u_off[b + 1] = static_cast<uint32_t>(u_idx.size());
        auto loc = [&](uint32_t pos) {
            return static_cast<uint16_t>(std::lower_bound(u.begin(), u.end(), pos) - u.begin());
        };
        if (dict_fmt) {
            d_val.insert(d_val.end(), dicts[b].begin(), dicts[b].end());
            max_dict = std::max<uint32_t>(max_dict, static_cast<uint32_t>(dicts[b].size()));
        }
        d_off[b + 1] = static_cast<uint32_t>(d_val.size());
        // slices: up to m consecutive rows with equal segment count q, segment-major lanes
        const size_t slice0 = s_tab.size();
        uint64_t r = r0;
        while (r < r1) {
            const uint64_t q = segs_of(M.ptr[r + 1] - M.ptr[r]);
            if (q > 31) fail(WBX_TOO_LARGE, "row longer than 31 segments");
            const uint64_t m = 32 / q, first = r;
            uint64_t cnt = 0;
            while (cnt < m && r < r1 && segs_of(M.ptr[r + 1] - M.ptr[r]) == q) {
                ++cnt;
                ++r;
            }
            uint64_t nq = 1;
            for (uint64_t i = 0; i < cnt; ++i) {
                const uint64_t len = M.ptr[first + i + 1] - M.ptr[first + i];
                for (uint64_t t = 0; t < q; ++t) nq = std::max<uint64_t>(nq, ((t + 1) * len / q - t * len / q + 3) / 4);
            }
            const uint64_t base = rec.size();
            const uint64_t head = dict_fmt ? 4 : nq * 32;  // pb words, or values
            rec.resize(base + head + nq * 16, make_uint4(0, 0, 0, 0));
            uint16_t* pb = reinterpret_cast<uint16_t*>(&rec[base]);
            float* vals = reinterpret_cast<float*>(&rec[base]);
            uint16_t* cols = reinterpret_cast<uint16_t*>(&rec[base + head]);
            for (uint64_t i = 0; i < cnt; ++i) {
                const uint64_t row = first + i, len = M.ptr[row + 1] - M.ptr[row];
                for (uint64_t t = 0; t < q; ++t) {
                    const uint64_t lane = t * m + i, beg = t * len / q, end = (t + 1) * len / q;
                    if (dict_fmt) {
                        const uint32_t o = roffs[b][row - r0] + static_cast<uint32_t>(t * 16);
                        if (o > 0xffffu) fail(WBX_TOO_LARGE, "dictionary offset exceeds 16 bits");
                        pb[lane] = static_cast<uint16_t>(o);
                    }
                    for (uint64_t j = 0; j < end - beg; ++j) {
                        const uint64_t k = M.ptr[row] + beg + j;
                        const uint64_t slot = ((j / 4) * 32 + lane) * 4 + j % 4;
                        if (!dict_fmt) vals[slot] = static_cast<float>(M.val[k]);
                        cols[slot] = loc(M.col[k]);
                    }
                }
            }
            if (base > 0xffffffffull) fail(WBX_TOO_LARGE, "window records exceed 32-bit offsets");
            s_tab.push_back(make_uint4(static_cast<uint32_t>(base),
                                       win_meta(static_cast<uint32_t>(nq), static_cast<uint32_t>(m),
                                                static_cast<uint32_t>(q), static_cast<uint32_t>(cnt)),
                                       static_cast<uint32_t>(first), 0));
        }
        s_off[b + 1] = static_cast<uint32_t>(s_tab.size());
        max_slices = std::max<uint32_t>(max_slices, static_cast<uint32_t>(s_tab.size() - slice0));
        // bank-aware placement of the window: the entries one gather instruction reads (one
        // element position across the 32 lanes of a slice) go to distinct shared-memory
        // banks where possible; records are rewritten from ranks to slots
        std::vector<uint16_t> slot;
        if (chunk) {  // chunk i -> window floats 4 cs .. 4 cs + 3 (a verbatim 16-byte copy)
            const std::vector<uint16_t> cs = place_chunks(rec, s_tab, slice0, dict_fmt, u, chunks, slot, &max_win);
            // the fill list in slot order: a warp's 16-byte copies land in consecutive smem
            std::vector<uint32_t> ord(cs.size());
            for (uint32_t i = 0; i < ord.size(); ++i) ord[i] = i;
            std::sort(ord.begin(), ord.end(), [&](uint32_t x, uint32_t y) { return cs[x] < cs[y]; });
            const size_t at = u_idx.size() - chunks.size();
            for (size_t i = 0; i < ord.size(); ++i) {
                u_idx[at + i] = chunks[ord[i]];
                u_slot.push_back(cs[ord[i]]);
            }
        } else {
            slot = place_window(rec, s_tab, slice0, dict_fmt, u.size(), &max_win);
            u_slot.insert(u_slot.end(), slot.begin(), slot.end());
        }
        for (size_t sidx = slice0; sidx < s_tab.size(); ++sidx) {
            const uint32_t nq = s_tab[sidx].y & 0xffu;
            uint16_t* cols = reinterpret_cast<uint16_t*>(&rec[s_tab[sidx].x + (dict_fmt ? 4 : nq * 32)]);
            for (uint32_t e = 0; e < nq * 128; ++e) cols[e] = slot[cols[e]];
        }
    }
    std::vector<uint32_t> r_off(G + 1);
    uint32_t max_rows = 0;
    for (uint32_t b = 0; b <= G; ++b) {
        r_off[b] = static_cast<uint32_t>(rb[b]);
        if (b < G) max_rows = std::max<uint32_t>(max_rows, static_cast<uint32_t>(rb[b + 1] - rb[b]));
    }
    if (u_idx.empty()) u_idx.push_back(0);
    if (u_slot.empty()) u_slot.push_back(0);
    if (s_tab.empty()) s_tab.push_back(make_uint4(0, 0, 0, 0));
    if (rec.empty()) rec.resize(1, make_uint4(0, 0, 0, 0));
    if (d_val.empty()) d_val.push_back(0.0f);
    out.G = G;
    out.chunk = chunk;
    out.max_u = max_u;
    out.max_win = std::max(max_win, max_u);
    out.max_rows = max_rows;
    out.max_slices = max_slices;
    out.max_dict = dict_fmt ? max_dict : 0;
    out.r_off.upload(r_off, st);
    out.u_off.upload(u_off, st);
    out.u_idx.upload(u_idx, st);
    out.u_slot.upload(u_slot, st);
    out.s_off.upload(s_off, st);
    out.s_tab.upload(s_tab, st);
    out.d_off.upload(d_off, st);
    out.d_val.upload(d_val, st);
    out.rec.upload(rec, st);
    out.bytes = out.r_off.bytes() + out.u_off.bytes() + out.u_idx.bytes() + out.u_slot.bytes() + out.s_off.bytes() + out.s_tab.bytes() +
                out.d_off.bytes() + out.d_val.bytes() + out.rec.bytes();
    WBX_CUDA(cudaStreamSynchronize(st));
}

WinView view_of(const WinSide& w) {
    WinView v;
    v.u_off = w.u_off.p;
    v.u_idx = w.u_idx.p;
    v.u_slot = w.u_slot.p;
    v.s_off = w.s_off.p;
    v.s_tab = w.s_tab.p;
    v.r_off = w.r_off.p;
    v.d_off = w.d_off.p;
    v.d_val = w.d_val.p;
    v.rec = w.rec.p;
    v.max_u = w.max_u;
    v.max_win = w.max_win;
    v.max_rows = w.max_rows;
    v.max_slices = w.max_slices;
    v.max_dict = w.max_dict;
    v.src_len = w.src_len;
    v.chunk = w.chunk ? 1u : 0u;
    return v;
}

}  // namespace wbx
